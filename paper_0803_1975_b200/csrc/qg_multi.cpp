// qg_multi.cpp — mul_common_compressed over several GPUs of one process
// (the C-ABI entry qg_host_mul_common_multi): rows of A and C
// are sharded over the devices; the right operand is assembled by an
// all-gather: device i uploads and packs only its own tile-column slot of B
// (compress_cols_forward is column-separable, gemm.hpp:122-140) and one
// grouped in-place ncclAllGather (NVLink 5 / NVSwitch on a B200 node) gives
// every device the whole packed CB_t, so every PCIe link carries 1/N of B.
// Each device uploads and packs its A shard on a second stream meanwhile,
// contracts its own slot's columns as soon as they are packed, and the rest
// once the gather has landed. Host buffers in and out, like
// qg_host_mul_common_gpu.
//
// NCCL is opened with dlopen at the first call (no link-time dependency: a
// process that already loaded libnccl.so.2 — e.g. through torch — shares it).
// Communicators are cached per device list. The one-process-per-GPU
// deployment (bench.py under torchrun) does the same all-gather through
// torch.distributed (paper_0803_1975_b200/dist.py).
#include <dlfcn.h>

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/qgemm_b200.h"
#include "qg_internal.h"

namespace {

// the few NCCL entry points used here (nccl.h ABI)
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
enum { ncclSuccess = 0, ncclUint64 = 5 };
struct Nccl {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(dlsym(h, "ncclCommInitAll"));
    n.AllGather = reinterpret_cast<decltype(n.AllGather)>(dlsym(h, "ncclAllGather"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(h, "ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.CommInitAll && n.AllGather && n.GroupStart && n.GroupEnd && n.GetErrorString;
    if (!n.ok) n.why = "libnccl.so.2 lacks an entry point";
  });
  return n;
}

int nccl_status(ncclResult_t r) {
  if (r == ncclSuccess) return QG_OK;
  return qg::fail(QG_NCCL_ERROR, std::string("NCCL: ") + nccl().GetErrorString(r));
}
int cuda_st(cudaError_t e) {
  if (e == cudaSuccess) return QG_OK;
  return qg::fail(QG_CUDA_ERROR, cudaGetErrorString(e));
}
#define MQ_TRY(x)                      \
  do {                                 \
    int st_ = (x);                     \
    if (st_ != QG_OK) return st_;      \
  } while (0)
#define MQ_CU(x) MQ_TRY(cuda_st(x))

std::vector<ncclComm_t>* comms_for(const std::vector<int>& devs, int* status) {
  static std::mutex mu;
  static std::map<std::vector<int>, std::vector<ncclComm_t>> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(devs);
  if (it != cache.end()) return &it->second;
  std::vector<ncclComm_t> c(devs.size(), nullptr);
  *status = nccl_status(nccl().CommInitAll(c.data(), (int)devs.size(), devs.data()));
  if (*status) return nullptr;
  return &(cache[devs] = c);
}

// balanced contiguous row shard, a multiple of 128 rows except the last
void shard(size_t m, int world, int r, size_t* row0, size_t* rows) {
  const size_t blocks = (m + 127) / 128, base = blocks / world, extra = blocks % world;
  const size_t b0 = r * base + (r < (int)extra ? r : extra), nb = base + (r < (int)extra ? 1 : 0);
  *row0 = b0 * 128 < m ? b0 * 128 : m;
  const size_t end = (b0 + nb) * 128 < m ? (b0 + nb) * 128 : m;
  *rows = end - *row0;
}

struct DevMem {
  void* p = nullptr;
  int dev = 0;
  ~DevMem() {
    if (p) {
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(dev);
      cudaFree(p);
      cudaSetDevice(cur);
    }
  }
};

}  // namespace

extern "C" int qg_host_mul_common_multi(const qg_gpu_plan* gplan, const int* devices, int ngpus, const uint32_t* a,
                                        const uint32_t* b, size_t m, size_t k, size_t n, uint32_t* c) {
  if (!gplan || !devices || ngpus < 1 || (m * k && !a) || (k * n && !b) || (m * n && !c)) return QG_INVALID_ARGUMENT;
  const qg_plan& pl = gplan->plan;
  if (pl.e < 1 || pl.t < 1 || pl.t > 31) return QG_PLAN_MISMATCH;
  if (m == 0 || n == 0) return QG_OK;
  if (k == 0) {
    std::memset(c, 0, m * n * sizeof(uint32_t));
    return QG_OK;
  }
  Nccl& nc = nccl();
  if (!nc.ok) return qg::fail(QG_NCCL_ERROR, nc.why);
  uint32_t bk = 0;
  MQ_TRY(qg_tiled_stage_words(gplan, k, &bk));
  const std::vector<int> devs(devices, devices + ngpus);
  int st = QG_OK;
  std::vector<ncclComm_t>* comms = comms_for(devs, &st);
  if (!comms) return st;
  int caller = 0;
  MQ_CU(cudaGetDevice(&caller));
  // gathered CB_t: ngpus equal slots of P tile columns (W words per tile column)
  const size_t W = qg_tiled_words(128, k, pl.e, bk), Nt = (n + 127) / 128, P = (Nt + ngpus - 1) / ngpus;
  const size_t slot_words = P * W;
  std::vector<DevMem> da(ngpus), dca(ngpus), dcb(ngpus), dc(ngpus);
  std::vector<cudaStream_t> sa(ngpus, nullptr), sb(ngpus, nullptr);
  std::vector<cudaEvent_t> own(ngpus, nullptr), all(ngpus, nullptr);
  std::vector<size_t> r0(ngpus), rows(ngpus), t0(ngpus), t1(ngpus);
  // contract tile columns [u0, u1) of device i's rows against its CB_t
  auto contract = [&](int i, size_t u0, size_t u1) -> int {
    const size_t c0 = u0 * 128, c1 = u1 * 128 < n ? u1 * 128 : n;
    if (c1 <= c0 || !rows[i]) return QG_OK;
    return qg_mul_common_tiled(gplan, (const double*)dca[i].p, (const double*)dcb[i].p + u0 * W, rows[i], c1 - c0, k,
                               (int32_t*)dc[i].p + c0, n, sa[i]);
  };
  auto run = [&]() -> int {
    for (int i = 0; i < ngpus; ++i) {
      shard(m, ngpus, i, &r0[i], &rows[i]);
      t0[i] = (size_t)i * P < Nt ? (size_t)i * P : Nt;
      t1[i] = t0[i] + P < Nt ? t0[i] + P : Nt;
      MQ_CU(cudaSetDevice(devs[i]));
      MQ_CU(cudaStreamCreateWithFlags(&sa[i], cudaStreamNonBlocking));
      MQ_CU(cudaStreamCreateWithFlags(&sb[i], cudaStreamNonBlocking));
      MQ_CU(cudaEventCreateWithFlags(&own[i], cudaEventDisableTiming));
      MQ_CU(cudaEventCreateWithFlags(&all[i], cudaEventDisableTiming));
      da[i].dev = dca[i].dev = dcb[i].dev = dc[i].dev = devs[i];
      MQ_CU(cudaMalloc(&dcb[i].p, ngpus * slot_words * 8));
      // this device's slot of B: up (2-D copy of its columns) and packed on sb
      const size_t bc0 = t0[i] * 128 < n ? t0[i] * 128 : n, bc1 = t1[i] * 128 < n ? t1[i] * 128 : n;
      MQ_TRY(qg_host_pack_b_slot_tiled(gplan, bk, b, n, k, bc0, bc1 - bc0, (double*)dcb[i].p + i * slot_words, sb[i]));
      MQ_CU(cudaEventRecord(own[i], sb[i]));
      if (rows[i]) {  // the A shard up and packed on sa meanwhile
        MQ_CU(cudaMalloc(&da[i].p, rows[i] * k * 4));
        MQ_CU(cudaMalloc(&dca[i].p, qg_tiled_words(rows[i], k, pl.e, bk) * 8));
        MQ_CU(cudaMalloc(&dc[i].p, rows[i] * n * 4));
        MQ_CU(cudaMemcpyAsync(da[i].p, a + r0[i] * k, rows[i] * k * 4, cudaMemcpyHostToDevice, sa[i]));
        MQ_TRY(qg_pack_a_tiled(gplan, bk, da[i].p, QG_U32, rows[i], k, k, (double*)dca[i].p, sa[i]));
      }
    }
    // every slot to every device: one grouped in-place all-gather on the sb streams
    MQ_TRY(nccl_status(nc.GroupStart()));
    for (int i = 0; i < ngpus; ++i) {
      const ncclResult_t r = nc.AllGather((const double*)dcb[i].p + i * slot_words, dcb[i].p, slot_words, ncclUint64,
                                          (*comms)[i], sb[i]);
      if (r != ncclSuccess) {
        nc.GroupEnd();
        return nccl_status(r);
      }
    }
    MQ_TRY(nccl_status(nc.GroupEnd()));
    for (int i = 0; i < ngpus; ++i) {
      MQ_CU(cudaSetDevice(devs[i]));
      MQ_CU(cudaEventRecord(all[i], sb[i]));
      // own columns first (local as soon as packed), the rest after the gather
      MQ_CU(cudaStreamWaitEvent(sa[i], own[i], 0));
      MQ_TRY(contract(i, t0[i], t1[i]));
      MQ_CU(cudaStreamWaitEvent(sa[i], all[i], 0));
      MQ_TRY(contract(i, t1[i], Nt));
      MQ_TRY(contract(i, 0, t0[i]));
      if (rows[i]) MQ_CU(cudaMemcpyAsync(c + r0[i] * n, dc[i].p, rows[i] * n * 4, cudaMemcpyDeviceToHost, sa[i]));
    }
    for (int i = 0; i < ngpus; ++i) {
      MQ_CU(cudaSetDevice(devs[i]));
      MQ_CU(cudaStreamSynchronize(sa[i]));
      MQ_CU(cudaStreamSynchronize(sb[i]));
    }
    return QG_OK;
  };
  st = run();
  for (int i = 0; i < ngpus; ++i) {
    cudaSetDevice(devs[i]);
    for (cudaStream_t x : {sa[i], sb[i]})
      if (x) {
        cudaStreamSynchronize(x);
        cudaStreamDestroy(x);
      }
    for (cudaEvent_t x : {own[i], all[i]})
      if (x) cudaEventDestroy(x);
  }
  cudaSetDevice(caller);
  return st;
}
