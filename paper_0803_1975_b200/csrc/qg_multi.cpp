// qg_multi.cpp — mul_common_compressed over several GPUs of one process
// (the C-ABI entry qg_host_mul_common_multi): rows of A and C
// are sharded over the devices, B is packed once on the first device into the
// tiled layout and broadcast as packed words with one grouped ncclBroadcast
// (NVLink 5 / NVSwitch on a B200 node), every device packs and contracts its
// own row shard. Host buffers in and out, like qg_host_mul_common_gpu.
//
// NCCL is opened with dlopen at the first call (no link-time dependency: a
// process that already loaded libnccl.so.2 — e.g. through torch — shares it).
// Communicators are cached per device list. The one-process-per-GPU
// deployment (bench.py under torchrun) uses torch.distributed for the same
// broadcast (paper_0803_1975_b200/dist.py).
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
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
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
    n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(dlsym(h, "ncclBroadcast"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(h, "ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.CommInitAll && n.Broadcast && n.GroupStart && n.GroupEnd && n.GetErrorString;
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
  const size_t wb = qg_tiled_words(n, k, pl.e, bk);  // packed CB_t words (broadcast size)
  std::vector<DevMem> da(ngpus), dca(ngpus), dcb(ngpus), dc(ngpus), db(1);
  std::vector<cudaStream_t> strm(ngpus, nullptr);
  std::vector<size_t> r0(ngpus), rows(ngpus);
  auto run = [&]() -> int {
    for (int i = 0; i < ngpus; ++i) {
      shard(m, ngpus, i, &r0[i], &rows[i]);
      MQ_CU(cudaSetDevice(devs[i]));
      MQ_CU(cudaStreamCreateWithFlags(&strm[i], cudaStreamNonBlocking));
      da[i].dev = dca[i].dev = dcb[i].dev = dc[i].dev = devs[i];
      MQ_CU(cudaMalloc(&dcb[i].p, wb * 8));
      if (rows[i]) {
        MQ_CU(cudaMalloc(&da[i].p, rows[i] * k * 4));
        MQ_CU(cudaMalloc(&dca[i].p, qg_tiled_words(rows[i], k, pl.e, bk) * 8));
        MQ_CU(cudaMalloc(&dc[i].p, rows[i] * n * 4));
        MQ_CU(cudaMemcpyAsync(da[i].p, a + r0[i] * k, rows[i] * k * 4, cudaMemcpyHostToDevice, strm[i]));
        MQ_TRY(qg_pack_a_tiled(gplan, bk, da[i].p, QG_U32, rows[i], k, k, (double*)dca[i].p, strm[i]));
      }
    }
    // B up and packed once, on the first device
    MQ_CU(cudaSetDevice(devs[0]));
    db[0].dev = devs[0];
    MQ_CU(cudaMalloc(&db[0].p, k * n * 4));
    MQ_CU(cudaMemcpyAsync(db[0].p, b, k * n * 4, cudaMemcpyHostToDevice, strm[0]));
    MQ_TRY(qg_pack_b_tiled(gplan, bk, db[0].p, QG_U32, k, n, n, (double*)dcb[0].p, strm[0]));
    // the packed words to every device (one grouped broadcast)
    MQ_TRY(nccl_status(nc.GroupStart()));
    for (int i = 0; i < ngpus; ++i) {
      const ncclResult_t r = nc.Broadcast(dcb[0].p, dcb[i].p, wb, ncclUint64, 0, (*comms)[i], strm[i]);
      if (r != ncclSuccess) {
        nc.GroupEnd();
        return nccl_status(r);
      }
    }
    MQ_TRY(nccl_status(nc.GroupEnd()));
    for (int i = 0; i < ngpus; ++i) {
      if (!rows[i]) continue;
      MQ_CU(cudaSetDevice(devs[i]));
      MQ_TRY(qg_mul_common_tiled(gplan, (const double*)dca[i].p, (const double*)dcb[i].p, rows[i], n, k,
                                 (int32_t*)dc[i].p, n, strm[i]));
      MQ_CU(cudaMemcpyAsync(c + r0[i] * n, dc[i].p, rows[i] * n * 4, cudaMemcpyDeviceToHost, strm[i]));
    }
    for (int i = 0; i < ngpus; ++i) {
      MQ_CU(cudaSetDevice(devs[i]));
      MQ_CU(cudaStreamSynchronize(strm[i]));
    }
    return QG_OK;
  };
  st = run();
  for (int i = 0; i < ngpus; ++i)
    if (strm[i]) {
      cudaSetDevice(devs[i]);
      cudaStreamSynchronize(strm[i]);
      cudaStreamDestroy(strm[i]);
    }
  cudaSetDevice(caller);
  return st;
}
