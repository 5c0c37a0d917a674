// K4A flush pattern vs warps per SMSP: register-resident fragments, MI x NI DMMA tiles per warp, every
// accumulator row mi restarts from a constant C quad at k-step mi % FLUSH of every FLUSH k-steps after
// its low word was masked into a digit sum (LOP3 + IADD). FLUSH = 0: plain accumulation.
//   8 warps x (8 x 4) = the shipped warp tile (64 x 32), 2 warps per SMSP
//  16 warps x (4 x 4) = 32 x 32 warp tiles, 4 warps per SMSP
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_flush_probe tools/dmma_flush_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int WARPS, int MI, int NI, int FLUSH>
__global__ void __launch_bounds__(WARPS * 32, 1) probe(double* out, int ksteps, uint32_t mask, double c0, double c1) {
  const int lane = threadIdx.x & 31;
  double acc[MI][NI][2];
  uint32_t ds[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      acc[i][j][0] = c0;
      acc[i][j][1] = c1;
      ds[i][j][0] = ds[i][j][1] = 0;
    }
  double af[MI], bf[NI];
#pragma unroll
  for (int i = 0; i < MI; ++i) af[i] = 1e-3 * (lane + i);
#pragma unroll
  for (int j = 0; j < NI; ++j) bf[j] = 2e-3 * (lane + j);
  constexpr int UNROLL = FLUSH > 0 ? FLUSH : 3;
  for (int ks = 0; ks < ksteps; ks += UNROLL) {
#pragma unroll
    for (int kk = 0; kk < UNROLL; ++kk)
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          if (FLUSH > 0 && kk == i % FLUSH) {
            ds[i][j][0] += (uint32_t)__double2loint(acc[i][j][0]) & mask;
            ds[i][j][1] += (uint32_t)__double2loint(acc[i][j][1]) & mask;
            dmma_c(acc[i][j][0], acc[i][j][1], af[i], bf[j], c0, c1);
          } else {
            dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
          }
        }
  }
  double s = 0;
  uint32_t u = 0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      s += acc[i][j][0] + acc[i][j][1];
      u += ds[i][j][0] ^ ds[i][j][1];
    }
  if (s == 1.2345 || u == 0x12345678u) out[0] = s + u;
}

template <int WARPS, int MI, int NI, int FLUSH>
void run(int sms) {
  double* out;
  cudaMalloc(&out, 8);
  const int ksteps = 12288;
  auto k = probe<WARPS, MI, NI, FLUSH>;
  k<<<sms, WARPS * 32>>>(out, 48, 0x7f80u, 1.5 * 0x1p85, 1.5 * 0x1p85 + 0x1p48);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, WARPS * 32>>>(out, ksteps, 0x7f80u, 1.5 * 0x1p85, 1.5 * 0x1p85 + 0x1p48);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 2.0 * 256 * sms * (double)WARPS * ksteps * MI * NI;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  printf("{\"warps\": %d, \"tile\": \"%dx%d\", \"flush_every_ksteps\": %d, \"regs\": %d, \"spill_bytes\": %zu, \"tflops\": %.3f, \"frac_of_37.09\": %.4f, \"err\": \"%s\"}\n",
         WARPS, MI * 8, NI * 8, FLUSH, fa.numRegs, fa.localSizeBytes, flop / ms / 1e9, flop / ms / 1e9 / 37.09,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<8, 8, 4, 0>(sms);
  run<8, 8, 4, 3>(sms);
  run<8, 8, 4, 7>(sms);
  run<16, 4, 4, 0>(sms);
  run<16, 4, 4, 3>(sms);
  run<16, 4, 4, 7>(sms);
  run<16, 8, 2, 3>(sms);
  run<12, 8, 4, 3>(sms);
  return 0;
}
