// DMMA issue-pattern probe: which part of the contraction mainloop keeps the
// FP64 tensor pipe below peak? One CTA of 8 warps per SM, each warp owning a
// 64x32 tile (32 DMMA.8x8x4 per 4-word k-step), as in qg_dot.cu.
//   P2 regs  : fragments in registers, no loads
//   P3 lds   : fragments loaded from shared memory every k-step (12 LDS.64)
//   P4 sync  : P3 + __syncthreads every 8 k-steps (one pipeline stage)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_pattern_probe dmma_pattern_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE, int MI, int NI, int DATA>
__global__ void __launch_bounds__(256, 1) probe(double* out, int ksteps) {
  extern __shared__ double dyn[];
  double* sA = dyn;              // 128 x 36 (32 k-words + pad)
  double* sB = dyn + 128 * 36;   // 32 x 132
  for (int i = threadIdx.x; i < 128 * 36; i += 256)
    sA[i] = DATA ? (double)((0x9E3779B97F4A7C15ull * (i + 1)) >> 12) : 1e-3 * i;   // ~52-bit integers
  for (int i = threadIdx.x; i < 32 * 132; i += 256)
    sB[i] = DATA ? (double)((0xBF58476D1CE4E5B9ull * (i + 7)) >> 12) : 2e-3 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int wm = warp / 4, wn = warp % 4;
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0;
  double af[MI], bf[NI];
#pragma unroll
  for (int i = 0; i < MI; ++i) af[i] = sA[(wm * 64 + i * 8 + g) * 36 + t];
#pragma unroll
  for (int j = 0; j < NI; ++j) bf[j] = sB[t * 132 + wn * 32 + j * 8 + g];
  for (int ks = 0; ks < ksteps; ks += 8) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      if (MODE >= 3) {
#pragma unroll
        for (int i = 0; i < MI; ++i) af[i] = sA[(wm * 64 + i * 8 + g) * 36 + kk * 4 + t];
#pragma unroll
        for (int j = 0; j < NI; ++j) bf[j] = sB[(kk * 4 + t) * 132 + wn * 32 + j * 8 + g];
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (MODE >= 4) __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) s += acc[i][j][0] + acc[i][j][1];
  if (s == 1.2345) out[0] = s;
}

template <int MODE, int MI, int NI, int DATA = 0>
void run(const char* name, int sms, int threads = 256) {
  double* out;
  cudaMalloc(&out, 8);
  const int ksteps = 8192;
  const int smem = (128 * 36 + 32 * 132) * 8;
  cudaFuncSetAttribute(probe<MODE, MI, NI, DATA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<MODE, MI, NI, DATA><<<sms, threads, smem>>>(out, 64);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<MODE, MI, NI, DATA><<<sms, threads, smem>>>(out, ksteps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 2.0 * 256 * sms * (threads / 32.0) * ksteps * MI * NI;  // 8 warps x 256 FMA x MI*NI per k-step
  printf("{\"threads\": %d, \"data\": %d, \"probe\": \"%s\", \"mi\": %d, \"ni\": %d, \"tflops\": %.3f, \"ms\": %.3f, \"err\": \"%s\"}\n", threads, DATA, name, MI, NI,
         flop / ms / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<2, 8, 4>("regs", sms);
  run<3, 8, 4>("lds", sms);
  run<4, 8, 4>("lds_sync", sms);
  run<2, 8, 4, 1>("regs", sms);
  run<3, 8, 4, 1>("lds", sms);
  run<4, 8, 4, 1>("lds_sync", sms);
  run<2, 8, 4>("regs", sms, 128);
  run<3, 8, 4>("lds", sms, 128);
  run<4, 8, 4>("lds_sync", sms, 128);
  run<2, 4, 4>("regs", sms);
  run<3, 4, 4>("lds", sms);
  run<4, 4, 4>("lds_sync", sms);
  return 0;
}
