// Throughput of the FP64 mma.sync shapes on sm_100a: m8n8k4 (the contraction's
// DMMA.8x8x4) against m16n8k4, m16n8k8 and m16n8k16 (PTX f64 shapes for
// sm_90+), register-resident, full chip. Prints TFLOP/s per shape and the SASS
// opcode is checked separately with cuobjdump.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_shapes_probe dmma_shapes_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void k884(double* out, int iters, double seed) {
  double acc[NACC][2] = {};
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5 + threadIdx.x * 1e-10;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1];
  if (s == 123.456) out[0] = s;
}
template <int NACC>
__global__ void k1684(double* out, int iters, double seed) {
  double acc[NACC][4] = {};
  double a0 = seed + threadIdx.x * 1e-9, a1 = a0 * 0.7, b = seed * 0.5 + threadIdx.x * 1e-10;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3]) : "d"(a0), "d"(a1), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 123.456) out[0] = s;
}
template <int NACC>
__global__ void k1688(double* out, int iters, double seed) {
  double acc[NACC][4] = {};
  double a0 = seed + threadIdx.x * 1e-9, a1 = a0 * 0.7, a2 = a0 * 0.3, a3 = a0 * 0.9, b0 = seed * 0.5, b1 = b0 * 0.6;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 123.456) out[0] = s;
}
template <int NACC>
__global__ void k16816(double* out, int iters, double seed) {
  double acc[NACC][4] = {};
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 1e-9 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = seed * 0.5 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 123.456) out[0] = s;
}

template <typename K>
static void run(const char* name, K kern, double flop_per_mma, int nacc, int warps) {
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  kern<<<sms, warps * 32>>>(out, 100, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<sms, warps * 32>>>(out, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = (double)sms * warps * iters * nacc * flop_per_mma;
  printf("%-10s warps/SM %2d acc %d: %.2f TFLOP/s\n", name, warps, nacc, flop / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  // one warp per SMSP (4 per SM) with the contraction's 32 independent
  // accumulators per k-step, against two per SMSP
  for (int w : {4, 8}) run("m8n8k4", k884<32>, 2.0 * 8 * 8 * 4, 32, w);
  for (int w : {8, 16}) {
    run("m8n8k4", k884<8>, 2.0 * 8 * 8 * 4, 8, w);
    run("m16n8k4", k1684<8>, 2.0 * 16 * 8 * 4, 8, w);
    run("m16n8k8", k1688<8>, 2.0 * 16 * 8 * 8, 8, w);
    run("m16n8k16", k16816<8>, 2.0 * 16 * 8 * 16, 8, w);
  }
  return 0;
}
