// Which integer instruction next to DMMA costs DMMA throughput? NOPS instructions of one kind per DMMA,
// on registers no DMMA writes. 8 warps per SM (2 per SMSP), 64 register-resident accumulators per warp.
// KIND 0: LOP3 (and/xor), 1: add (IADD3 or IMAD.IADD, ptxas's choice), 2: IMAD (mul-add), 3: PRMT, 4: SHF,
// 5: FP32 FADD, 6: FP32 FFMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_int_probe2 tools/dmma_int_probe2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int KIND, int NOPS>
__global__ void __launch_bounds__(256, 1) probe(double* out, int ksteps, uint32_t m1, uint32_t m2) {
  constexpr int MI = 8, NI = 4;
  const int lane = threadIdx.x & 31;
  double acc[MI][NI][2];
  uint32_t x[16];
  float f[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { x[i] = lane * 7 + i; f[i] = lane + i; }
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double af[MI], bf[NI];
#pragma unroll
  for (int i = 0; i < MI; ++i) af[i] = 1e-3 * (lane + i);
#pragma unroll
  for (int j = 0; j < NI; ++j) bf[j] = 2e-3 * (lane + j);
  for (int ks = 0; ks < ksteps; ks += 2) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
#pragma unroll
          for (int q = 0; q < NOPS; ++q) {
            const int r = (i * NI + j + q * 5) % 16;
            if (KIND == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(x[r]) : "r"(m1), "r"(m2));
            if (KIND == 1) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[r]) : "r"(m1));
            if (KIND == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[r]) : "r"(m1), "r"(m2));
            if (KIND == 3) asm volatile("prmt.b32 %0, %0, %1, 0x1032;" : "+r"(x[r]) : "r"(m1));
            if (KIND == 4) asm volatile("shf.l.wrap.b32 %0, %0, %1, 7;" : "+r"(x[r]) : "r"(m1));
            if (KIND == 5) asm volatile("add.f32 %0, %0, %1;" : "+f"(f[r]) : "f"(1.5f));
            if (KIND == 6) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[r]) : "f"(1.0001f), "f"(0.5f));
          }
        }
  }
  double s = 0;
  uint32_t u = 0;
  float g = 0;
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) s += acc[i][j][0] + acc[i][j][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) { u ^= x[i]; g += f[i]; }
  if (s == 1.2345 || u == 0x12345678u || g == 1.25f) out[0] = s + u + g;
}

template <int KIND, int NOPS>
void run(int sms, const char* name) {
  double* out;
  cudaMalloc(&out, 8);
  const int ksteps = 12288;
  auto k = probe<KIND, NOPS>;
  k<<<sms, 256>>>(out, 64, 0x7f80u, 0x1234u);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 256>>>(out, ksteps, 0x7f80u, 0x1234u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flop = 2.0 * 256 * sms * 8.0 * ksteps * 32;
  printf("{\"kind\": \"%s\", \"ops_per_dmma\": %d, \"tflops\": %.3f, \"frac_of_37.09\": %.4f}\n", name, NOPS, flop / ms / 1e9,
         flop / ms / 1e9 / 37.09);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, 0>(sms, "none");
  run<0, 1>(sms, "lop3"); run<0, 2>(sms, "lop3"); run<0, 4>(sms, "lop3");
  run<1, 1>(sms, "add"); run<1, 2>(sms, "add"); run<1, 4>(sms, "add");
  run<2, 1>(sms, "imad"); run<2, 2>(sms, "imad"); run<2, 4>(sms, "imad");
  run<3, 1>(sms, "prmt"); run<3, 2>(sms, "prmt"); run<3, 4>(sms, "prmt");
  run<4, 1>(sms, "shf"); run<4, 2>(sms, "shf"); run<4, 4>(sms, "shf");
  run<5, 1>(sms, "fadd"); run<5, 2>(sms, "fadd"); run<5, 4>(sms, "fadd");
  run<6, 1>(sms, "ffma"); run<6, 2>(sms, "ffma"); run<6, 4>(sms, "ffma");
  return 0;
}
