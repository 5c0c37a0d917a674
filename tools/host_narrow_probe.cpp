// Host-side narrowing bandwidth probe: T threads convert a 128 MiB uint32
// residue buffer (pinned, as the e2e host path sees it) into uint8, and widen
// 64 MiB of uint8 back to uint32. Decides whether narrowing residues before
// the H2D copy (4x fewer PCIe bytes) can beat the PCIe-bound host path.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

static double run(int T, size_t n, const uint32_t* src, uint8_t* dst, bool widen, uint32_t* wout) {
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int i = 0; i < T; ++i)
    th.emplace_back([=] {
      const size_t a = n * i / T, b = n * (i + 1) / T;
      if (!widen)
        for (size_t j = a; j < b; ++j) dst[j] = (uint8_t)src[j];
      else
        for (size_t j = a; j < b; ++j) wout[j] = dst[j];
    });
  for (auto& x : th) x.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
  const size_t n = 32u << 20;  // 32 Mi residues = 128 MiB uint32
  uint32_t *src, *wout;
  uint8_t* dst;
  cudaHostAlloc(&src, n * 4, 0);
  cudaHostAlloc(&dst, n, 0);
  cudaHostAlloc(&wout, n * 4, 0);
  for (size_t i = 0; i < n; ++i) src[i] = (uint32_t)(i * 2654435761u % 7);
  std::memset(dst, 0, n);
  std::memset(wout, 0, n * 4);
  const unsigned hw = std::thread::hardware_concurrency();
  for (int T : {1, 2, 4, 8, 16, 32}) {
    if ((unsigned)T > 2 * hw) break;
    double best = 1e9, bestw = 1e9;
    for (int r = 0; r < 3; ++r) {
      best = std::min(best, run(T, n, src, dst, false, nullptr));
      bestw = std::min(bestw, run(T, n, src, dst, true, wout));
    }
    std::printf("threads %2d narrow %.3f ms (%.1f GB/s of uint32 read)  widen %.3f ms (%.1f GB/s of uint32 written)\n",
                T, best * 1e3, n * 4 / best / 1e9, bestw * 1e3, n * 4 / bestw / 1e9);
  }
  std::printf("hardware_concurrency %u\n", hw);
  return 0;
}
