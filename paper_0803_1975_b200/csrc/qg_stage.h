// qg_stage.h — host<->device copies of the pipelined host paths for PAGEABLE
// host buffers (a reference caller's std::vector, matrix.hpp:14-26).
//
// cudaMemcpyAsync from pageable memory is staged by the driver and blocks the
// calling thread, so a pipeline that enqueues its transfers ahead of its
// kernels serialises (config 5 e2e: 1.45 s pageable vs 0.39 s pinned, r2).
// HostStager keeps a ring of pinned slots per (thread, device):
//   H2D: the caller's thread copies a piece of the pageable source into a free
//        slot (parallel memcpy over a small worker pool), then queues the
//        async DMA slot -> device on the pipeline's stream;
//   D2H: the DMA device -> slot is queued on the stream; a drain thread waits
//        for it and copies the slot into the pageable destination, so the
//        pipeline thread keeps enqueueing.
// Pinned sources / destinations bypass the slots (plain async copies).
#pragma once
#include <condition_variable>
#include <cstddef>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

namespace qg {

bool host_pinned(const void* p);

class HostStager {
 public:
  HostStager();
  ~HostStager();
  HostStager(const HostStager&) = delete;
  HostStager& operator=(const HostStager&) = delete;
  // 2-D copies (width bytes x height rows); 1-D is height 1
  cudaError_t h2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                  cudaStream_t s);
  cudaError_t d2h(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                  cudaStream_t s);
  // waits until every staged D2H of this call has reached its destination
  cudaError_t finish();

 private:
  struct Slot {
    char* buf = nullptr;
    cudaEvent_t done = nullptr;  // DMA that last used the slot
    bool busy = false;           // D2H slot: waiting for the drain thread
  };
  struct Drain {
    Slot* slot;
    char* dst;
    size_t dpitch, width, rows;
  };
  bool ensure();
  Slot* acquire_out();
  void drain_loop();

  static constexpr size_t kSlotBytes = size_t(32) << 20;
  static constexpr int kSlots = 4;
  std::vector<Slot> in_, out_;
  int next_in_ = 0, next_out_ = 0;
  bool ready_ = false;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Drain> queue_;
  size_t pending_ = 0;
  cudaError_t drain_error_ = cudaSuccess;
  bool stop_ = false;
  std::thread drainer_;
};

}  // namespace qg
