// qg_stage.cpp — pinned staging of pageable host buffers for the pipelined
// host paths (see qg_stage.h).
#include "qg_stage.h"

#include <cstring>
#include <functional>

namespace qg {

bool host_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // an unknown pointer is pageable: clear the sticky query error
    return false;
  }
  return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeManaged;
}

namespace {

// A small process-wide pool that runs one parallel copy at a time per caller:
// the rows of a 2-D copy are split into contiguous ranges, one per worker.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  void copy2d(char* dst, size_t dpitch, const char* src, size_t spitch, size_t width, size_t rows) {
    const size_t bytes = width * rows;
    const int parts = bytes < (size_t(1) << 20) ? 1 : nthreads_;
    if (parts <= 1 || rows == 0) {
      rows2d(dst, dpitch, src, spitch, width, 0, rows, rows);
      return;
    }
    // split by rows when there are enough, else split a single row by bytes;
    // `left` is decremented under `m` so the waiter cannot return (and destroy
    // m / done) before the last worker has released them
    int left = parts;
    std::mutex m;
    std::condition_variable done;
    for (int i = 0; i < parts; ++i) {
      submit([=, &left, &m, &done] {
        if (rows >= (size_t)parts) {
          rows2d(dst, dpitch, src, spitch, width, rows * i / parts, rows * (i + 1) / parts, rows);
        } else {
          for (size_t r = 0; r < rows; ++r) {
            const size_t b0 = width * i / parts, b1 = width * (i + 1) / parts;
            std::memcpy(dst + r * dpitch + b0, src + r * spitch + b0, b1 - b0);
          }
        }
        std::lock_guard<std::mutex> lk(m);
        if (--left == 0) done.notify_all();
      });
    }
    std::unique_lock<std::mutex> lk(m);
    done.wait(lk, [&] { return left == 0; });
  }

 private:
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    nthreads_ = (int)(hw >= 16 ? 8 : (hw >= 4 ? hw / 2 : 1));
    for (int i = 0; i < nthreads_; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  static void rows2d(char* dst, size_t dpitch, const char* src, size_t spitch, size_t width, size_t r0, size_t r1,
                     size_t) {
    if (dpitch == width && spitch == width) {
      std::memcpy(dst + r0 * width, src + r0 * width, (r1 - r0) * width);
      return;
    }
    for (size_t r = r0; r < r1; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, width);
  }
  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      jobs_.push_back(std::move(f));
    }
    cv_.notify_one();
  }
  void loop() {
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
        if (stop_ && jobs_.empty()) return;
        f = std::move(jobs_.front());
        jobs_.pop_front();
      }
      f();
    }
  }
  int nthreads_ = 1;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> jobs_;
  bool stop_ = false;
};

}  // namespace

HostStager::HostStager() : in_(kSlots), out_(kSlots) {}

HostStager::~HostStager() {
  if (drainer_.joinable()) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    drainer_.join();
  }
  for (auto* v : {&in_, &out_})
    for (Slot& s : *v) {
      if (s.buf) cudaFreeHost(s.buf);
      if (s.done) cudaEventDestroy(s.done);
    }
}

bool HostStager::ensure() {
  if (ready_) return true;
  for (auto* v : {&in_, &out_})
    for (Slot& s : *v) {
      if (!s.buf && cudaHostAlloc(reinterpret_cast<void**>(&s.buf), kSlotBytes, cudaHostAllocDefault) != cudaSuccess)
        return false;
      if (!s.done && cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming) != cudaSuccess) return false;
    }
  drainer_ = std::thread([this] { drain_loop(); });
  ready_ = true;
  return true;
}

cudaError_t HostStager::h2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                            cudaStream_t s) {
  if (width == 0 || height == 0) return cudaSuccess;
  if (host_pinned(src))
    return height == 1 ? cudaMemcpyAsync(dst, src, width, cudaMemcpyHostToDevice, s)
                       : cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyHostToDevice, s);
  if (!ensure()) return cudaErrorMemoryAllocation;
  // pieces of whole rows (a row wider than a slot goes in column pieces)
  const size_t rows_per = width <= kSlotBytes ? kSlotBytes / width : 0;
  for (size_t r0 = 0; r0 < height;) {
    Slot& sl = in_[next_in_];
    next_in_ = (next_in_ + 1) % kSlots;
    cudaError_t e = cudaEventSynchronize(sl.done);  // its previous DMA has read it
    if (e != cudaSuccess) return e;
    if (rows_per) {
      const size_t rows = (height - r0) < rows_per ? (height - r0) : rows_per;
      CopyPool::get().copy2d(sl.buf, width, static_cast<const char*>(src) + r0 * spitch, spitch, width, rows);
      e = rows == 1 || dpitch == width
              ? cudaMemcpyAsync(static_cast<char*>(dst) + r0 * dpitch, sl.buf, rows * width, cudaMemcpyHostToDevice, s)
              : cudaMemcpy2DAsync(static_cast<char*>(dst) + r0 * dpitch, dpitch, sl.buf, width, width, rows,
                                  cudaMemcpyHostToDevice, s);
      r0 += rows;
      if (e == cudaSuccess) e = cudaEventRecord(sl.done, s);
      if (e != cudaSuccess) return e;
    } else {  // one very wide row, in slot-sized column pieces
      for (size_t c0 = 0; c0 < width; c0 += kSlotBytes) {
        Slot& sc = c0 ? in_[next_in_] : sl;
        if (c0) {
          next_in_ = (next_in_ + 1) % kSlots;
          if ((e = cudaEventSynchronize(sc.done)) != cudaSuccess) return e;
        }
        const size_t w = (width - c0) < kSlotBytes ? (width - c0) : kSlotBytes;
        CopyPool::get().copy2d(sc.buf, w, static_cast<const char*>(src) + r0 * spitch + c0, spitch, w, 1);
        e = cudaMemcpyAsync(static_cast<char*>(dst) + r0 * dpitch + c0, sc.buf, w, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaEventRecord(sc.done, s);
        if (e != cudaSuccess) return e;
      }
      ++r0;
    }
  }
  return cudaSuccess;
}

HostStager::Slot* HostStager::acquire_out() {
  Slot* sl = &out_[next_out_];
  next_out_ = (next_out_ + 1) % kSlots;
  std::unique_lock<std::mutex> lk(mu_);
  cv_.wait(lk, [&] { return !sl->busy; });
  sl->busy = true;
  return sl;
}

cudaError_t HostStager::d2h(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                            cudaStream_t s) {
  if (width == 0 || height == 0) return cudaSuccess;
  if (host_pinned(dst))
    return height == 1 ? cudaMemcpyAsync(dst, src, width, cudaMemcpyDeviceToHost, s)
                       : cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost, s);
  if (!ensure()) return cudaErrorMemoryAllocation;
  const size_t rows_per = width <= kSlotBytes ? kSlotBytes / width : 0;
  if (!rows_per) {  // a row wider than a slot: no staging (rare; synchronous driver copy)
    return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToHost, s);
  }
  for (size_t r0 = 0; r0 < height;) {
    const size_t rows = (height - r0) < rows_per ? (height - r0) : rows_per;
    Slot* sl = acquire_out();
    cudaError_t e = rows == 1 || spitch == width
                        ? cudaMemcpyAsync(sl->buf, static_cast<const char*>(src) + r0 * spitch, rows * width,
                                          cudaMemcpyDeviceToHost, s)
                        : cudaMemcpy2DAsync(sl->buf, width, static_cast<const char*>(src) + r0 * spitch, spitch, width,
                                            rows, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaEventRecord(sl->done, s);
    if (e != cudaSuccess) {
      std::lock_guard<std::mutex> lk(mu_);
      sl->busy = false;
      return e;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      queue_.push_back(Drain{sl, static_cast<char*>(dst) + r0 * dpitch, dpitch, width, rows});
      ++pending_;
    }
    cv_.notify_all();
    r0 += rows;
  }
  return cudaSuccess;
}

void HostStager::drain_loop() {
  for (;;) {
    Drain d;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || !queue_.empty(); });
      if (queue_.empty()) return;
      d = queue_.front();
      queue_.pop_front();
    }
    cudaError_t e = cudaEventSynchronize(d.slot->done);
    if (e == cudaSuccess) CopyPool::get().copy2d(d.dst, d.dpitch, d.slot->buf, d.width, d.width, d.rows);
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (e != cudaSuccess && drain_error_ == cudaSuccess) drain_error_ = e;
      d.slot->busy = false;
      --pending_;
    }
    cv_.notify_all();
  }
}

cudaError_t HostStager::finish() {
  std::unique_lock<std::mutex> lk(mu_);
  cv_.wait(lk, [&] { return pending_ == 0; });
  const cudaError_t e = drain_error_;
  drain_error_ = cudaSuccess;
  return e;
}

}  // namespace qg
