// host_stage.cpp -- pinned bounce staging for pageable host operands (see
// host_stage.h).
#include "host_stage.h"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>

namespace rectri_cu {
namespace {

// FIFO pool of host threads for memcpy pieces.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* pool = new HostPool();  // never destroyed: threads may outlive static teardown
    return *pool;
  }
  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(std::move(f));
    }
    cv_.notify_one();
  }
  int size() const { return static_cast<int>(threads_.size()); }

 private:
  HostPool() {
    const char* e = getenv("RECTRI_CU_HOST_THREADS");
    int n = e ? atoi(e) : static_cast<int>(std::thread::hardware_concurrency());
    n = std::max(1, std::min(n, 32));
    for (int i = 0; i < n; ++i) threads_.emplace_back([this] { run(); });
    for (auto& t : threads_) t.detach();
  }
  void run() {
    for (;;) {
      std::function<void()> f;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [this] { return !q_.empty(); });
        f = std::move(q_.front());
        q_.pop_front();
      }
      f();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  std::vector<std::thread> threads_;
};

// The cached pinned bounce buffers (0: A, 1: B), held for a whole call.
std::mutex g_bounce_mu;
void* g_bounce[2] = {nullptr, nullptr};
size_t g_bounce_bytes[2] = {0, 0};

char* bounce(int k, size_t bytes) {
  if (g_bounce_bytes[k] < bytes) {
    if (g_bounce[k]) cudaFreeHost(g_bounce[k]);
    g_bounce[k] = nullptr;
    g_bounce_bytes[k] = 0;
    if (cudaHostAlloc(&g_bounce[k], bytes, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      throw std::runtime_error("pinned bounce allocation failed");
    }
    g_bounce_bytes[k] = bytes;
  }
  return static_cast<char*>(g_bounce[k]);
}

constexpr size_t kPiece = size_t{4} << 20;  // bytes per memcpy task

// Splits a 2D rectangle (height rows of `width` bytes) into row ranges of
// about kPiece bytes and runs f(row0, row1) for each on the pool.
template <typename F>
int split_rows(size_t width, size_t height, F&& f) {
  const size_t per = std::max<size_t>(1, kPiece / std::max<size_t>(width, 1));
  int pieces = 0;
  for (size_t r0 = 0; r0 < height; r0 += per) {
    const size_t r1 = std::min(height, r0 + per);
    f(r0, r1);
    ++pieces;
  }
  return pieces;
}

void copy_rows(char* dst, size_t dpitch, const char* src, size_t spitch, size_t width, size_t r0, size_t r1) {
  for (size_t r = r0; r < r1; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, width);
}

}  // namespace

struct PageableStager::Ticket {
  std::atomic<int> remaining{0};
  std::mutex mu;
  std::condition_variable cv;
  bool done = false;
  void piece_done() {
    if (remaining.fetch_sub(1) == 1) {
      std::lock_guard<std::mutex> lk(mu);
      done = true;
      cv.notify_all();
    }
  }
  void wait() {
    std::unique_lock<std::mutex> lk(mu);
    cv.wait(lk, [this] { return done; });
  }
};

namespace {
void CUDART_CB wait_ticket(void* p) { static_cast<PageableStager::Ticket*>(p)->wait(); }
}  // namespace

bool is_pageable_host(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

PageableStager::PageableStager(int device, const void* a_base, size_t a_bytes, void* b_base, size_t b_bytes)
    : device_(device), bounce_lock_(g_bounce_mu) {
  if (a_base && a_bytes) a_ = Region{static_cast<const char*>(a_base), bounce(0, a_bytes), a_bytes};
  if (b_base && b_bytes) b_ = Region{static_cast<const char*>(b_base), bounce(1, b_bytes), b_bytes};
  HostPool::get();
  waiter_ = std::thread([this] { waiter_loop(); });
}

PageableStager::~PageableStager() {
  finish();
  for (cudaEvent_t e : events_) cudaEventDestroy(e);
}

const PageableStager::Region* PageableStager::region_of(const void* p) const {
  const char* c = static_cast<const char*>(p);
  if (a_.user && c >= a_.user && c < a_.user + a_.bytes) return &a_;
  if (b_.user && c >= b_.user && c < b_.user + b_.bytes) return &b_;
  return nullptr;
}

bool PageableStager::covers(const void* p) const { return region_of(p) != nullptr; }

void PageableStager::h2d(void* dst_dev, size_t dpitch, const void* src_host, size_t spitch, size_t width,
                         size_t height, cudaStream_t s) {
  const Region* r = region_of(src_host);
  const char* src = static_cast<const char*>(src_host);
  char* bsrc = r->bounce + (src - r->user);
  auto t = std::make_shared<Ticket>();
  tickets_.push_back(t);
  const size_t per = std::max<size_t>(1, kPiece / std::max<size_t>(width, 1));
  t->remaining = static_cast<int>((height + per - 1) / per);
  if (height == 0) {
    t->done = true;
  } else {
    Ticket* tp = t.get();
    split_rows(width, height, [&](size_t r0, size_t r1) {
      HostPool::get().submit([=] {
        copy_rows(bsrc, spitch, src, spitch, width, r0, r1);
        tp->piece_done();
      });
    });
  }
  cudaError_t e = cudaLaunchHostFunc(s, wait_ticket, t.get());
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(dst_dev, dpitch, bsrc, spitch, width, height, cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("staged H2D: ") + cudaGetErrorString(e));
}

void PageableStager::d2h(void* dst_host, size_t dpitch, const void* src_dev, size_t spitch, size_t width,
                         size_t height, cudaStream_t s) {
  const Region* r = region_of(dst_host);
  char* dst = static_cast<char*>(dst_host);
  char* bdst = r->bounce + (dst - r->user);
  cudaEvent_t ev = nullptr;
  cudaError_t e = cudaMemcpy2DAsync(bdst, dpitch, src_dev, spitch, width, height, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev, s);
  if (e != cudaSuccess) throw std::runtime_error(std::string("staged D2H: ") + cudaGetErrorString(e));
  events_.push_back(ev);
  {
    std::lock_guard<std::mutex> lk(mu_);
    backs_.push_back(Back{ev, bdst, dst, dpitch, dpitch, width, height});
    ++outstanding_;  // released when its pieces are queued
  }
  cv_.notify_one();
}

void PageableStager::waiter_loop() {
  cudaSetDevice(device_);
  for (;;) {
    Back b;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [this] { return closing_ || !backs_.empty(); });
      if (backs_.empty()) return;
      b = backs_.front();
      backs_.pop_front();
    }
    cudaEventSynchronize(b.ev);
    const size_t per = std::max<size_t>(1, kPiece / std::max<size_t>(b.width, 1));
    outstanding_ += static_cast<long>((b.height + per - 1) / per);
    split_rows(b.width, b.height, [&](size_t r0, size_t r1) {
      HostPool::get().submit([this, b, r0, r1] {
        copy_rows(b.dst, b.pitch_dst, b.src, b.pitch_src, b.width, r0, r1);
        if (--outstanding_ == 0) {
          std::lock_guard<std::mutex> lk(done_mu_);
          done_cv_.notify_all();
        }
      });
    });
    if (--outstanding_ == 0) {  // this rectangle's own count
      std::lock_guard<std::mutex> lk(done_mu_);
      done_cv_.notify_all();
    }
  }
}

void PageableStager::finish() {
  if (waiter_.joinable()) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      closing_ = true;
    }
    cv_.notify_all();
    waiter_.join();
  }
  std::unique_lock<std::mutex> lk(done_mu_);
  done_cv_.wait(lk, [this] { return outstanding_.load() == 0; });
  // copy-in tickets: the streams were synchronised by the caller, so every
  // host function (and hence every ticket) has completed
}

void release_pageable_bounce() {
  std::lock_guard<std::mutex> lk(g_bounce_mu);
  for (int k = 0; k < 2; ++k) {
    if (g_bounce[k]) cudaFreeHost(g_bounce[k]);
    g_bounce[k] = nullptr;
    g_bounce_bytes[k] = 0;
  }
}

}  // namespace rectri_cu
