// host_stage.h -- pinned bounce staging for PAGEABLE host operands.
//
// The reference's callers hand it std::vector-backed MatrixBuffers
// (include/rectri/matrix.hpp:18-70, used by src/bench.cpp:184-192): plain
// pageable memory.  cudaMemcpy*Async from pageable memory is synchronous for
// the calling thread (the driver stages it through its own small pinned
// buffer), which would serialise the streamed host path's enqueue loop on
// every copy.  Instead, every host rectangle the streamed path moves goes
// through a pinned bounce buffer that mirrors the operand's layout:
//   H2D: a pool of host threads memcpy's the rectangle into the bounce
//        buffer (in issue order, split into pieces across the threads); the
//        copy stream waits for it with a host function, then copies
//        bounce -> device asynchronously;
//   D2H: device -> bounce asynchronously, an event after it; a waiter thread
//        hands the rectangle to the pool once the event completes, which
//        memcpy's bounce -> user memory.
// So the host copies run ahead of (H2D) and behind (D2H) the GPU and overlap
// its compute, like the pinned path's transfers.  Pool tasks never block (the
// waiter thread does the event waits), so copy-ins are never stuck behind
// copy-backs.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <deque>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace rectri_cu {

// True when p is host memory the CUDA runtime does not know as pinned.
bool is_pageable_host(const void* p);

class PageableStager {
 public:
  // Regions [base, base + bytes) of the user's host A and B views that are
  // pageable (pass nullptr / 0 for an operand that is not).
  PageableStager(int device, const void* a_base, size_t a_bytes, void* b_base, size_t b_bytes);
  ~PageableStager();
  PageableStager(const PageableStager&) = delete;
  PageableStager& operator=(const PageableStager&) = delete;

  bool covers(const void* p) const;
  // cudaMemcpy2DAsync semantics (pitches and width in bytes, height rows).
  void h2d(void* dst_dev, size_t dpitch, const void* src_host, size_t spitch, size_t width, size_t height,
           cudaStream_t s);
  void d2h(void* dst_host, size_t dpitch, const void* src_dev, size_t spitch, size_t width, size_t height,
           cudaStream_t s);
  // Waits until every copy-back has reached user memory; rethrows nothing
  // (CUDA errors surface through the caller's own stream synchronisation).
  void finish();

  struct Ticket;

 private:
  struct Region {
    const char* user = nullptr;
    char* bounce = nullptr;
    size_t bytes = 0;
  };
  const Region* region_of(const void* p) const;
  void waiter_loop();

  int device_;
  Region a_, b_;
  std::unique_lock<std::mutex> bounce_lock_;  // the global bounce buffers, for this call
  std::vector<std::shared_ptr<Ticket>> tickets_;
  // copy-backs: (event, bounce rectangle, user rectangle)
  struct Back {
    cudaEvent_t ev;
    const char* src;
    char* dst;
    size_t pitch_src, pitch_dst, width, height;
  };
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<Back> backs_;
  bool closing_ = false;
  std::atomic<long> outstanding_{0};  // copy-back pieces not yet written
  std::mutex done_mu_;
  std::condition_variable done_cv_;
  std::thread waiter_;
  std::vector<cudaEvent_t> events_;
};

// Frees the cached pinned bounce buffers (rectri_cu_release_staging).
void release_pageable_bounce();

}  // namespace rectri_cu
