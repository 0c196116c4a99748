// Pageable host memory <-> device transfers for the overlapped host path (mk_strassen_host).
//
// A plain numpy array is pageable: cudaMemcpyAsync from it is staged by the driver one
// buffer at a time on the calling thread (~11 GB/s measured) and cannot overlap compute.
// The Stager moves each block through small pinned bounce slots instead: the whole
// transfer schedule is enqueued up front on two alternating copy streams as
//   [host function: parallel memcpy pageable -> slot] [DMA slot -> device] [event]
// (uploads) and [wait event] [DMA device -> slot] [host function: slot -> pageable]
// (downloads). The host functions run on the driver's callback thread and split their rows
// over a persistent thread pool; while one stream's DMA runs, the other stream's host copy
// fills the next slot, so PCIe and host memory bandwidth overlap.
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

namespace mk {

// Whether p points to pageable (unregistered) host memory.
bool is_pageable(const void* p);

class Stager {
 public:
  // Prepare for one mk_strassen_host call whose first copy stream is `s0`; allocates (or
  // reuses) the pinned slots and the second stream. False if pinned memory is unavailable.
  bool prepare(cudaStream_t s0);
  // Enqueue an upload of a rows x cols block (host leading dimension hld, device dld);
  // `done` (may be null) is recorded once the whole block is on the device.
  cudaError_t upload(double* dev, int64_t dld, const double* host, int64_t hld, int64_t rows, int64_t cols,
                     cudaEvent_t done);
  // Enqueue a download of a rows x cols block once `ready` (may be null) has completed.
  cudaError_t download(double* host, int64_t hld, const double* dev, int64_t dld, int64_t rows, int64_t cols,
                       cudaEvent_t ready);
  // Wait for every enqueued transfer; releases per-call state.
  cudaError_t finish();
  ~Stager();

  struct Job {  // one chunk: rows x cols between a bounce slot and the pageable host block
    bool up;
    double* pinned;
    double* host;
    int64_t hld, rows, cols;
  };

 private:
  cudaStream_t s_[2] = {nullptr, nullptr};
  bool active_ = false;  // between a successful prepare() and finish()
  int next_ = 0;  // stream / slot of the next chunk
  std::vector<std::unique_ptr<Job>> jobs_;
  std::vector<cudaEvent_t> temps_;
};

}  // namespace mk
