// Pageable host memory <-> device transfers through pinned bounce slots (see mk_hoststage.h).
#include "mk_hoststage.h"

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>

namespace mk {

bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // older drivers report unregistered memory as an error
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

namespace {

// Persistent worker pool for row-parallel host copies (the caller's thread works too).
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int n = (int)std::min(8u, hw) - 1;
    for (int i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // f(i) for i in [0, n), spread over the pool; returns when all are done
  void run(int n, const std::function<void(int)>& f) {
    std::lock_guard<std::mutex> one(run_mu_);  // host functions of both streams may call in
    std::unique_lock<std::mutex> lk(m_);
    job_ = &f;
    n_ = n;
    next_ = 0;
    busy_ = (int)th_.size();
    ++gen_;
    lk.unlock();
    cv_.notify_all();
    work();
    lk.lock();
    done_cv_.wait(lk, [this] { return busy_ == 0; });
    job_ = nullptr;
  }

 private:
  void work() {
    for (int i; (i = next_.fetch_add(1)) < n_;) (*job_)(i);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      lk.unlock();
      work();
      lk.lock();
      if (--busy_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex run_mu_, m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* job_ = nullptr;
  std::atomic<int> next_{0};
  int n_ = 0, busy_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

constexpr size_t kSlotBytes = 32u << 20;  // one bounce slot per copy stream

struct Shared {
  std::mutex call_mu;  // one mk_strassen_host call at a time uses the slots
  double* slot[2] = {nullptr, nullptr};
  cudaStream_t second = nullptr;
  int device = -1;
  CopyPool* pool = nullptr;
};
Shared& shared() {
  static Shared s;
  return s;
}

}  // namespace

static void CUDART_CB run_job(void* p) {
  const Stager::Job& j = *static_cast<const Stager::Job*>(p);
  const size_t row_bytes = (size_t)j.cols * sizeof(double);
  const int64_t per = std::max<int64_t>(1, (int64_t)((1u << 20) / std::max<size_t>(row_bytes, 1)));  // ~1 MiB tasks
  const int tasks = (int)((j.rows + per - 1) / per);
  shared().pool->run(tasks, [&](int t) {
    const int64_t r0 = t * per, r1 = std::min(j.rows, r0 + per);
    for (int64_t r = r0; r < r1; ++r) {
      double* pin = j.pinned + r * j.cols;
      double* h = j.host + r * j.hld;
      if (j.up)
        std::memcpy(pin, h, row_bytes);
      else
        std::memcpy(h, pin, row_bytes);
    }
  });
}

bool Stager::prepare(cudaStream_t s0) {
  Shared& sh = shared();
  sh.call_mu.lock();
  int dev = 0;
  cudaGetDevice(&dev);
  if (sh.device != dev) {  // slots and stream belong to one device
    if (sh.second) cudaStreamDestroy(sh.second);
    for (auto& p : sh.slot)
      if (p) cudaFreeHost(p), p = nullptr;
    sh.second = nullptr;
    sh.device = dev;
  }
  bool ok = true;
  for (auto& p : sh.slot)
    if (!p && cudaHostAlloc(reinterpret_cast<void**>(&p), kSlotBytes, cudaHostAllocDefault) != cudaSuccess) {
      p = nullptr;
      ok = false;
    }
  if (ok && !sh.second && cudaStreamCreateWithFlags(&sh.second, cudaStreamNonBlocking) != cudaSuccess) ok = false;
  if (!sh.pool) sh.pool = new CopyPool();  // lives for the process
  if (!ok) {
    cudaGetLastError();
    sh.call_mu.unlock();
    return false;
  }
  s_[0] = s0;  // may be the legacy default stream (0)
  s_[1] = sh.second;
  active_ = true;
  // the second stream starts where the first one is
  cudaEvent_t e;
  if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
    active_ = false;
    sh.call_mu.unlock();
    return false;
  }
  cudaEventRecord(e, s0);
  cudaStreamWaitEvent(s_[1], e, 0);
  temps_.push_back(e);
  return true;
}

cudaError_t Stager::upload(double* dev, int64_t dld, const double* host, int64_t hld, int64_t rows, int64_t cols,
                           cudaEvent_t done) {
  const int64_t per = std::max<int64_t>(1, (int64_t)(kSlotBytes / ((size_t)cols * sizeof(double))));
  int last[2] = {-1, -1};
  for (int64_t r0 = 0; r0 < rows; r0 += per) {
    const int k = next_;
    next_ ^= 1;
    const int64_t nr = std::min(per, rows - r0);
    jobs_.emplace_back(new Job{true, shared().slot[k], const_cast<double*>(host) + r0 * hld, hld, nr, cols});
    cudaError_t e = cudaLaunchHostFunc(s_[k], run_job, jobs_.back().get());
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(dev + r0 * dld, dld * sizeof(double), shared().slot[k], cols * sizeof(double),
                            cols * sizeof(double), nr, cudaMemcpyHostToDevice, s_[k]);
    if (e != cudaSuccess) return e;
    last[k] = 1;
  }
  if (!done) return cudaSuccess;
  // done = both streams past their last chunk of this block
  if (last[0] > 0 && last[1] > 0) {
    cudaEvent_t t;
    cudaError_t e = cudaEventCreateWithFlags(&t, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    temps_.push_back(t);
    const int lastk = next_ ^ 1;  // stream of the block's last chunk
    if ((e = cudaEventRecord(t, s_[lastk ^ 1])) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(s_[lastk], t, 0)) != cudaSuccess) return e;
    return cudaEventRecord(done, s_[lastk]);
  }
  return cudaEventRecord(done, s_[last[0] > 0 ? 0 : 1]);
}

cudaError_t Stager::download(double* host, int64_t hld, const double* dev, int64_t dld, int64_t rows, int64_t cols,
                             cudaEvent_t ready) {
  const int64_t per = std::max<int64_t>(1, (int64_t)(kSlotBytes / ((size_t)cols * sizeof(double))));
  bool waited[2] = {false, false};
  for (int64_t r0 = 0; r0 < rows; r0 += per) {
    const int k = next_;
    next_ ^= 1;
    const int64_t nr = std::min(per, rows - r0);
    cudaError_t e = cudaSuccess;
    if (ready && !waited[k]) {
      e = cudaStreamWaitEvent(s_[k], ready, 0);
      waited[k] = true;
    }
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(shared().slot[k], cols * sizeof(double), dev + r0 * dld, dld * sizeof(double),
                            cols * sizeof(double), nr, cudaMemcpyDeviceToHost, s_[k]);
    if (e != cudaSuccess) return e;
    jobs_.emplace_back(new Job{false, shared().slot[k], host + r0 * hld, hld, nr, cols});
    if ((e = cudaLaunchHostFunc(s_[k], run_job, jobs_.back().get())) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t Stager::finish() {
  cudaError_t e = cudaSuccess;
  if (active_) {
    const cudaError_t e0 = cudaStreamSynchronize(s_[0]);
    const cudaError_t e1 = cudaStreamSynchronize(s_[1]);
    e = e0 != cudaSuccess ? e0 : e1;
    for (cudaEvent_t t : temps_) cudaEventDestroy(t);
    temps_.clear();
    jobs_.clear();
    s_[0] = s_[1] = nullptr;
    active_ = false;
    shared().call_mu.unlock();
  }
  return e;
}

Stager::~Stager() { finish(); }

}  // namespace mk
