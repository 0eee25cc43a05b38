// egs_pool.h — a process-wide pool of host worker threads for the one-shot
// path's host work (weight narrowing during the upload, measure widening
// during the read-back): spawning 15-16 std::threads per call cost up to a
// millisecond at the ends of the transfer.  One job at a time; a caller that
// finds the pool busy (several ranks of one process uploading at once) gets
// fresh threads instead.  Internal to libegs_b200.so.
#pragma once

#include <unistd.h>

#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace egs_host {

class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  // A running job: fn(t) for t in [0, n) on worker threads; wait() joins it.
  class Job {
   public:
    Job() = default;
    Job(const Job&) = delete;
    Job& operator=(const Job&) = delete;
    ~Job() { wait(); }
    void wait() {
      if (pool_) {
        std::unique_lock<std::mutex> lk(pool_->mu_);
        pool_->done_cv_.wait(lk, [&] { return pool_->running_ == 0; });
        pool_->fn_ = nullptr;
        lk.unlock();
        pool_->busy_.unlock();
        pool_ = nullptr;
      }
      for (auto& th : own_)
        if (th.joinable()) th.join();
      own_.clear();
    }

   private:
    friend class Pool;
    Pool* pool_ = nullptr;
    std::vector<std::thread> own_;
  };

  void launch(Job& job, unsigned n, std::function<void(unsigned)> fn) {
    if (n == 0) return;
    // another caller's job, or a forked child (the workers did not survive
    // the fork): threads of its own
    if (getpid() != pid_ || !busy_.try_lock()) {
      for (unsigned t = 0; t < n; ++t) job.own_.emplace_back(fn, t);
      return;
    }
    std::unique_lock<std::mutex> lk(mu_);
    while (workers_.size() < n) {
      const unsigned id = (unsigned)workers_.size();
      workers_.emplace_back([this, id] { loop(id); });
    }
    fn_ = std::move(fn);
    want_ = n;
    running_ = n;
    ++gen_;
    lk.unlock();
    cv_.notify_all();
    job.pool_ = this;
  }

 private:
  Pool() = default;
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& th : workers_) th.join();
  }
  void loop(unsigned id) {
    unsigned long long seen = 0;
    for (;;) {
      std::function<void(unsigned)>* fn = nullptr;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && id < want_); });
        if (stop_) return;
        seen = gen_;
        fn = &fn_;
      }
      (*fn)(id);
      std::lock_guard<std::mutex> lk(mu_);
      if (--running_ == 0) done_cv_.notify_all();
    }
  }
  const pid_t pid_ = getpid();
  std::mutex busy_;  // held by the running job
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> workers_;
  std::function<void(unsigned)> fn_;
  unsigned want_ = 0, running_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

}  // namespace egs_host
