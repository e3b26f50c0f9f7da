// host_pool.hpp — a small persistent pool of host threads for the staged
// uploads (psg_points.cu h2d_copy): spawning threads per 32 MiB chunk cost
// more than the copies they made.  run(tasks, fn) calls fn(0..tasks-1) on the
// workers and the calling thread and returns when all are done.
#pragma once

#include <algorithm>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace psg {

class HostPool {
 public:
  explicit HostPool(unsigned workers) {
    for (unsigned k = 0; k < workers; ++k) th_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (std::thread& t : th_) t.join();
  }
  unsigned size() const { return static_cast<unsigned>(th_.size()) + 1; }
  void run(unsigned tasks, const std::function<void(unsigned)>& fn) {
    std::unique_lock<std::mutex> g(mu_);
    fn_ = &fn;
    tasks_ = tasks;
    next_ = 0;
    pending_ = tasks;
    ++gen_;
    g.unlock();
    cv_.notify_all();
    work();  // the caller takes tasks too
    g.lock();
    done_cv_.wait(g, [this] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void work() {
    for (;;) {
      unsigned k;
      const std::function<void(unsigned)>* fn;
      {
        std::lock_guard<std::mutex> g(mu_);
        if (!fn_ || next_ >= tasks_) return;
        k = next_++;
        fn = fn_;
      }
      (*fn)(k);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  void loop() {
    unsigned long long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(unsigned)>* fn_ = nullptr;
  unsigned tasks_ = 0, next_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
};

}  // namespace psg
