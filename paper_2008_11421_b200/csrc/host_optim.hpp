#pragma once
#include <condition_variable>
#include <cstddef>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "optim.hpp"

namespace krt {

// Fixed fork-join pool: run(fn) calls fn(thread_index) on every thread.
class ThreadPool {
 public:
  explicit ThreadPool(int n);
  ~ThreadPool();
  int size() const { return n_; }
  void run(const std::function<void(int)>& fn);

 private:
  void loop(int id);
  int n_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::function<void(int)> job_;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

void host_update_range(float* p, float* m, float* v, const float* grad, void* weights,
                       int weight_dtype, size_t lo, size_t hi, const OptimScalars& s);
void host_update(ThreadPool* pool, float* p, float* m, float* v, const float* grad, void* weights,
                 int weight_dtype, size_t n, const OptimScalars& s);

}  // namespace krt
