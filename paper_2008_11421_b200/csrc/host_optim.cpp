// Host-side SGD / Adam over fp32 master shards: the
// weight update of every block whose gradients leave the GPU.  Compiled with
// -ffp-contract=off so the expression sequence matches kernels.cu exactly.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "optim.hpp"
#include "host_optim.hpp"

namespace krt {

// x86-64: AVX-512 / AVX2 clones picked at load time (ifunc), baseline
// otherwise; every clone evaluates the same IEEE sequence (no contraction), so
// the result does not depend on the host ISA.
#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
#define KRT_SIMD_CLONES __attribute__((target_clones("avx512f", "avx2", "default")))
#else
#define KRT_SIMD_CLONES
#endif

KRT_SIMD_CLONES void host_update_range(float* __restrict p, float* __restrict m, float* __restrict v,
                       const float* __restrict grad, void* weights, int weight_dtype, size_t lo,
                       size_t hi, const OptimScalars& s) {
  const float wd = s.weight_decay, gs = s.grad_scale;
  if (s.optimizer == 1) {
    const float w = s.lerp_w, b2 = s.beta2, omb2 = s.one_m_b2, bc2s = s.bc2_sqrt, eps = s.eps,
                ns = s.neg_step;
    const bool lo_branch = w < 0.5f;
    const float omw = 1.0f - w;
#pragma omp simd
    for (size_t i = lo; i < hi; ++i) {
      float g = grad[i] * gs;
      float pi = p[i];
      if (wd != 0.0f) g = g + wd * pi;
      float mi = m[i];
      float d = g - mi;
      mi = lo_branch ? mi + w * d : g - d * omw;
      float vi = v[i] * b2 + (omb2 * g) * g;
      float denom = std::sqrt(vi) / bc2s + eps;
      pi = pi + ns * (mi / denom);
      m[i] = mi;
      v[i] = vi;
      p[i] = pi;
    }
  } else {
    const float nlr = -s.lr, mom = s.momentum;
#pragma omp simd
    for (size_t i = lo; i < hi; ++i) {
      float g = grad[i] * gs;
      float pi = p[i];
      if (wd != 0.0f) g = g + wd * pi;
      if (mom != 0.0f) {
        float b = s.first_step ? g : m[i] * mom + g;
        m[i] = b;
        g = b;
      }
      p[i] = pi + nlr * g;
    }
  }
  if (weight_dtype == 1) {
    uint16_t* wb = static_cast<uint16_t*>(weights);
    for (size_t i = lo; i < hi; ++i) wb[i] = f32_to_bf16_rne(p[i]);
  } else if (weights != nullptr && weights != (void*)p) {
    std::memcpy(static_cast<float*>(weights) + lo, p + lo, (hi - lo) * sizeof(float));
  }
}

ThreadPool::ThreadPool(int n) : n_(std::max(1, n)) {
  for (int i = 1; i < n_; ++i) workers_.emplace_back([this, i] { loop(i); });
}

ThreadPool::~ThreadPool() {
  {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
  }
  cv_.notify_all();
  for (auto& t : workers_) t.join();
}

void ThreadPool::loop(int id) {
  uint64_t seen = 0;
  for (;;) {
    std::function<void(int)> fn;
    {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      fn = job_;
    }
    fn(id);
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
}

void ThreadPool::run(const std::function<void(int)>& fn) {
  if (n_ == 1) {
    fn(0);
    return;
  }
  {
    std::lock_guard<std::mutex> lk(mu_);
    job_ = fn;
    pending_ = n_ - 1;
    ++gen_;
  }
  cv_.notify_all();
  fn(0);
  std::unique_lock<std::mutex> lk(mu_);
  done_cv_.wait(lk, [&] { return pending_ == 0; });
}

void host_update(ThreadPool* pool, float* p, float* m, float* v, const float* grad, void* weights,
                 int weight_dtype, size_t n, const OptimScalars& s) {
  int nt = pool ? pool->size() : 1;
  // split on 64-element boundaries (cache lines, bf16 pairs)
  size_t chunk = ((n + nt - 1) / nt + 63) / 64 * 64;
  auto body = [&](int t) {
    size_t lo = std::min(n, (size_t)t * chunk), hi = std::min(n, lo + chunk);
    if (lo < hi) host_update_range(p, m, v, grad, weights, weight_dtype, lo, hi, s);
  };
  if (pool && n >= (size_t)1 << 16) pool->run(body);
  else host_update_range(p, m, v, grad, weights, weight_dtype, 0, n, s);
}

}  // namespace krt
