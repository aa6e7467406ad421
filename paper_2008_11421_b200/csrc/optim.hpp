// Optimizer arithmetic shared by the host update (the paper's "stand-alone
// direct CPU kernel") and the device update of blocks that
// never leave HBM (distsim.py:14-16: resident blocks update in place).
// Both paths evaluate the same fp32 expression sequence with no FMA
// contraction, so they agree bit for bit.
#pragma once
#include <cmath>
#include <cstdint>

namespace krt {

struct OptimScalars {
  int optimizer;      // 0 SGD, 1 Adam
  float lr, beta1, beta2, eps, weight_decay, momentum;
  float lerp_w;       // 1 - beta1
  float one_m_b2;     // 1 - beta2
  float bc2_sqrt;     // sqrt(1 - beta2^t)   (computed in double, like torch)
  float neg_step;     // -lr / (1 - beta1^t)
  float grad_scale;   // applied to the incoming gradient first
  int first_step;     // SGD momentum buffer initialisation (torch: buf = grad)
};

inline OptimScalars make_scalars(int optimizer, float lr, float b1, float b2, float eps, float wd,
                                 float mom, int step, float grad_scale) {
  OptimScalars s;
  s.optimizer = optimizer;
  s.lr = lr; s.beta1 = b1; s.beta2 = b2; s.eps = eps; s.weight_decay = wd; s.momentum = mom;
  s.lerp_w = (float)(1.0 - (double)b1);
  s.one_m_b2 = (float)(1.0 - (double)b2);
  double bc1 = 1.0 - std::pow((double)b1, step);
  double bc2 = 1.0 - std::pow((double)b2, step);
  s.bc2_sqrt = (float)std::sqrt(bc2);
  s.neg_step = (float)(-(double)lr / bc1);
  s.grad_scale = grad_scale;
  s.first_step = step == 1;
  return s;
}

inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  __builtin_memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);  // quiet NaN
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

}  // namespace krt
