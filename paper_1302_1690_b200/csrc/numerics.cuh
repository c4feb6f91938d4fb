// numerics.cuh — the device arithmetic shared by every libmpf kernel: TF32 operand rounding
// and the SFU activations.  One definition, so that every producer of a tensor-core operand
// rounds the same way (DESIGN.md §7 "Precision").
#pragma once
#include <math.h>
#include <stdint.h>

namespace mpf {

// TF32 rounding of an MMA operand, nearest-even, as one F2FP instruction on sm_100a
// (cvt.rn.satfinite; the guarded cvt.rna form takes four).  satfinite clamps +-Inf to
// +-MAX_TF32: use this form only where the value is bounded by construction (the head's dh:
// softmax probabilities times W_L times act', finite whenever the loss is).
__device__ __forceinline__ float tf32_rn_sat(float x) {
  uint32_t r;
  asm("cvt.rn.satfinite.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// The same rounding with +-Inf kept (two more instructions): an overflow in an activation,
// a delta or a weight stays non-finite, so the loss / gradient checks of the line searches
// see it.  NaN stays NaN in both forms.
__device__ __forceinline__ float tf32_rn(float x) {
  const float r = tf32_rn_sat(x);
  return fabsf(x) == INFINITY ? x : r;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// branch-free SFU tanh: 1 - 2 / (2^(2 v log2 e) + 1), absolute error ~1e-7 (far below the
// TF32 rounding of every tensor-core operand); saturates to +-1 at +-inf
__device__ __forceinline__ float fast_tanh(float v) {
  return fmaf(-2.f, rcp_approx(ex2_approx(2.8853900817779268f * v) + 1.f), 1.f);
}
__device__ __forceinline__ float fast_logistic(float v) { return rcp_approx(1.f + ex2_approx(-1.4426950408889634f * v)); }

}  // namespace mpf
