// head_common.cuh — per-position label lookup shared by the softmax-head kernels.
#pragma once
#include <stdint.h>

#include "mpf_internal.h"

namespace mpf {

constexpr int kLabBeyond = -1, kLabPad = -2;

// Label of head position `pos` (fragment-major index inside image `img`): kLabBeyond past
// the image's last position, kLabPad on the padded part of the fragment grid, 255 outside
// the O_H x O_W output grid or unlabelled, else the class.  Training fetches the label
// through the fragment -> pixel map y = r1 + k1 (r2 + k2 (... + kL i)) (R2, R7); the
// forward-only pass returns 0 for every valid position.  Labels >= C raise `a.err`.
__device__ __forceinline__ int head_label(const HeadArgs& a, int img, long long pos, long long per_img, int frag_sz,
                                          bool train) {
  if (pos >= per_img) return kLabBeyond;
  const int gl = (int)(pos / frag_sz);
  const int rem = (int)(pos - (long long)gl * frag_sz);
  const int i = rem / a.gc, j = rem - (rem / a.gc) * a.gc;
  if (i >= a.vr || j >= a.vc) return kLabPad;
  if (!train) return 0;
  int yy = i, xx = j, rf = gl;
  for (int l = a.n_levels - 1; l >= 0; --l) {
    const int kq = a.pool_k[l];
    const int d = rf % (kq * kq);
    rf /= kq * kq;
    yy = d / kq + kq * yy;
    xx = d % kq + kq * xx;
  }
  int lab = 255;
  if (yy < a.O_H && xx < a.O_W) lab = a.labels[((long long)img * a.O_H + yy) * a.O_W + xx];
  if (lab != 255 && lab >= a.C) atomicOr(a.err, 1);
  return lab;
}

// Split form for software pipelining: issue the label load now (`raw`, not yet consumed,
// so the load stays in flight), resolve the code later with head_label_finish.
struct HeadLabel {
  int code;  // >= 0: `raw` holds the label; else kLabBeyond / kLabPad
  int raw;
};
__device__ __forceinline__ HeadLabel head_label_issue(const HeadArgs& a, int img, long long pos, long long per_img,
                                                      int frag_sz) {
  HeadLabel r{kLabBeyond, 255};
  if (pos >= per_img) return r;
  const int gl = (int)(pos / frag_sz);
  const int rem = (int)(pos - (long long)gl * frag_sz);
  const int i = rem / a.gc, j = rem - (rem / a.gc) * a.gc;
  if (i >= a.vr || j >= a.vc) {
    r.code = kLabPad;
    return r;
  }
  int yy = i, xx = j, rf = gl;
  for (int l = a.n_levels - 1; l >= 0; --l) {
    const int kq = a.pool_k[l];
    const int d = rf % (kq * kq);
    rf /= kq * kq;
    yy = d / kq + kq * yy;
    xx = d % kq + kq * xx;
  }
  r.code = 0;
  if (yy < a.O_H && xx < a.O_W) r.raw = __ldg(a.labels + ((long long)img * a.O_H + yy) * a.O_W + xx);
  return r;
}
__device__ __forceinline__ int head_label_finish(const HeadArgs& a, HeadLabel r) {
  if (r.code < 0) return r.code;
  if (r.raw != 255 && r.raw >= a.C) atomicOr(a.err, 1);
  return r.raw;
}

}  // namespace mpf
