// conv_tc.h — tensor-core (tcgen05 / TMEM, kind::tf32) implicit-GEMM convolutions.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/mpf.h"

namespace mpf {

constexpr int kMaxSplits = 296;  // split-K partial slots of the weight-gradient GEMMs (2 x 148 SMs)

// Forward conv and dgrad (a forward correlation of the delta with the rotated pack).
// x: [n_frag][gr][gc][cin] (NHWC, all grid positions readable; dgrad: delta with zero padding)
// out: [n_frag][gr][gc][cout] (same grid); valid region out_vr x out_vc
// out(y, x) = act(bias + sum_{ky,kx,ci} w[co][ky][kx][ci] * x(y + shift + ky, x + shift + kx))
// with x(.) = 0 outside the fragment.
struct TcConvArgs {
  const float* x;
  int n_frag, gr, gc, cin;
  const float* w;     // [cout][k][k][cin], tf32-rounded
  const float* bias;  // nullable
  int k, cout;
  float* out;
  int out_vr, out_vc;
  int act;
  int shift;          // 0 (forward) or -(k-1) (dgrad)
  int round_out;      // round the stored result to tf32 (operand of the next MMA)
  int zero_pad;       // (SIMT path) write zeros outside the valid region; the TC path always does
  const float* mul_dact;  // nullable: multiply by act'(mul_dact[same position])
  int dact;
  uint32_t flags;     // MPF_FLAG_* kernel selection (mpf.h)
  // forward of the last hidden layer: also write the softmax FC's logits (bias excluded)
  // z[p][c] = sum_co head_w[c][co] * out[p][co] of the stored output (nullable)
  const float* head_w;  // [head_C][cout]
  float* head_z;        // [n_frag * gr * gc][head_C]
  int head_C;
};

// Weight gradient: part[s][co][(ky*k+kx)*cin+ci] = sum_{p in split s} dy[p][co] * x[p+(ky,kx)][ci]
struct TcWgradArgs {
  const float* x;
  const float* dy;    // [n_frag][gr][gc][cout], zero outside the valid region
  int n_frag, gr, gc, vr_out, vc_out;
  int cin, cout, k;
  float* part;
  size_t part_cap_floats;
  uint32_t flags;     // MPF_FLAG_* kernel selection (mpf.h)
};

bool tc_supported(int cin, int cout, int k);
bool tc_wgrad_supported(int cin, int cout, int k);
cudaError_t launch_conv_tc(const TcConvArgs& a, cudaStream_t s, int* grid_out = nullptr);
cudaError_t launch_wgrad_tc(const TcWgradArgs& a, int* splits, cudaStream_t s);
// fp32 tensor map: dims[0] innermost, strides[i] = bytes between steps of dim i+1; zero fill
// out of bounds on loads, clipped stores
cudaError_t make_tmap_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                          const uint32_t* box, bool sw128);

}  // namespace mpf
