// kernels.cu — bandwidth-bound kernels of the MPF training path and the CUDA-core
// (SIMT) convolutions used for narrow layers and as the fp32 reference mode.
//
// Paper references: C layer §2 (54-55); MPF forward Alg. 3 (157-172);
// MPF backward Alg. 4 (174-186) with accumulation of shared maxima (Fig. 2, 143-145);
// gradient accumulation over fragments Alg. 2 (131-140); MCCE per pixel (197);
// class-weighted MCCE (252); SGD (210).  Readings R1-R19: DESIGN.md.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "mpf_internal.h"
#include "numerics.cuh"

namespace mpf {

static inline long long mpf_min_ll(long long a, long long b) { return a < b ? a : b; }


__device__ __forceinline__ float act_fwd(int act, float v) {
  if (act == MPF_TANH) return tanhf(v);
  if (act == MPF_LOGISTIC) return 1.f / (1.f + expf(-v));
  return v;
}

// derivative of the activation from its output
__device__ __forceinline__ float act_der(int act, float y) {
  if (act == MPF_TANH) return 1.f - y * y;
  if (act == MPF_LOGISTIC) return y * (1.f - y);
  return 1.f;
}

// ============================================================================ conv (SIMT)
// out[f][y][x][co] = act(bias[co] + sum_{ky,kx,ci} w[co][ky][kx][ci] * in[f][y+oy+ky][x+ox+kx][ci])
// Used for: forward of narrow layers (C_in = 1 first layers), dgrad (with the rotated
// pack and oy = ox = -(k-1)), and everything in MPF_PREC_FP32 mode.
constexpr int kTW = 16, kTH = 16, kCOT = 8, kCIC = 8;

template <int IMG>
__global__ void __launch_bounds__(256) conv_simt_kernel(ConvArgs a, int tiles_x) {
  extern __shared__ float sm[];
  const int k = a.k;
  const int IW = kTW + k - 1, IH = kTH + k - 1;
  float* s_in = sm;                      // [CIC][IH][IW]
  float* s_w = sm + kCIC * IH * IW;      // [COT][k*k][CIC]
  const int bx = blockIdx.x % tiles_x, cg = blockIdx.x / tiles_x;
  const int co0 = cg * kCOT;
  const int y0 = blockIdx.y * kTH, x0 = bx * kTW;
  const long long f = blockIdx.z;
  const int tx = threadIdx.x % kTW, ty = threadIdx.x / kTW;
  float acc[kCOT];
#pragma unroll
  for (int o = 0; o < kCOT; ++o) acc[o] = 0.f;
  const int cin = a.cin, cout = a.cout, kk = k * k;
  for (int ci0 = 0; ci0 < cin; ci0 += kCIC) {
    for (int e = threadIdx.x; e < IH * IW * kCIC; e += blockDim.x) {
      const int c = e % kCIC, t = e / kCIC, ix = t % IW, iy = t / IW;
      const int gy = y0 + a.off_y + iy, gx = x0 + a.off_x + ix, ci = ci0 + c;
      float v = 0.f;
      if (ci < cin && gy >= 0 && gy < a.in_vr && gx >= 0 && gx < a.in_vc) {
        if (IMG)
          v = a.in[((f * cin + ci) * a.in_gr + gy) * a.in_gc + gx];
        else
          v = a.in[((f * a.in_gr + gy) * a.in_gc + gx) * cin + ci];
      }
      s_in[(c * IH + iy) * IW + ix] = v;
    }
    for (int e = threadIdx.x; e < kCOT * kk * kCIC; e += blockDim.x) {
      const int c = e % kCIC, t = e / kCIC, q = t % kk, o = t / kk;
      const int co = co0 + o, ci = ci0 + c;
      s_w[e] = (co < cout && ci < cin) ? a.w[((long long)co * kk + q) * cin + ci] : 0.f;
    }
    __syncthreads();
    for (int ky = 0; ky < k; ++ky)
      for (int kx = 0; kx < k; ++kx) {
        const int q = ky * k + kx;
#pragma unroll
        for (int c = 0; c < kCIC; ++c) {
          const float v = s_in[(c * IH + ty + ky) * IW + tx + kx];
#pragma unroll
          for (int o = 0; o < kCOT; ++o) acc[o] += v * s_w[(o * kk + q) * kCIC + c];
        }
      }
    __syncthreads();
  }
  const int y = y0 + ty, x = x0 + tx;
  if (y >= a.out_gr || x >= a.out_gc) return;
  const bool valid = y < a.out_vr && x < a.out_vc;
  if (!valid && !a.zero_pad) return;
  const long long base = ((f * a.out_gr + y) * a.out_gc + x) * cout;
#pragma unroll
  for (int o = 0; o < kCOT; ++o) {
    const int co = co0 + o;
    if (co >= cout) break;
    float v = 0.f;
    if (valid) {
      v = acc[o] + (a.bias ? a.bias[co] : 0.f);
      v = act_fwd(a.act, v);
      if (a.mul_dact) v *= act_der(a.dact, a.mul_dact[base + co]);
      if (a.round_tf32) v = tf32_rn(v);
    }
    a.out[base + co] = v;
  }
}

cudaError_t launch_conv_simt(const ConvArgs& a, cudaStream_t s) {
  const int tiles_x = (a.out_gc + kTW - 1) / kTW;
  const int groups = (a.cout + kCOT - 1) / kCOT;
  dim3 grid(tiles_x * groups, (a.out_gr + kTH - 1) / kTH, a.n_frag_total);
  const int IW = kTW + a.k - 1, IH = kTH + a.k - 1;
  const size_t smem = sizeof(float) * (kCIC * IH * IW + kCOT * a.k * a.k * kCIC);
  if (a.image_mode) {
    cudaFuncSetAttribute(conv_simt_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    conv_simt_kernel<1><<<grid, 256, smem, s>>>(a, tiles_x);
  } else {
    cudaFuncSetAttribute(conv_simt_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    conv_simt_kernel<0><<<grid, 256, smem, s>>>(a, tiles_x);
  }
  return cudaGetLastError();
}

// ============================================================================ wgrad (SIMT)
// part_w[s][co][(ky*k+kx)*cin+ci] = sum_{p in chunk s} dy[p][co] * x[p + (ky,kx)][ci]
// part_b[s][co] = sum_{p in chunk s} dy[p][co]
// Alg. 2: the sum over all fragments and positions is the K-reduction of this GEMM.
constexpr int kWP = 32;  // positions per smem stage

template <int IMG>
__global__ void __launch_bounds__(256) wgrad_simt_kernel(WgradArgs a, long long chunk, int co_tiles,
                                                          long long P_total) {
  __shared__ float s_d[kWP][17];
  __shared__ float s_x[kWP][17];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int cot = blockIdx.x % co_tiles, kt = blockIdx.x / co_tiles;
  const int co = cot * 16 + ty;
  const int K = a.k * a.k * a.cin;
  const int kidx = kt * 16 + tx;
  int ky = 0, kx = 0, ci = 0;
  if (kidx < K) {
    ci = kidx % a.cin;
    const int q = kidx / a.cin;
    ky = q / a.k;
    kx = q % a.k;
  }
  const long long p0 = (long long)blockIdx.y * chunk;
  const long long p1 = (P_total < p0 + chunk) ? P_total : p0 + chunk;
  const long long per_frag = (long long)a.y_vr * a.y_vc;
  float acc = 0.f, accb = 0.f;
  for (long long pb = p0; pb < p1; pb += kWP) {
    // stage deltas [kWP][16 co] and shifted inputs [kWP][16 K]
    for (int e = threadIdx.x; e < kWP * 16; e += 256) {
      const int j = e / 16, c = e % 16;
      const long long p = pb + j;
      float dv = 0.f, xv = 0.f;
      if (p < p1) {
        const long long f = p / per_frag;
        const int r = (int)(p % per_frag);
        const int y = r / a.y_vc, x = r % a.y_vc;
        const int cc = cot * 16 + c;
        if (cc < a.cout) dv = a.dy[((f * a.y_gr + y) * a.y_gc + x) * a.cout + cc];
        const int kq = kt * 16 + c;
        if (kq < K) {
          const int ci2 = kq % a.cin, q2 = kq / a.cin;
          const int yy = y + q2 / a.k, xx = x + q2 % a.k;
          if (yy < a.x_vr && xx < a.x_vc) {
            if (IMG)
              xv = a.x[((f * a.cin + ci2) * a.x_gr + yy) * a.x_gc + xx];
            else
              xv = a.x[((f * a.x_gr + yy) * a.x_gc + xx) * a.cin + ci2];
          }
        }
      }
      s_d[j][c] = dv;
      s_x[j][c] = xv;
    }
    __syncthreads();
#pragma unroll 8
    for (int j = 0; j < kWP; ++j) {
      const float d = s_d[j][ty];
      acc += d * s_x[j][tx];
      accb += d;
    }
    __syncthreads();
  }
  (void)ky; (void)kx; (void)ci;
  if (co < a.cout && kidx < K) a.part_w[((long long)blockIdx.y * a.cout + co) * K + kidx] = acc;
  if (kt == 0 && tx == 0 && co < a.cout) a.part_b[(long long)blockIdx.y * a.cout + co] = accb;
}

int wgrad_simt_splits(long long positions) {
  long long s = (positions + 4095) / 4096;
  if (s < 1) s = 1;
  if (s > 256) s = 256;
  return (int)s;
}

cudaError_t launch_wgrad_simt(const WgradArgs& a, cudaStream_t s) {
  const long long P_total = (long long)a.n_frag_total * a.y_vr * a.y_vc;
  const int K = a.k * a.k * a.cin;
  const int co_tiles = (a.cout + 15) / 16, k_tiles = (K + 15) / 16;
  const long long chunk = (P_total + a.n_split - 1) / a.n_split;
  dim3 grid(co_tiles * k_tiles, a.n_split);
  if (a.image_mode)
    wgrad_simt_kernel<1><<<grid, 256, 0, s>>>(a, chunk, co_tiles, P_total);
  else
    wgrad_simt_kernel<0><<<grid, 256, 0, s>>>(a, chunk, co_tiles, P_total);
  return cudaGetLastError();
}

// gw (+)= sum_i pw[i] over n_split partials [n_split][cout][K] (K = (ky, kx, ci)), fixed order.
// A block owns 32 V consecutive partial elements (V = 4: float4 lanes when the partial rows
// are 16-byte aligned); warp w sums splits w, w + 8, ... (four interleaved accumulators, one
// coalesced 32 V-float read per split), and the 8 warp sums meet in shared memory in order.
template <int V>
__global__ void __launch_bounds__(256) wgrad_reduce_kernel(const float* __restrict__ pw, int n_split, int cout,
                                                           int cin, int k, float* gw) {
  __shared__ float red[8][32 * V + 1];
  const int K = k * k * cin;
  const long long total = (long long)cout * K;
  const int c = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long e0 = (blockIdx.x * 32LL + c) * V;
  float t[4][V];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < V; ++v) t[u][v] = 0.f;
  if (e0 < total) {
    auto ld = [&](int i, float (&acc)[V]) {
      const float* src = pw + (long long)i * total + e0;
      if constexpr (V == 4) {
        const float4 q = __ldcg(reinterpret_cast<const float4*>(src));
        acc[0] += q.x; acc[1] += q.y; acc[2] += q.z; acc[3] += q.w;
      } else {
        acc[0] += __ldcg(src);
      }
    };
    int i = w;
    for (; i + 24 < n_split; i += 32) {
      ld(i, t[0]); ld(i + 8, t[1]); ld(i + 16, t[2]); ld(i + 24, t[3]);
    }
    for (; i < n_split; i += 8) ld(i, t[0]);
  }
#pragma unroll
  for (int v = 0; v < V; ++v) red[w][c * V + v] = (t[0][v] + t[1][v]) + (t[2][v] + t[3][v]);
  __syncthreads();
  for (int j = threadIdx.x; j < 32 * V; j += 256) {
    const long long e = blockIdx.x * 32LL * V + j;
    if (e >= total) continue;
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += red[q][j];
    const int co = (int)(e / K), kidx = (int)(e % K);
    const int ci = kidx % cin, q = kidx / cin;
    const int ky = q / k, kx = q % k;
    gw[(((long long)co * cin + ci) * k + ky) * k + kx] += s;
  }
}

cudaError_t launch_wgrad_reduce(const float* pw, int n_split, int cout, int cin, int k, float* gw,
                                cudaStream_t s) {
  const long long total = (long long)cout * k * k * cin;
  if (total <= 0) return cudaSuccess;
  if (total % 4 == 0 && ((uintptr_t)pw & 15) == 0)
    wgrad_reduce_kernel<4><<<(unsigned)((total + 127) / 128), 256, 0, s>>>(pw, n_split, cout, cin, k, gw);
  else
    wgrad_reduce_kernel<1><<<(unsigned)((total + 31) / 32), 256, 0, s>>>(pw, n_split, cout, cin, k, gw);
  return cudaGetLastError();
}

// ============================================================================ Armijo helpers
// ||g||^2 in double, deterministic: block b sums its contiguous chunk (fixed tree order)
// into part[b], then one block sums part[0..nb) in order.
__global__ void sqnorm_part_kernel(const float* __restrict__ g, long long n, long long chunk, double* part) {
  __shared__ double s[256];
  const long long b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  double t = 0.0;
  for (long long e = b0 + threadIdx.x; e < b1; e += blockDim.x) t += (double)g[e] * (double)g[e];
  s[threadIdx.x] = t;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}
__global__ void sqnorm_final_kernel(const double* __restrict__ part, int nb, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < nb; ++b) t += part[b];
    *out = t;
  }
}
cudaError_t launch_sqnorm(const float* g, long long n, double* part, int nb, double* out, cudaStream_t s) {
  const long long chunk = (n + nb - 1) / nb;
  sqnorm_part_kernel<<<nb, 256, 0, s>>>(g, n, chunk, part);
  sqnorm_final_kernel<<<1, 32, 0, s>>>(part, nb, out);
  return cudaGetLastError();
}
// theta = theta0 - alpha * scale * g   (the Armijo trial point along d = -g)
__global__ void armijo_axpy_kernel(float* __restrict__ theta, const float* __restrict__ theta0,
                                   const float* __restrict__ g, long long n, float step) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    theta[e] = theta0[e] - step * g[e];
}
cudaError_t launch_armijo_axpy(float* theta, const float* theta0, const float* g, long long n, float step,
                               cudaStream_t s) {
  const long long blocks = mpf_min_ll((n + 255) / 256, 148 * 8);
  armijo_axpy_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(theta, theta0, g, n, step);
  return cudaGetLastError();
}

// ============================================================================ L-BFGS vectors
// The two-loop recursion (reading R21) on the flat
// parameter vector.  Every pass is one sweep: v <- f(v, x) with a coefficient formed from
// the previous pass's dot product, then this block's partial of the next dot z . v over the
// SAME contiguous chunk it just updated, so no pass needs a grid-wide barrier.  Each block
// re-sums the nb partials of the previous pass itself in one fixed order (identical in
// every block), so the scalars are deterministic and never leave the device.
namespace {
__device__ __forceinline__ double lb_block_sum(double t, double* sh) {
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = t;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r += sh[i];
  return r;  // valid in thread 0
}
// sum of nb partials, same order in every block; broadcast to all threads
__device__ __forceinline__ double lb_sum_parts(const double* __restrict__ part, int nb, double* sh) {
  if (threadIdx.x < 32) {
    double t = 0.0;
    for (int i = threadIdx.x; i < nb; i += 32) t += part[i];
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) sh[32] = t;
  }
  __syncthreads();
  const double r = sh[32];
  __syncthreads();
  return r;
}
}  // namespace

// gprev = scale * g
__global__ void lbfgs_gset_kernel(float* __restrict__ gprev, const float* __restrict__ g, long long n, float scale) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    gprev[e] = scale * g[e];
}
// the new curvature pair: s = theta - theta0, y = scale g - gprev; gprev <- scale g;
// partials of s.y and y.y
__global__ void lbfgs_pair_kernel(float* __restrict__ S, float* __restrict__ Y, float* __restrict__ gprev,
                                  const float* __restrict__ theta, const float* __restrict__ theta0,
                                  const float* __restrict__ g, long long n, long long chunk, float scale,
                                  double* __restrict__ part) {
  __shared__ double sh[40];
  const long long b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  double sy = 0.0, yy = 0.0;
  for (long long e = b0 + threadIdx.x; e < b1; e += blockDim.x) {
    const float s = theta[e] - theta0[e];
    const float gn = scale * g[e];
    const float y = gn - gprev[e];
    S[e] = s;
    Y[e] = y;
    gprev[e] = gn;
    sy += (double)s * (double)y;
    yy += (double)y * (double)y;
  }
  sy = lb_block_sum(sy, sh);
  __syncthreads();
  yy = lb_block_sum(yy, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = sy;
    part[gridDim.x + blockIdx.x] = yy;
  }
}
// mode 0: v = x.  mode 1 (first loop): a = rho (sum part_in); *a_slot = a; v = (v - a x) * post.
// mode 2 (second loop): b = rho (sum part_in); v = v + (*a_slot - b) x.  Then partials of z.v.
__global__ void lbfgs_pass_kernel(double* __restrict__ v, const float* __restrict__ x, const float* __restrict__ z,
                                  long long n, long long chunk, const double* __restrict__ part_in, int mode,
                                  double rho, double* a_slot, double post, double* __restrict__ part_out) {
  __shared__ double sh[40];
  double coef = 0.0;
  if (mode != 0) {
    const double d = lb_sum_parts(part_in, gridDim.x, sh);
    if (mode == 1) {
      coef = -rho * d;
      if (blockIdx.x == 0 && threadIdx.x == 0) *a_slot = rho * d;
    } else {
      coef = *a_slot - rho * d;
    }
  }
  const long long b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  double t = 0.0;
  for (long long e = b0 + threadIdx.x; e < b1; e += blockDim.x) {
    double ve;
    if (mode == 0) ve = (double)x[e];
    else if (mode == 1) ve = (v[e] + coef * (double)x[e]) * post;
    else ve = v[e] + coef * (double)x[e];
    v[e] = ve;
    if (z) t += (double)z[e] * ve;
  }
  t = lb_block_sum(t, sh);
  if (threadIdx.x == 0) part_out[blockIdx.x] = t;
}
// theta = theta0 - alpha v   (the trial point theta0 + alpha d, d = -H g = -v)
__global__ void lbfgs_trial_kernel(float* __restrict__ theta, const float* __restrict__ theta0,
                                   const double* __restrict__ v, long long n, double alpha) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    theta[e] = (float)((double)theta0[e] - alpha * v[e]);
}

cudaError_t launch_lbfgs_gset(float* gprev, const float* g, long long n, float scale, cudaStream_t s) {
  const long long blocks = mpf_min_ll((n + 255) / 256, 148 * 8);
  lbfgs_gset_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(gprev, g, n, scale);
  return cudaGetLastError();
}
cudaError_t launch_lbfgs_pair(float* S, float* Y, float* gprev, const float* theta, const float* theta0, const float* g,
                              long long n, float scale, double* part, int nb, cudaStream_t s) {
  const long long chunk = (n + nb - 1) / nb;
  lbfgs_pair_kernel<<<nb, 256, 0, s>>>(S, Y, gprev, theta, theta0, g, n, chunk, scale, part);
  return cudaGetLastError();
}
cudaError_t launch_lbfgs_pass(double* v, const float* x, const float* z, long long n, const double* part_in, int mode,
                              double rho, double* a_slot, double post, double* part_out, int nb, cudaStream_t s) {
  const long long chunk = (n + nb - 1) / nb;
  lbfgs_pass_kernel<<<nb, 256, 0, s>>>(v, x, z, n, chunk, part_in, mode, rho, a_slot, post, part_out);
  return cudaGetLastError();
}
cudaError_t launch_lbfgs_trial(float* theta, const float* theta0, const double* v, long long n, double alpha,
                               cudaStream_t s) {
  const long long blocks = mpf_min_ll((n + 255) / 256, 148 * 8);
  lbfgs_trial_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(theta, theta0, v, n, alpha);
  return cudaGetLastError();
}

// ============================================================================ mirror padding
// Same-size output ("pixels outside of the boundary of testing images are
// synthesized by mirroring -- which allows to preserve the size of the output"): the
// padded image's pixel (yp, xp) is the original pixel reflected about the border pixel
// (no repeat of the edge; reading R20): y = yp - pad_top, y < 0 -> -y, y >= H -> 2(H-1) - y.
// One thread per output float; rows are coalesced (reflection only at the two ends).
__global__ void mirror_pad_kernel(const float* __restrict__ in, float* __restrict__ out, long long planes, int H, int W,
                                  int pt, int pl, int Hp, int Wp) {
  const long long total = planes * Hp * Wp;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int xp = (int)(e % Wp);
    const long long t = e / Wp;
    const int yp = (int)(t % Hp);
    const long long pl_i = t / Hp;
    int y = yp - pt, x = xp - pl;
    y = y < 0 ? -y : (y >= H ? 2 * (H - 1) - y : y);
    x = x < 0 ? -x : (x >= W ? 2 * (W - 1) - x : x);
    out[e] = in[(pl_i * H + y) * W + x];
  }
}

cudaError_t launch_mirror_pad(const float* in, float* out, long long planes, int H, int W, int pt, int pl, int Hp, int Wp,
                              cudaStream_t s) {
  const long long total = planes * Hp * Wp;
  const long long blocks = mpf_min_ll((total + 255) / 256, 148 * 16);
  mirror_pad_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(in, out, planes, H, W, pt, pl, Hp, Wp);
  return cudaGetLastError();
}

// ============================================================================ small kernels
// labelled pixels per image: integer partial counts combined with integer atomics
// (exact, order-independent)
__global__ void label_count_kernel(const uint8_t* __restrict__ labels, int hw, int classes, int* nlab) {
  __shared__ int s_red[32];
  const int img = blockIdx.y;
  int c = 0;
  const uint8_t* L = labels + (long long)img * hw;
  const int stride = gridDim.x * blockDim.x;
  int head = 0;  // bytes before the first 16-byte aligned address
  if (((uintptr_t)L & 15) != 0) head = min(hw, (int)(16 - ((uintptr_t)L & 15)));
  const int nv = (hw - head) >> 4;
  const uint4* V = reinterpret_cast<const uint4*>(L + head);
  for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
    const uint4 q = __ldg(V + v);
    const uint32_t wd[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int b = 0; b < 4; ++b) c += (int)((wd[j] >> (8 * b)) & 255u) < classes;
  }
  const int tail0 = head + (nv << 4);
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < head) c += L[g] < classes;
  if (g < hw - tail0) c += L[tail0 + g] < classes;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += s_red[w];
    if (t) atomicAdd(nlab + img, t);
  }
}

// per-class pixel counts over n label maps (255 and labels >= classes are not counted);
// block histograms in shared memory, integer atomics (exact, order-independent)
__global__ void class_hist_kernel(const uint8_t* __restrict__ labels, long long total, int classes,
                                  unsigned long long* counts) {
  __shared__ unsigned int s_h[256];
  for (int c = threadIdx.x; c < 256; c += blockDim.x) s_h[c] = 0u;
  __syncthreads();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int l = labels[e];
    if (l < classes) atomicAdd(&s_h[l], 1u);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < classes; c += blockDim.x)
    if (s_h[c]) atomicAdd(counts + c, (unsigned long long)s_h[c]);
}

cudaError_t launch_class_hist(const uint8_t* labels, long long total, int classes, unsigned long long* counts,
                              cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(unsigned long long) * classes, s);
  if (e != cudaSuccess) return e;
  const long long blocks = mpf_min_ll((total + 255) / 256, 148 * 8);
  class_hist_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(labels, total, classes, counts);
  return cudaGetLastError();
}

cudaError_t launch_label_count(const uint8_t* labels, int n, int hw, int classes, int* nlab, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(nlab, 0, sizeof(int) * n, s);
  if (e != cudaSuccess) return e;
  if (hw <= 0) return cudaSuccess;
  // 16 labels per thread per pass; about 4 resident blocks per SM over the whole batch
  int bx = (int)mpf_min_ll(((long long)hw + 256 * 16 * 2 - 1) / (256 * 16 * 2), (148 * 4 + n - 1) / n);
  if (bx < 1) bx = 1;
  label_count_kernel<<<dim3(bx, n), 256, 0, s>>>(labels, hw, classes, nlab);
  return cudaGetLastError();
}

// per-image loss = (sum of the per-tile partials, fixed order) / n_lab.  Grid (chunks, n):
// block (ch, img) sums parts [ch*len, (ch+1)*len) of its image (fixed tree), writes
// tmp[img][ch]; the last block of an image (cnt[img], reset afterwards) sums the chunks in order.
__global__ void __launch_bounds__(256) loss_finalize_kernel(const float* __restrict__ part, int parts, int len,
                                                            const int* __restrict__ nlab, float* loss, float* tmp,
                                                            unsigned* cnt) {
  __shared__ float s[256];
  __shared__ bool last;
  const int img = blockIdx.y, ch = blockIdx.x, nch = gridDim.x;
  const int p0 = ch * len, p1 = min(parts, p0 + len);
  float t = 0.f;
  for (int i = p0 + threadIdx.x; i < p1; i += 256) t += part[(long long)img * parts + i];
  s[threadIdx.x] = t;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (nch == 1) {
    if (threadIdx.x == 0) loss[img] = nlab[img] > 0 ? s[0] / (float)nlab[img] : 0.f;
    return;
  }
  if (threadIdx.x == 0) {
    tmp[(long long)img * nch + ch] = s[0];
    __threadfence();
    last = atomicAdd(cnt + img, 1u) == (unsigned)nch - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  float u = 0.f;
  for (int q = 0; q < nch; ++q) u += __ldcg(tmp + (long long)img * nch + q);
  loss[img] = nlab[img] > 0 ? u / (float)nlab[img] : 0.f;
  cnt[img] = 0u;  // ready for the next launch
}

cudaError_t launch_loss_finalize(const float* part, int parts, const int* nlab, int n, float* loss, float* tmp,
                                 unsigned* cnt, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int nch = (parts + 2047) / 2048;
  if (nch > kLossChunks) nch = kLossChunks;
  if (nch < 1) nch = 1;
  const int len = (parts + nch - 1) / nch;
  loss_finalize_kernel<<<dim3(nch, n), 256, 0, s>>>(part, parts, len, nlab, loss, tmp, cnt);
  return cudaGetLastError();
}

__global__ void sgd_kernel(float* __restrict__ p, float* __restrict__ g, long long n, float step) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    p[e] -= step * g[e];
    g[e] = 0.f;
  }
}

cudaError_t launch_sgd(float* params, float* grads, long long n, float lr, float scale, cudaStream_t s) {
  const int blocks = (int)mpf_min_ll((n + 255) / 256, 1024);
  sgd_kernel<<<blocks, 256, 0, s>>>(params, grads, n, lr * scale);
  return cudaGetLastError();
}

// canonical W[co][ci][ky][kx] -> fwd pack [co][ky][kx][ci], dgrad pack [ci][k-1-ky][k-1-kx][co]
__global__ void pack_kernel(const float* __restrict__ w, int cout, int cin, int k, float* wp, float* dp,
                            int round_fwd, int round_dgrad) {
  const long long n = (long long)cout * cin * k * k;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int kx = (int)(e % k);
    long long t = e / k;
    const int ky = (int)(t % k);
    t /= k;
    const int ci = (int)(t % cin);
    const int co = (int)(t / cin);
    const float v = w[e];
    wp[(((long long)co * k + ky) * k + kx) * cin + ci] = round_fwd ? tf32_rn(v) : v;
    if (dp) dp[(((long long)ci * k + (k - 1 - ky)) * k + (k - 1 - kx)) * cout + co] = round_dgrad ? tf32_rn(v) : v;
  }
}

cudaError_t launch_pack_weights(const float* w, int cout, int cin, int k, float* wp, float* dp, int round_fwd,
                                int round_dgrad, cudaStream_t s) {
  const long long n = (long long)cout * cin * k * k;
  const int blocks = (int)mpf_min_ll((n + 255) / 256, 1024);
  pack_kernel<<<blocks, 256, 0, s>>>(w, cout, cin, k, wp, dp, round_fwd, round_dgrad);
  return cudaGetLastError();
}

// Defragmentation: pix[n][c][y][x] = frag[n*F + f(y,x)][i(y)][j(x)][c]
struct Frag2PixArgs {
  const float* frag;
  float* pix;
  int n, C, F, fr, fc, O_H, O_W, L;
  int k[kMaxL];
};

__global__ void frag2pix_kernel(Frag2PixArgs a, long long total) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(e % a.O_W);
    long long t = e / a.O_W;
    const int y = (int)(t % a.O_H);
    t /= a.O_H;
    const int c = (int)(t % a.C);
    const long long img = t / a.C;
    int yy = y, xx = x, g = 0;
    for (int l = 0; l < a.L; ++l) {  // level 1 is the most significant digit (R2)
      const int kq = a.k[l];
      const int r = yy % kq, cc = xx % kq;
      yy /= kq;
      xx /= kq;
      g = g * kq * kq + r * kq + cc;
    }
    a.pix[e] = a.frag[(((img * a.F + g) * a.fr + yy) * a.fc + xx) * a.C + c];
  }
}

cudaError_t launch_frag2pix(const float* frag, float* pix, int n, int C, int F, int fr, int fc, int O_H, int O_W,
                            int n_levels, const int* pool_k, cudaStream_t s) {
  Frag2PixArgs a;
  a.frag = frag; a.pix = pix; a.n = n; a.C = C; a.F = F; a.fr = fr; a.fc = fc; a.O_H = O_H; a.O_W = O_W;
  a.L = n_levels;
  for (int l = 0; l < n_levels; ++l) a.k[l] = pool_k[l];
  const long long total = (long long)n * C * O_H * O_W;
  if (total == 0) return cudaSuccess;
  const int blocks = (int)mpf_min_ll((total + 255) / 256, 148LL * 32);
  frag2pix_kernel<<<blocks, 256, 0, s>>>(a, total);
  return cudaGetLastError();
}

__global__ void compact_kernel(const float* __restrict__ src, int gr, int gc, int vr, int vc, int C,
                               long long total, float* dst) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(e % C);
    long long t = e / C;
    const int x = (int)(t % vc);
    t /= vc;
    const int y = (int)(t % vr);
    const long long f = t / vr;
    dst[e] = src[((f * gr + y) * gc + x) * C + c];
  }
}

cudaError_t launch_compact_copy(const float* src, int gr, int gc, int vr, int vc, int C, long long nf,
                                float* dst, cudaStream_t s) {
  const long long total = nf * vr * vc * C;
  if (total == 0) return cudaSuccess;
  const int blocks = (int)mpf_min_ll((total + 255) / 256, 148LL * 32);
  compact_kernel<<<blocks, 256, 0, s>>>(src, gr, gc, vr, vc, C, total, dst);
  return cudaGetLastError();
}

}  // namespace mpf
