// conv_first.cu — the first convolution layer (one input map: the raw image), forward
// and weight gradient, on CUDA cores in fp32.
//
// Alg. 1 for the first layer: the input storage holds a single
// fragment, the zero-padded image (reading R7 padding), so the first layer
// is one valid k x k cross-correlation (R10) per image, + bias + tanh.
// With C_in = 1 the GEMM K dimension is only k^2 (9..49), far too thin for the tensor
// cores to pay; the layer is bound by its fp32 output stream (forward) and its delta
// stream (wgrad), so both kernels stage the image tile in shared memory and use
// register-blocked outer products (4 positions x 8 maps forward; 8 maps x 4 taps
// wgrad) to stay near the FFMA/HBM ceilings.
//
// Weight gradient (Alg. 2): dW[co][ky][kx] = sum over every position
// p of the image of dY[p][co] * img[p + (ky, kx)], with dY zero outside the valid
// region.  Persistent CTAs accumulate in registers over their tiles and write one
// partial per CTA; a fixed-order reduction finishes the sum (deterministic).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "mpf_internal.h"
#include "numerics.cuh"

namespace mpf {

namespace {


// SFU activations, as in the tensor-core epilogues: tanh(v) = 1 - 2 / (2^(2 v log2 e) + 1)
// (absolute error ~1e-7; tanhf's ~25 instructions were a third of this kernel's issue)
__device__ __forceinline__ float act_fwd(int act, float v) {
  if (act == MPF_TANH) return fast_tanh(v);
  if (act == MPF_LOGISTIC) return fast_logistic(v);
  return v;
}

constexpr int kFTH = 16, kFTW = 16;  // forward tile (positions)
constexpr int kFPX = 4;              // positions per thread (horizontal strip)
constexpr int kFCO = 8;              // maps per thread

// blockDim.x = 64 strips x n_cog channel groups
template <int K>
__global__ void __launch_bounds__(256) conv_first_fwd_kernel(FirstConvArgs a) {
  extern __shared__ float sm[];
  constexpr int IW = kFTW + K - 1, IH = kFTH + K - 1;
  const int coutp = a.n_cog * kFCO;
  constexpr int IMG = (IH * IW + 3) / 4 * 4;  // keep the float4 tiles 16-B aligned
  float* s_img = sm;                 // [IH][IW]
  float* s_w = sm + IMG;             // [K*K][coutp]
  float* s_b = s_w + K * K * coutp;  // [coutp]
  const int img = blockIdx.z;
  const int y0 = blockIdx.y * kFTH, x0 = blockIdx.x * kFTW;
  for (int e = threadIdx.x; e < IH * IW; e += blockDim.x) {
    const int iy = e / IW, ix = e % IW;
    const int gy = y0 + iy, gx = x0 + ix;
    float v = 0.f;
    if (gy < a.H && gx < a.W) v = a.img[((size_t)img * a.H + gy) * a.W + gx];
    s_img[e] = v;
  }
  if (blockDim.x % coutp == 0) {  // canonical W[co][0][ky][kx] -> s_w[tap][coutp]: a thread keeps
    // one co and steps taps by blockDim / coutp (no division per element; the launcher's
    // blockDim = 64 n_cog = 8 coutp always takes this path)
    const int co = threadIdx.x % coutp, tstep = blockDim.x / coutp;
    const bool real = co < a.cout;
    for (int t = threadIdx.x / coutp; t < K * K; t += tstep) s_w[t * coutp + co] = real ? a.w[co * K * K + t] : 0.f;
  } else {
    for (int e = threadIdx.x; e < K * K * coutp; e += blockDim.x) {
      const int t = e / coutp, co = e % coutp;
      s_w[e] = co < a.cout ? a.w[co * K * K + t] : 0.f;
    }
  }
  for (int e = threadIdx.x; e < coutp; e += blockDim.x) s_b[e] = e < a.cout ? a.bias[e] : 0.f;
  __syncthreads();
  const int cog = threadIdx.x % a.n_cog, strip = threadIdx.x / a.n_cog;
  const int ty = strip / (kFTW / kFPX), tx = (strip % (kFTW / kFPX)) * kFPX;
  float acc[kFPX][kFCO];
#pragma unroll
  for (int q = 0; q < kFPX; ++q)
#pragma unroll
    for (int o = 0; o < kFCO; ++o) acc[q][o] = 0.f;
#pragma unroll
  for (int ky = 0; ky < K; ++ky) {
    float row[kFPX + K - 1];
#pragma unroll
    for (int i = 0; i < kFPX + K - 1; ++i) row[i] = s_img[(ty + ky) * IW + tx + i];
#pragma unroll
    for (int kx = 0; kx < K; ++kx) {
      const float4* wp = reinterpret_cast<const float4*>(s_w + (ky * K + kx) * coutp + cog * kFCO);
      const float4 w0 = wp[0], w1 = wp[1];
      const float wv[kFCO] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int q = 0; q < kFPX; ++q)
#pragma unroll
        for (int o = 0; o < kFCO; ++o) acc[q][o] = fmaf(row[q + kx], wv[o], acc[q][o]);
    }
  }
  const int y = y0 + ty;
  if (y >= a.out_gr) return;
#pragma unroll
  for (int q = 0; q < kFPX; ++q) {
    const int x = x0 + tx + q;
    if (x >= a.out_gc) continue;
    const bool valid = y < a.out_vr && x < a.out_vc;
    if (!valid && !a.zero_pad) continue;
    float* dst = a.out + (((size_t)img * a.out_gr + y) * a.out_gc + x) * a.cout + cog * kFCO;
    float v[kFCO];
#pragma unroll
    for (int o = 0; o < kFCO; ++o) {
      float t = 0.f;
      if (valid) {
        t = act_fwd(a.act, acc[q][o] + s_b[cog * kFCO + o]);
        if (a.round_tf32) t = tf32_rn(t);
      }
      v[o] = t;
    }
    if (a.cout % kFCO == 0) {
      reinterpret_cast<float4*>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
#pragma unroll
      for (int o = 0; o < kFCO; ++o)
        if (cog * kFCO + o < a.cout) dst[o] = v[o];
    }
  }
}

// ------------------------------------------------------------------------------ wgrad
constexpr int kWTH = 8, kWTW = 32;  // wgrad tile: 256 positions
constexpr int kWCO = 8, kWT = 4;    // accumulators per thread: 8 maps x 4 taps

// WT taps per thread: 4, or a whole kernel row (WT = K, K >= 5; 2 CTAs per SM) so each
// staged delta vector feeds 8 K FMAs instead of 32.
template <int K, int WT>
__global__ void __launch_bounds__(256, WT > 4 ? 2 : 3) conv_first_wgrad_kernel(FirstWgradArgs a) {
  extern __shared__ float sm[];
  constexpr int kWT = WT;
  constexpr int IW = kWTW + K - 1, IH = kWTH + K - 1;
  constexpr int NT = (K * K + kWT - 1) / kWT;  // tap groups
  const int coutp = a.n_cog * kWCO;
  constexpr int IMG = (IH * IW + 3) / 4 * 4;
  // two buffers of [image tile | delta tile], filled with cp.async one tile ahead
  const int buf_floats = IMG + kWTH * kWTW * coutp;
  float* s_red = sm;             // end-of-kernel reduction (aliases buffer 0)
  const bool async = coutp == a.cout;  // delta rows are whole 16-B vectors (cout % 8 == 0)
  const int per_stream = a.n_cog * NT;
  const int n_streams = blockDim.x / per_stream;
  const int stream = threadIdx.x / per_stream, r = threadIdx.x % per_stream;
  const int cog = r % a.n_cog, tg = r / a.n_cog;
  const bool active = stream < n_streams;
  int toff[kWT];
#pragma unroll
  for (int u = 0; u < kWT; ++u) {
    const int t = tg * kWT + u;
    toff[u] = t < K * K ? (t / K) * IW + (t % K) : 0;
  }
  float acc[kWCO][kWT];
#pragma unroll
  for (int o = 0; o < kWCO; ++o)
#pragma unroll
    for (int u = 0; u < kWT; ++u) acc[o][u] = 0.f;
  const int tiles_x = (a.gc + kWTW - 1) / kWTW, tiles_y = (a.gr + kWTH - 1) / kWTH;
  const long long total = (long long)a.n * tiles_x * tiles_y;
  // stage tile `tile` into buffer `b`: image tile (zero outside H x W) and delta tile
  // [256 positions][cout] (zero outside the grid)
  auto stage = [&](long long tile, int b) {
    float* s_img = sm + b * buf_floats;
    float* s_dy = s_img + IMG;
    const int tx_ = (int)(tile % tiles_x);
    const long long t2 = tile / tiles_x;
    const int ty_ = (int)(t2 % tiles_y), img = (int)(t2 / tiles_y);
    const int y0 = ty_ * kWTH, x0 = tx_ * kWTW;
    for (int e = threadIdx.x; e < IH * IW; e += blockDim.x) {
      const int iy = e / IW, ix = e % IW;
      const int gy = y0 + iy, gx = x0 + ix;
      const bool in = gy < a.H && gx < a.W;
      const float* src = a.img + (in ? ((size_t)img * a.H + gy) * a.W + gx : 0);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(s_img + e)),
                   "l"(src), "r"(in ? 4 : 0)
                   : "memory");
    }
    if (async) {
      const int vec = coutp / 4;
      for (int e = threadIdx.x; e < kWTH * kWTW * vec; e += blockDim.x) {
        const int v4 = e % vec, p = e / vec;
        const int y = y0 + p / kWTW, x = x0 + p % kWTW;
        const bool in = y < a.gr && x < a.gc;
        const float* src = a.dy + (in ? (((size_t)img * a.gr + y) * a.gc + x) * a.cout + 4 * v4 : 0);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(s_dy + p * coutp + 4 * v4)),
                     "l"(src), "r"(in ? 16 : 0)
                     : "memory");
      }
    } else {
      for (int e = threadIdx.x; e < kWTH * kWTW * coutp; e += blockDim.x) {
        const int co = e % coutp, p = e / coutp;
        const int y = y0 + p / kWTW, x = x0 + p % kWTW;
        float v = 0.f;
        if (co < a.cout && y < a.gr && x < a.gc) v = a.dy[(((size_t)img * a.gr + y) * a.gc + x) * a.cout + co];
        s_dy[e] = v;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (blockIdx.x < total) stage(blockIdx.x, 0);
  int it = 0;
  for (long long tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
    const int tx_ = (int)(tile % tiles_x);
    (void)tx_;
    if (tile + gridDim.x < total) stage(tile + gridDim.x, (it + 1) & 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // this tile's group has landed
    __syncthreads();
    const float* s_img = sm + (it & 1) * buf_floats;
    const float* s_dy = s_img + IMG;
    if (active) {
      for (int p = stream; p < kWTH * kWTW; p += n_streams) {
        const int py = p / kWTW, px = p % kWTW;
        const float4* dp = reinterpret_cast<const float4*>(s_dy + p * coutp + cog * kWCO);
        const float4 d0 = dp[0], d1 = dp[1];
        const float dv[kWCO] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
        const float* ib = s_img + py * IW + px;
        float iv[kWT];
#pragma unroll
        for (int u = 0; u < kWT; ++u) iv[u] = ib[toff[u]];
#pragma unroll
        for (int o = 0; o < kWCO; ++o)
#pragma unroll
          for (int u = 0; u < kWT; ++u) acc[o][u] = fmaf(dv[o], iv[u], acc[o][u]);
      }
    }
    __syncthreads();  // this buffer is free for the stage issued next iteration
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  // fixed-order reduction over streams, then one partial per CTA: part[blk][co][tap]
  __syncthreads();
  const int KK = K * K;
  if (active) {
#pragma unroll
    for (int o = 0; o < kWCO; ++o)
#pragma unroll
      for (int u = 0; u < kWT; ++u) {
        const int co = cog * kWCO + o, t = tg * kWT + u;
        if (t < KK) s_red[(stream * coutp + co) * KK + t] = acc[o][u];
      }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < a.cout * KK; e += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < n_streams; ++q) s += s_red[q * coutp * KK + e];
    a.part[(size_t)blockIdx.x * a.cout * KK + e] = s;
  }
}

// Row-streamed variant (K >= 5, default): the tile is TH x 32 positions with TH = the number
// of thread streams, and stream s owns tile row s, so a thread walks 32 consecutive
// positions of one row: its kernel-row window img[y + ky][x .. x + K - 1] slides by one
// column per position (one shared load instead of K, no per-tap address math), while the
// delta vector of each position feeds 8 K FMAs.  Same sums in the same per-CTA order as the
// other variant within a thread, then the same fixed-order reductions.
template <int K>
__global__ void __launch_bounds__(256, 2) conv_first_wgrad_rows_kernel(FirstWgradArgs a, int TH) {
  extern __shared__ float sm[];
  constexpr int IW = kWTW + K - 1;
  const int IH = TH + K - 1;
  const int coutp = a.n_cog * kWCO;
  const int IMG = (IH * IW + 3) / 4 * 4;
  const int buf_floats = IMG + TH * kWTW * coutp;
  float* s_red = sm;
  const bool async = coutp == a.cout;
  const int per_stream = a.n_cog * K;
  const int stream = threadIdx.x / per_stream, r = threadIdx.x % per_stream;
  const int cog = r % a.n_cog, ky = r / a.n_cog;
  const bool active = stream < TH;
  float acc[kWCO][K];
#pragma unroll
  for (int o = 0; o < kWCO; ++o)
#pragma unroll
    for (int u = 0; u < K; ++u) acc[o][u] = 0.f;
  const int tiles_x = (a.gc + kWTW - 1) / kWTW, tiles_y = (a.gr + TH - 1) / TH;
  const long long total = (long long)a.n * tiles_x * tiles_y;
  auto stage = [&](long long tile, int b) {
    float* s_img = sm + b * buf_floats;
    float* s_dy = s_img + IMG;
    const int tx_ = (int)(tile % tiles_x);
    const long long t2 = tile / tiles_x;
    const int ty_ = (int)(t2 % tiles_y), img = (int)(t2 / tiles_y);
    const int y0 = ty_ * TH, x0 = tx_ * kWTW;
    for (int e = threadIdx.x; e < IH * IW; e += blockDim.x) {
      const int iy = e / IW, ix = e % IW;
      const int gy = y0 + iy, gx = x0 + ix;
      const bool in = gy < a.H && gx < a.W;
      const float* src = a.img + (in ? ((size_t)img * a.H + gy) * a.W + gx : 0);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(s_img + e)),
                   "l"(src), "r"(in ? 4 : 0)
                   : "memory");
    }
    if (async && blockDim.x % (coutp / 4) == 0) {  // a thread keeps one 16-B column: no division per copy
      const int vec = coutp / 4, v4 = threadIdx.x % vec, pstep = blockDim.x / vec;
      for (int p = threadIdx.x / vec; p < TH * kWTW; p += pstep) {
        const int y = y0 + p / kWTW, x = x0 + p % kWTW;
        const bool in = y < a.gr && x < a.gc;
        const float* src = a.dy + (in ? (((size_t)img * a.gr + y) * a.gc + x) * a.cout + 4 * v4 : 0);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(s_dy + p * coutp + 4 * v4)),
                     "l"(src), "r"(in ? 16 : 0)
                     : "memory");
      }
    } else if (async) {
      const int vec = coutp / 4;
      for (int e = threadIdx.x; e < TH * kWTW * vec; e += blockDim.x) {
        const int v4 = e % vec, p = e / vec;
        const int y = y0 + p / kWTW, x = x0 + p % kWTW;
        const bool in = y < a.gr && x < a.gc;
        const float* src = a.dy + (in ? (((size_t)img * a.gr + y) * a.gc + x) * a.cout + 4 * v4 : 0);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(s_dy + p * coutp + 4 * v4)),
                     "l"(src), "r"(in ? 16 : 0)
                     : "memory");
      }
    } else {
      for (int e = threadIdx.x; e < TH * kWTW * coutp; e += blockDim.x) {
        const int co = e % coutp, p = e / coutp;
        const int y = y0 + p / kWTW, x = x0 + p % kWTW;
        float v = 0.f;
        if (co < a.cout && y < a.gr && x < a.gc) v = a.dy[(((size_t)img * a.gr + y) * a.gc + x) * a.cout + co];
        s_dy[e] = v;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  if (blockIdx.x < total) stage(blockIdx.x, 0);
  int it = 0;
  for (long long tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
    if (tile + gridDim.x < total) stage(tile + gridDim.x, (it + 1) & 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const float* s_img = sm + (it & 1) * buf_floats;
    const float* s_dy = s_img + IMG;
    if (active) {
      const float* irow = s_img + (stream + ky) * IW;
      const float* drow = s_dy + (stream * kWTW) * coutp + cog * kWCO;
      float win[K];
#pragma unroll
      for (int u = 0; u < K; ++u) win[u] = irow[u];
#pragma unroll 8
      for (int px = 0; px < kWTW; ++px) {
        const float4* dp = reinterpret_cast<const float4*>(drow + px * coutp);
        const float4 d0 = dp[0], d1 = dp[1];
        const float dv[kWCO] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
        for (int o = 0; o < kWCO; ++o)
#pragma unroll
          for (int u = 0; u < K; ++u) acc[o][u] = fmaf(dv[o], win[u], acc[o][u]);
#pragma unroll
        for (int u = 0; u + 1 < K; ++u) win[u] = win[u + 1];
        win[K - 1] = irow[px + K];  // the last read (px = 31) lands in the row's halo
      }
    }
    __syncthreads();
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  const int KK = K * K;
  if (active) {
#pragma unroll
    for (int o = 0; o < kWCO; ++o)
#pragma unroll
      for (int u = 0; u < K; ++u) s_red[(stream * coutp + cog * kWCO + o) * KK + ky * K + u] = acc[o][u];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < a.cout * KK; e += blockDim.x) {
    float s = 0.f;
    for (int q = 0; q < TH; ++q) s += s_red[q * coutp * KK + e];
    a.part[(size_t)blockIdx.x * a.cout * KK + e] = s;
  }
}

// ------------------------------------------------------------------ fused conv + MPF
// First convolution + activation + the MaxPoolingFragment layer after it (Alg. 1 then
// Alg. 3) in one pass: the conv outputs of a 16 x 16 tile of
// pool windows plus a P - 1 halo are computed into shared memory with exactly the
// arithmetic of conv_first_fwd_kernel (same FMA order, same SFU activation), and pooled
// there with exactly the rule of mpf_fwd_kernel (row-major first maximum) — so the pooled
// values and argmax bytes equal the two-kernel path bit for bit, while the conv output
// (the largest tensor of the network) never reaches HBM.
constexpr int kCT = 16;  // conv outputs per tile side: (16 - P + 1)^2 pool windows, one
                         // 4-wide strip per thread for 4 map groups (no idle second round)

template <int K, int P>
__global__ void __launch_bounds__(256, 3) conv_first_mpf_kernel(FirstConvArgs a, MpfArgs m) {
  extern __shared__ float smf[];
  constexpr int kPT = kCT - P + 1;                       // pool windows per tile side
  constexpr int RY = kCT, RX = kCT;                      // conv outputs needed by the tile
  constexpr int NS = (RX + kFPX - 1) / kFPX;             // 4-wide strips per conv row
  constexpr int IW = NS * kFPX + K - 1, IH = RY + K - 1;  // image tile
  constexpr int IMG = (IH * IW + 3) / 4 * 4;
  const int coutp = a.n_cog * kFCO;
  float* s_img = smf;                    // [IH][IW]
  float* s_w = smf + IMG;                // [K*K][coutp]
  float* s_b = s_w + K * K * coutp;      // [coutp]
  float* s_y = s_b + coutp;              // [RY][RX][coutp]
  const int img = blockIdx.z;
  const int wy0 = blockIdx.y * kPT, wx0 = blockIdx.x * kPT;  // first window = first conv output
  for (int e = threadIdx.x; e < IH * IW; e += blockDim.x) {
    const int iy = e / IW, ix = e % IW;
    const int gy = wy0 + iy, gx = wx0 + ix;
    float v = 0.f;
    if (gy < a.H && gx < a.W) v = a.img[((size_t)img * a.H + gy) * a.W + gx];
    s_img[e] = v;
  }
  for (int e = threadIdx.x; e < K * K * coutp; e += blockDim.x) {
    const int co = e % coutp, t = e / coutp;
    s_w[e] = co < a.cout ? a.w[co * K * K + t] : 0.f;
  }
  for (int e = threadIdx.x; e < coutp; e += blockDim.x) s_b[e] = e < a.cout ? a.bias[e] : 0.f;
  __syncthreads();
  // ---- conv outputs of the tile (4 positions x 8 maps per thread, as conv_first_fwd_kernel)
  const int cog = threadIdx.x % a.n_cog, strip0 = threadIdx.x / a.n_cog, nstrip = blockDim.x / a.n_cog;
  for (int strip = strip0; strip < RY * NS; strip += nstrip) {
    const int ty = strip / NS, tx = (strip % NS) * kFPX;
    float acc[kFPX][kFCO];
#pragma unroll
    for (int q = 0; q < kFPX; ++q)
#pragma unroll
      for (int o = 0; o < kFCO; ++o) acc[q][o] = 0.f;
#pragma unroll
    for (int ky = 0; ky < K; ++ky) {
      float row[kFPX + K - 1];
#pragma unroll
      for (int i = 0; i < kFPX + K - 1; ++i) row[i] = s_img[(ty + ky) * IW + tx + i];
#pragma unroll
      for (int kx = 0; kx < K; ++kx) {
        const float4* wp = reinterpret_cast<const float4*>(s_w + (ky * K + kx) * coutp + cog * kFCO);
        const float4 w0 = wp[0], w1 = wp[1];
        const float wv[kFCO] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int q = 0; q < kFPX; ++q)
#pragma unroll
          for (int o = 0; o < kFCO; ++o) acc[q][o] = fmaf(row[q + kx], wv[o], acc[q][o]);
      }
    }
#pragma unroll
    for (int q = 0; q < kFPX; ++q) {
      if (tx + q >= RX) continue;
      float* dst = s_y + (ty * RX + tx + q) * coutp + cog * kFCO;
#pragma unroll
      for (int o = 0; o < kFCO; ++o) dst[o] = act_fwd(a.act, acc[q][o] + s_b[cog * kFCO + o]);
    }
  }
  __syncthreads();
  // ---- MPF forward of the tile's windows (first maximum in row-major order, R6)
  const int C = a.cout, CV = C / 4;
  const int Yw = P * m.m_r, Xw = P * m.m_c;
  for (int e = threadIdx.x; e < kPT * kPT * CV; e += blockDim.x) {
    const int cv = e % CV, w = e / CV, ty = w / kPT, tx = w % kPT;
    const int wy = wy0 + ty, wx = wx0 + tx;
    if (wy >= Yw || wx >= Xw) continue;
    float best[4];
    uint8_t arg[4];
#pragma unroll
    for (int dy = 0; dy < P; ++dy) {
      float hm[4];
      uint8_t ha[4];
#pragma unroll
      for (int dx = 0; dx < P; ++dx) {
        const float4 v = *reinterpret_cast<const float4*>(s_y + ((ty + dy) * RX + tx + dx) * coutp + cv * 4);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (dx == 0 || vv[u] > hm[u]) { hm[u] = vv[u]; ha[u] = (uint8_t)dx; }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (dy == 0 || hm[u] > best[u]) { best[u] = hm[u]; arg[u] = (uint8_t)(dy * P + ha[u]); }
    }
    if (m.round_tf32) {
#pragma unroll
      for (int u = 0; u < 4; ++u) best[u] = tf32_rn(best[u]);
    }
    const int f = (wy % P) * P + (wx % P);
    const size_t o = ((((size_t)img * P * P + f) * m.m_r + wy / P) * m.m_c + wx / P) * C + cv * 4;
    *reinterpret_cast<float4*>(m.out + o) = make_float4(best[0], best[1], best[2], best[3]);
    *reinterpret_cast<uchar4*>(m.idx + o) = make_uchar4(arg[0], arg[1], arg[2], arg[3]);
  }
}

template <int K, int P>
cudaError_t fused_kp(FirstConvArgs a, const MpfArgs& m, cudaStream_t s) {
  a.n_cog = (a.cout + kFCO - 1) / kFCO;
  const int coutp = a.n_cog * kFCO;
  constexpr int RY = kCT, RX = kCT, NS = (RX + kFPX - 1) / kFPX;
  constexpr int IW = NS * kFPX + K - 1, IH = RY + K - 1, IMG = (IH * IW + 3) / 4 * 4;
  const size_t smem = sizeof(float) * (IMG + K * K * coutp + coutp + (size_t)RY * RX * coutp);
  cudaError_t e = cudaFuncSetAttribute(conv_first_mpf_kernel<K, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  constexpr int kPT = kCT - P + 1;
  dim3 grid((P * m.m_c + kPT - 1) / kPT, (P * m.m_r + kPT - 1) / kPT, a.n);
  conv_first_mpf_kernel<K, P><<<grid, 256, smem, s>>>(a, m);
  return cudaGetLastError();
}

template <int K>
cudaError_t fused_k(const FirstConvArgs& a, const MpfArgs& m, cudaStream_t s) {
  if (m.k == 2) return fused_kp<K, 2>(a, m, s);
  if (m.k == 3) return fused_kp<K, 3>(a, m, s);
  return cudaErrorInvalidValue;
}


template <int K>
size_t fwd_smem(int coutp) {
  return sizeof(float) * (((kFTH + K - 1) * (kFTW + K - 1) + 3) / 4 * 4 + K * K * coutp + coutp);
}

template <int K>
cudaError_t fwd_k(const FirstConvArgs& a, cudaStream_t s) {
  const int coutp = a.n_cog * kFCO;
  const size_t smem = fwd_smem<K>(coutp);
  cudaError_t e = cudaFuncSetAttribute(conv_first_fwd_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((a.out_gc + kFTW - 1) / kFTW, (a.out_gr + kFTH - 1) / kFTH, a.n);
  conv_first_fwd_kernel<K><<<grid, 64 * a.n_cog, smem, s>>>(a);
  return cudaGetLastError();
}

// K >= 5: the row-streamed kernel (WT = K taps per thread); K < 5: WT = kWT
static bool wgrad_row(int k) { return k >= 5; }

template <int K, int WT>
size_t wgrad_smem(int n_cog) {
  const int coutp = n_cog * kWCO;
  constexpr int NT = (K * K + WT - 1) / WT;
  const int n_streams = 256 / (n_cog * NT);
  const size_t tile = (size_t)kWTH * kWTW * coutp;
  const size_t red = (size_t)n_streams * coutp * K * K;
  const size_t bufs = 2 * ((((kWTH + K - 1) * (kWTW + K - 1) + 3) / 4 * 4) + tile);
  return sizeof(float) * (bufs > red ? bufs : red);
}

template <int K, int WT>
cudaError_t wgrad_kw(const FirstWgradArgs& a, cudaStream_t s) {
  const size_t smem = wgrad_smem<K, WT>(a.n_cog);
  cudaError_t e = cudaFuncSetAttribute(conv_first_wgrad_kernel<K, WT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  conv_first_wgrad_kernel<K, WT><<<a.n_blocks, 256, smem, s>>>(a);
  return cudaGetLastError();
}
template <int K>
cudaError_t wgrad_k(const FirstWgradArgs& a, cudaStream_t s) {
  if constexpr (K >= 5) {
    {  // row-streamed tiles: TH = thread streams rows of 32
      const int coutp = a.n_cog * kWCO;
      const int TH = 256 / (a.n_cog * K);
      const size_t img = ((size_t)(TH + K - 1) * (kWTW + K - 1) + 3) / 4 * 4;
      const size_t bufs = 2 * (img + (size_t)TH * kWTW * coutp);
      const size_t red = (size_t)TH * coutp * K * K;
      const size_t smem = sizeof(float) * (bufs > red ? bufs : red);
      cudaError_t e = cudaFuncSetAttribute(conv_first_wgrad_rows_kernel<K>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      conv_first_wgrad_rows_kernel<K><<<a.n_blocks, 256, smem, s>>>(a, TH);
      return cudaGetLastError();
    }
  }
  return wgrad_kw<K, kWT>(a, s);
}

}  // namespace

// Fused first conv + MPF (SURVEY §8(f) 1 for the first layer): C_out a multiple of 8 (float4
// pooling, 8-map groups), pool 2 or 3.  Opt-in (MPF_FLAG_FUSE_FIRST_POOL): bitwise equal to
// the two kernels but measured slower -- 1.66 vs 0.97 + 0.42 ms on cfg4, 0.60 vs 0.23 + 0.21 ms
// on cfg5: the halo (14-31 % more conv outputs), the per-tile weight staging and the
// serialised conv -> pool phases of a CTA cost more than the conv output's HBM round trip
// saves.
bool first_conv_mpf_supported(int cout, int k, int pool_k) {
  return cout % 8 == 0 && cout <= 32 && k >= 2 && k <= 8 && (pool_k == 2 || pool_k == 3);
}

cudaError_t launch_first_conv_mpf(const FirstConvArgs& a, const MpfArgs& m, cudaStream_t s) {
  switch (a.k) {
    case 2: return fused_k<2>(a, m, s);
    case 3: return fused_k<3>(a, m, s);
    case 4: return fused_k<4>(a, m, s);
    case 5: return fused_k<5>(a, m, s);
    case 6: return fused_k<6>(a, m, s);
    case 7: return fused_k<7>(a, m, s);
    case 8: return fused_k<8>(a, m, s);
    default: return cudaErrorInvalidValue;
  }
}

bool first_conv_supported(int cin, int cout, int k) {
  if (cin != 1 || cout < 1 || cout > 32 || k < 2 || k > 8) return false;
  const int n_cog = (cout + kFCO - 1) / kFCO;
  const int NT = (k * k + kWT - 1) / kWT;
  return n_cog * NT <= 256;
}

// co-resident CTAs per SM overlap staging with compute: 3 (2 for the row variant)
int first_wgrad_blocks(int k) { return 148 * (k > 0 && wgrad_row(k) ? 2 : 3); }

cudaError_t launch_first_conv(FirstConvArgs a, cudaStream_t s) {
  a.n_cog = (a.cout + kFCO - 1) / kFCO;
  switch (a.k) {
    case 2: return fwd_k<2>(a, s);
    case 3: return fwd_k<3>(a, s);
    case 4: return fwd_k<4>(a, s);
    case 5: return fwd_k<5>(a, s);
    case 6: return fwd_k<6>(a, s);
    case 7: return fwd_k<7>(a, s);
    case 8: return fwd_k<8>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_first_wgrad(FirstWgradArgs a, cudaStream_t s) {
  a.n_cog = (a.cout + kWCO - 1) / kWCO;
  switch (a.k) {
    case 2: return wgrad_k<2>(a, s);
    case 3: return wgrad_k<3>(a, s);
    case 4: return wgrad_k<4>(a, s);
    case 5: return wgrad_k<5>(a, s);
    case 6: return wgrad_k<6>(a, s);
    case 7: return wgrad_k<7>(a, s);
    case 8: return wgrad_k<8>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace mpf
