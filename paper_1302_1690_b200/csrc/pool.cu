// pool.cu — MaxPoolingFragment forward / backward (HBM-bound) and the deterministic
// per-channel reductions that produce bias gradients.
//
// MPF forward, Alg. 3.  For input fragment g and offset (r, c)
// (row-major, reading R2) output fragment g*k^2 + r*k + c holds, at cell (i, j), the
// max of the k x k block with top-left (r + k i, c + k j) and its argmax (first maximum
// in row-major scan, R6).  Every block position Y = r + k i, X = c + k j is a distinct
// point of the stride-1 "window grid" [0, k m_r) x [0, k m_c), so the kernel walks that
// grid: one thread owns a column X and one 4-channel vector and slides down a band of
// rows keeping the k horizontal row maxima in registers — each input element comes
// from HBM once and from L1 k times (instead of k^2).
//
// MPF backward, Alg. 4 (reading R3) as a gather: conv-output element
// (Y', X') sums, in fixed (dy, dx) order, the deltas of every window (Y'-dy, X'-dx)
// whose recorded argmax is (dy, dx) — shared maxima ADD (Fig. 2) —
// times act'(y) taken from the pooled value of a selecting window (it equals y at
// (Y', X')).  Deterministic, no atomics.  The same pass adds the delta into a
// per-block, per-channel partial sum: the bias gradient of the conv that produced y
// (Alg. 2: the sum over all fragments and positions), finished by bias_reduce in a
// fixed order.
//
// All index arithmetic is 32-bit per fragment; only final offsets are 64-bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "mpf_internal.h"
#include "numerics.cuh"

namespace mpf {

namespace {


__device__ __forceinline__ float act_der(int act, float y) {
  if (act == MPF_TANH) return 1.f - y * y;
  if (act == MPF_LOGISTIC) return y * (1.f - y);
  return 1.f;
}

template <int V>
struct Vec {
  float v[V];
};

template <int V>
__device__ __forceinline__ Vec<V> ldv(const float* p) {
  Vec<V> r;
  if constexpr (V == 4) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    r.v[0] = q.x; r.v[1] = q.y; r.v[2] = q.z; r.v[3] = q.w;
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) r.v[i] = __ldg(p + i);
  }
  return r;
}

template <int V>
__device__ __forceinline__ void stv(float* p, const float (&v)[V]) {
  if constexpr (V == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) p[i] = v[i];
  }
}

template <int V>
__device__ __forceinline__ void stidx(uint8_t* p, const uint8_t (&a)[V]) {
  if constexpr (V == 4) {
    *reinterpret_cast<uchar4*>(p) = make_uchar4(a[0], a[1], a[2], a[3]);
  } else {
#pragma unroll
    for (int i = 0; i < V; ++i) p[i] = a[i];
  }
}

constexpr int kBand = 16;  // window rows per thread (forward) / output rows per thread (backward)

int block_dims(int C, int V, dim3* blk) {
  const int CV = C / V;
  int ty = 256 / CV;
  if (ty < 1) ty = 1;
  *blk = dim3(CV, ty, 1);
  return ty;
}

// ----------------------------------------------------------------------------- forward
template <int K, int V>
__global__ void __launch_bounds__(256, K <= 3 ? 4 : 2) mpf_fwd_kernel(MpfArgs a) {
  const int cv = threadIdx.x;
  const int X = blockIdx.x * blockDim.y + threadIdx.y;
  const int Xw = K * a.m_c, Yw = K * a.m_r;
  if (X >= Xw) return;
  const int y0 = blockIdx.y * kBand;
  const int y1 = min(y0 + kBand, Yw);
  const int c = X % K, j = X / K;
  const int C = a.C;
  for (int g = blockIdx.z; g < a.n_frag_in; g += gridDim.z) {
    const float* src = a.y + ((size_t)g * a.gr * a.gc + X) * C + cv * V;
    // raw loads of row r, issued two window rows ahead of their use (ring of two row
    // buffers) so that two rows of loads are in flight per thread: the loop is
    // load-latency-bound otherwise
    auto lrow = [&](int r, Vec<V> (&q)[K]) {
      const float* p = src + (size_t)r * a.gc * C;
#pragma unroll
      for (int dx = 0; dx < K; ++dx) q[dx] = ldv<V>(p + dx * C);
    };
    float hm[K][V];
    uint8_t ha[K][V];
    // horizontal max of a loaded row over dx = 0..K-1 (first maximum) into hm/ha[d]
    auto hrow = [&](const Vec<V> (&q)[K], int d) {
#pragma unroll
      for (int v = 0; v < V; ++v) { hm[d][v] = q[0].v[v]; ha[d][v] = 0; }
#pragma unroll
      for (int dx = 1; dx < K; ++dx)
#pragma unroll
        for (int v = 0; v < V; ++v)
          if (q[dx].v[v] > hm[d][v]) { hm[d][v] = q[dx].v[v]; ha[d][v] = (uint8_t)dx; }
    };
    Vec<V> rawA[K], rawB[K];
#pragma unroll
    for (int d = 1; d < K; ++d) {
      lrow(y0 + d - 1, rawA);
      hrow(rawA, d);
    }
    lrow(y0 + K - 1, rawA);
    if (y0 + 1 < y1) lrow(y0 + K, rawB);
    const size_t frag_base = (size_t)g * K * K;
    // one output row: consume `cur` (window row Y+K-1), refill it with row Y+K+1
    auto step = [&](int Y, Vec<V> (&cur)[K]) {
#pragma unroll
      for (int d = 0; d < K - 1; ++d) {
#pragma unroll
        for (int v = 0; v < V; ++v) { hm[d][v] = hm[d + 1][v]; ha[d][v] = ha[d + 1][v]; }
      }
      hrow(cur, K - 1);
      if (Y + 2 < y1) lrow(Y + K + 1, cur);
      float best[V];
      uint8_t arg[V];
#pragma unroll
      for (int v = 0; v < V; ++v) { best[v] = hm[0][v]; arg[v] = ha[0][v]; }
#pragma unroll
      for (int d = 1; d < K; ++d)
#pragma unroll
        for (int v = 0; v < V; ++v)
          if (hm[d][v] > best[v]) { best[v] = hm[d][v]; arg[v] = (uint8_t)(d * K + ha[d][v]); }
      const int r = Y % K, i = Y / K;
      const size_t o = (((frag_base + r * K + c) * a.m_r + i) * a.m_c + j) * C + cv * V;
      if (a.round_tf32) {
#pragma unroll
        for (int v = 0; v < V; ++v) best[v] = tf32_rn(best[v]);
      }
      stv<V>(a.out + o, best);
      stidx<V>(a.idx + o, arg);
    };
    for (int Y = y0; Y < y1; Y += 2) {
      step(Y, rawA);
      if (Y + 1 < y1) step(Y + 1, rawB);
    }
  }
}

template <int K, int V>
cudaError_t fwd_launch(const MpfArgs& a, cudaStream_t s) {
  dim3 blk;
  const int ty = block_dims(a.C, V, &blk);
  const int Xw = K * a.m_c, Yw = K * a.m_r;
  dim3 grid((Xw + ty - 1) / ty, (Yw + kBand - 1) / kBand, a.n_frag_in < 65535 ? a.n_frag_in : 65535);
  mpf_fwd_kernel<K, V><<<grid, blk, 0, s>>>(a);
  return cudaGetLastError();
}

// generic k (any pooling factor): plain k x k scan per window
template <int V>
__global__ void __launch_bounds__(256) mpf_fwd_generic_kernel(MpfArgs a) {
  const int cv = threadIdx.x;
  const int K = a.k;
  const int X = blockIdx.x * blockDim.y + threadIdx.y;
  const int Xw = K * a.m_c, Yw = K * a.m_r;
  if (X >= Xw) return;
  const int y0 = blockIdx.y * kBand, y1 = min(y0 + kBand, Yw);
  const int c = X % K, j = X / K;
  for (int g = blockIdx.z; g < a.n_frag_in; g += gridDim.z) {
    for (int Y = y0; Y < y1; ++Y) {
      const float* src = a.y + (((size_t)g * a.gr + Y) * a.gc + X) * a.C + cv * V;
      float best[V];
      uint8_t arg[V];
      Vec<V> q = ldv<V>(src);
#pragma unroll
      for (int v = 0; v < V; ++v) { best[v] = q.v[v]; arg[v] = 0; }
      for (int dy = 0; dy < K; ++dy)
        for (int dx = 0; dx < K; ++dx) {
          if (dy == 0 && dx == 0) continue;
          q = ldv<V>(src + ((size_t)dy * a.gc + dx) * a.C);
#pragma unroll
          for (int v = 0; v < V; ++v)
            if (q.v[v] > best[v]) { best[v] = q.v[v]; arg[v] = (uint8_t)(dy * K + dx); }
        }
      const int r = Y % K, i = Y / K;
      const size_t o = ((((size_t)g * K * K + r * K + c) * a.m_r + i) * a.m_c + j) * a.C + cv * V;
      if (a.round_tf32) {
#pragma unroll
        for (int v = 0; v < V; ++v) best[v] = tf32_rn(best[v]);
      }
      stv<V>(a.out + o, best);
      stidx<V>(a.idx + o, arg);
    }
  }
}

template <int V>
cudaError_t fwd_dispatch(const MpfArgs& a, cudaStream_t s) {
  if (a.k == 2) return fwd_launch<2, V>(a, s);
  if (a.k == 3) return fwd_launch<3, V>(a, s);
  if (a.k == 4) return fwd_launch<4, V>(a, s);
  dim3 blk;
  const int ty = block_dims(a.C, V, &blk);
  const int Xw = a.k * a.m_c, Yw = a.k * a.m_r;
  dim3 grid((Xw + ty - 1) / ty, (Yw + kBand - 1) / kBand, a.n_frag_in < 65535 ? a.n_frag_in : 65535);
  mpf_fwd_generic_kernel<V><<<grid, blk, 0, s>>>(a);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- backward
template <int V>
__global__ void __launch_bounds__(256) mpf_bwd_kernel(MpfBwdArgs a) {
  extern __shared__ float s_red[];  // [blockDim.y][C]
  const int cv = threadIdx.x;
  const int K = a.k, KK = K * K;
  const int X = blockIdx.x * blockDim.y + threadIdx.y;
  const int Xw = K * a.m_c, Yw = K * a.m_r;
  const int y0 = blockIdx.y * kBand, y1 = min(y0 + kBand, a.gr);
  const int C = a.C;
  float bsum[V];
#pragma unroll
  for (int v = 0; v < V; ++v) bsum[v] = 0.f;
  if (X < a.gc) {
    for (int g = blockIdx.z; g < a.n_frag_in; g += gridDim.z) {
      const size_t cell_frag0 = (size_t)g * KK;
      for (int Y = y0; Y < y1; ++Y) {
        float acc[V], val[V];
        bool hit[V];
#pragma unroll
        for (int v = 0; v < V; ++v) { acc[v] = 0.f; val[v] = 0.f; hit[v] = false; }
        if (Y < a.vr && X < a.vc) {
          for (int dy = 0; dy < K; ++dy) {
            const int wy = Y - dy;
            if (wy < 0) break;
            if (wy >= Yw) continue;
            const int r = wy % K, i = wy / K;
            for (int dx = 0; dx < K; ++dx) {
              const int wx = X - dx;
              if (wx < 0) break;
              if (wx >= Xw) continue;
              const int c = wx % K, j = wx / K;
              const size_t cell = (((cell_frag0 + r * K + c) * a.m_r + i) * a.m_c + j) * C + cv * V;
              const uint8_t want = (uint8_t)(dy * K + dx);
              uint8_t id[V];
              if constexpr (V == 4) {
                const uchar4 q = __ldg(reinterpret_cast<const uchar4*>(a.idx + cell));
                id[0] = q.x; id[1] = q.y; id[2] = q.z; id[3] = q.w;
              } else {
#pragma unroll
                for (int v = 0; v < V; ++v) id[v] = __ldg(a.idx + cell + v);
              }
              bool any = false;
#pragma unroll
              for (int v = 0; v < V; ++v) any |= (id[v] == want);
              if (any) {
                const Vec<V> d = ldv<V>(a.dout + cell);
                const Vec<V> pv = a.premul ? d : ldv<V>(a.pooled + cell);
#pragma unroll
                for (int v = 0; v < V; ++v)
                  if (id[v] == want) { acc[v] += d.v[v]; val[v] = pv.v[v]; hit[v] = true; }
              }
            }
          }
        }
        float o[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const float dv = hit[v] ? (a.premul ? acc[v] : acc[v] * act_der(a.act, val[v])) : 0.f;
          bsum[v] += dv;
          o[v] = a.round_tf32 ? tf32_rn(dv) : dv;
        }
        stv<V>(a.din + (((size_t)g * a.gr + Y) * a.gc + X) * C + cv * V, o);
      }
    }
  }
  if (a.bias_part == nullptr) return;
  // fixed-order block reduction of the bias partials over threadIdx.y
#pragma unroll
  for (int v = 0; v < V; ++v) s_red[threadIdx.y * C + cv * V + v] = bsum[v];
  __syncthreads();
  if (threadIdx.y == 0) {
    const size_t blin = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float t = 0.f;
      for (int q = 0; q < (int)blockDim.y; ++q) t += s_red[q * C + cv * V + v];
      a.bias_part[blin * C + cv * V + v] = t;
    }
  }
}

// Shared-memory tiled gather (premul deltas, 4-channel vectors, any K <= 4).  A CTA owns
// a TY x TX tile of conv-output positions of one input fragment and walks down the
// fragment's rows tile by tile.  Per tile it first stages, with fully coalesced and
// mutually independent loads, the argmax bytes and deltas of every window that can
// select a tile element ((TY+K-1) x (TX+K-1) windows, absent windows marked 0xFF), then
// every element gathers its K^2 candidates from shared memory in the same fixed (dy, dx)
// order as the other MPF backward kernels (bitwise-identical results).  No dependent
// global-load chains remain; the halo re-reads hit L2.
// Shared-memory layout, channel-vector-major so that every candidate window of an element
// sits at a compile-time offset from the element's own cell (LDS [base + imm], no
// per-window address arithmetic); S = cells per channel vector, odd, so that the lanes
// of a warp (consecutive cv) hit distinct banks:
//   argmax words  s_id[(cv / 4) * S * 4 + cell * 4 + cv % 4]   (4 cv per 16-byte chunk)
//   deltas        s_d [cv * S + cell]                          (float4)
__host__ __device__ constexpr int tile_cells_padded(int wy, int wx) { return (wy * wx) | 1; }

template <int K, int kTBY, int kTBX>
__global__ void __launch_bounds__(256) mpf_bwd_tile_kernel(MpfBwdArgs a, int rows_per_cta, int nbuf) {
  extern __shared__ __align__(16) uint8_t sm_raw[];
  constexpr int WY = kTBY + K - 1, WX = kTBX + K - 1, S = tile_cells_padded(WY, WX);
  const int C = a.C, CV = C / 4, CVP = (CV + 3) & ~3;
  // nbuf staging buffers [argmax words | deltas], then the bias reduction area
  const size_t buf_bytes = (size_t)CVP * S * 4 + (size_t)CV * S * 16;
  float* s_red = reinterpret_cast<float*>(sm_raw + nbuf * buf_bytes);  // [256 / CV][C]
  const int Xw = K * a.m_c, Yw = K * a.m_r;
  const int MM = a.m_r * a.m_c;
  const int X0 = blockIdx.x * kTBX;
  const int tid = threadIdx.x;
  const int cv = tid % CV, pt = tid / CV, npt = 256 / CV;  // compute mapping (pt < npt)
  float bsum[4] = {0.f, 0.f, 0.f, 0.f};
  const int ybeg = blockIdx.y * rows_per_cta, yend = min(ybeg + rows_per_cta, a.gr);
  // argmax bytes are staged in 16-byte chunks (4 channel vectors) when C allows it
  const bool idx16 = C % 16 == 0;
  const int CI = idx16 ? C / 16 : CV;
  const int ci = tid % CI, pi = tid / CI, npi = 256 / CI;
  // per-fragment strides (32-bit: one input fragment's pooled output is < 2^31 elements)
  const int MMC = MM * C, mcC = a.m_c * C;
  // this CTA's tiles: (input fragment g, first row Y0), g-major
  const int n_yt = yend > ybeg ? (yend - ybeg + kTBY - 1) / kTBY : 0;
  const int n_g = blockIdx.z < a.n_frag_in ? (a.n_frag_in - blockIdx.z + gridDim.z - 1) / gridDim.z : 0;
  const int n_tiles = n_yt * n_g;

  // ---- stage tile `it` into buffer `buf`: windows wy in [Y0-K+1, Y0+kTBY), wx in
  // [X0-K+1, X0+kTBX).  cp.async: global -> shared without a register round trip, so
  // every thread keeps all of its staging loads in flight; absent windows read as idx
  // 0xFF.., delta 0.  Division-free apart from the compile-time WX and K.
  auto stage = [&](int it, int buf) {
    const int g = blockIdx.z + (it / n_yt) * gridDim.z, Y0 = ybeg + (it % n_yt) * kTBY;
    const size_t fbase = (size_t)g * K * K * MM * C;
    const float* dsrc = a.dout + fbase;
    const uint8_t* isrc = a.idx + fbase;
    uint32_t* s_id = reinterpret_cast<uint32_t*>(sm_raw + buf * buf_bytes);       // [CVP / 4][S][4]
    float4* s_d = reinterpret_cast<float4*>(sm_raw + buf * buf_bytes + (size_t)CVP * S * 4);  // [CV][S]
    if (pt < npt) {
      float4* s_d_cv = s_d + cv * S;
      for (int t = pt; t < WY * WX; t += npt) {
        const int wyl = t / WX, wxl = t - wyl * WX;
        const int wy = Y0 - K + 1 + wyl, wx = X0 - K + 1 + wxl;
        float4* dst = s_d_cv + t;
        if ((unsigned)wy < (unsigned)Yw && (unsigned)wx < (unsigned)Xw) {
          const unsigned uy = wy, ux = wx;
          const int off = (int)((uy % K) * K + ux % K) * MMC + (int)(uy / K) * mcC + (int)(ux / K) * C + cv * 4;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                       "l"(dsrc + off)
                       : "memory");
        } else {
          *dst = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
    if (pi < npi) {
      for (int t = pi; t < WY * WX; t += npi) {
        const int wyl = t / WX, wxl = t - wyl * WX;
        const int wy = Y0 - K + 1 + wyl, wx = X0 - K + 1 + wxl;
        const bool in = (unsigned)wy < (unsigned)Yw && (unsigned)wx < (unsigned)Xw;
        const unsigned uy = in ? wy : 0, ux = in ? wx : 0;
        const int off = (int)((uy % K) * K + ux % K) * MMC + (int)(uy / K) * mcC + (int)(ux / K) * C;
        if (idx16) {
          uint32_t* dst = s_id + (ci * S + t) * 4;
          if (in)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                         "l"(isrc + off + ci * 16)
                         : "memory");
          else
            *reinterpret_cast<uint4*>(dst) = make_uint4(~0u, ~0u, ~0u, ~0u);
        } else {
          uint32_t* dst = s_id + ((ci >> 2) * S + t) * 4 + (ci & 3);
          if (in)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
                         "l"(isrc + off + ci * 4)
                         : "memory");
          else
            *dst = ~0u;
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };

  // Two buffers: tile it + 1 is in flight while tile it is gathered.
  if (n_tiles > 0) stage(0, 0);
  for (int it = 0; it < n_tiles; ++it) {
    const int buf = nbuf == 2 ? (it & 1) : 0;
    if (nbuf == 2 && it + 1 < n_tiles) {
      stage(it + 1, buf ^ 1);  // that buffer was last read by tile it - 1 (barrier below)
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // tile it's staging (all threads' copies and fills) is visible
    const int g = blockIdx.z + (it / n_yt) * gridDim.z, Y0 = ybeg + (it % n_yt) * kTBY;
    float* const dst_g = a.din + (size_t)g * a.gr * a.gc * C + cv * 4;  // one fragment < 2^31 elements
    // ---- gather: element (Y0+ty, X0+tx) sums window (ty+K-1-dy, tx+K-1-dx) where idx == dy*K+dx
    if (pt < npt) {
      const uint32_t* s_id_cv =
          reinterpret_cast<const uint32_t*>(sm_raw + buf * buf_bytes) + (cv >> 2) * S * 4 + (cv & 3);
      const float4* s_d_cv = reinterpret_cast<const float4*>(sm_raw + buf * buf_bytes + (size_t)CVP * S * 4) + cv * S;
      for (unsigned q = pt; q < kTBY * kTBX; q += npt) {
        const int ty = q / kTBX, tx = q % kTBX;
        const int Y = Y0 + ty, X = X0 + tx;
        if (Y >= yend || X >= a.gc) continue;
        const int cell = (ty + K - 1) * WX + (tx + K - 1);
        const uint32_t* pid = s_id_cv + cell * 4;
        const float4* pd = s_d_cv + cell;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int dy = 0; dy < K; ++dy)
#pragma unroll
          for (int dx = 0; dx < K; ++dx) {
            const int wo = dy * WX + dx;  // compile-time after unrolling
            // byte v of `x` is zero iff channel v of this window selected (dy, dx)
            const uint32_t x = pid[-wo * 4] ^ ((uint32_t)(dy * K + dx) * 0x01010101u);
            const float4 d = pd[-wo];
            if (!(x & 0xFFu)) acc[0] += d.x;
            if (!(x & 0xFF00u)) acc[1] += d.y;
            if (!(x & 0xFF0000u)) acc[2] += d.z;
            if (!(x & 0xFF000000u)) acc[3] += d.w;
          }
        float o[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          bsum[v] += acc[v];
          o[v] = a.round_tf32 ? tf32_rn(acc[v]) : acc[v];
        }
        stv<4>(dst_g + (Y * a.gc + X) * C, o);
      }
    }
    __syncthreads();  // buffer `buf` fully consumed before it is refilled
    if (nbuf == 1 && it + 1 < n_tiles) stage(it + 1, 0);
  }
  if (a.bias_part == nullptr) return;
  __syncthreads();
  if (pt < npt) {
#pragma unroll
    for (int v = 0; v < 4; ++v) s_red[pt * C + cv * 4 + v] = bsum[v];
  }
  __syncthreads();
  if (tid < CV) {
    const size_t blin = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      float t = 0.f;
      for (int q2 = 0; q2 < npt; ++q2) t += s_red[q2 * C + tid * 4 + v];
      a.bias_part[blin * C + tid * 4 + v] = t;
    }
  }
}

// Bias partials of the register-blocked gathers (thread = channel vector cv of group sub):
// for C / 4 <= 32 one row per warp -- leader lane l < C/4 adds the lanes l + j C/4 of its
// channel vector by shuffles (fixed order) -- else one row per (CTA, group); the fixed-order
// reduction kernel sums the rows.  No shared memory, so a CTA fits beside a tensor-core CTA
// on an SM (the weight gradients run concurrently on the side stream).
__device__ __forceinline__ void write_bias_rows(const MpfBwdArgs& a, const float (&bsum)[4], int sub, int nsub,
                                                int cv) {
  if (a.bias_part == nullptr) return;
  const int C = a.C, CV = C / 4;
  if (CV <= 32) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float s[4] = {bsum[0], bsum[1], bsum[2], bsum[3]};
    for (int j = 1; j * CV < 32; ++j) {
      const int src = lane + j * CV;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float v = __shfl_sync(0xffffffffu, bsum[q], src & 31);
        if (src < 32) s[q] += v;
      }
    }
    if (lane < CV) {
      const int cls = (int)(threadIdx.x % CV);
#pragma unroll
      for (int q = 0; q < 4; ++q) a.bias_part[((size_t)blockIdx.x * 8 + warp) * C + cls * 4 + q] = s[q];
    }
    return;
  }
  if (sub >= nsub) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) a.bias_part[((size_t)blockIdx.x * nsub + sub) * C + cv * 4 + q] = bsum[q];
}

// Register-blocked gather for k = 2 (premul deltas, 4-channel vectors): a thread owns a
// 2 x 2 block of conv-output elements (rows 2i, 2i+1, columns 2j, 2j+1) of one channel
// vector.  Every candidate window of the block lies in the 3 x 3 window patch rows
// 2i-1 .. 2i+1, columns 2j-1 .. 2j+1, so the thread loads those 9 windows' argmax words and
// deltas once (18 independent loads in flight, neighbouring blocks' overlap hits L1) and
// gathers each element's k^2 candidates from registers in the same fixed (dy, dx) order as
// the other MPF backward kernels (bitwise-identical results).  No shared-memory staging,
// no barriers; CTAs stride over groups of consecutive blocks of one row.
__global__ void __launch_bounds__(256, 3) mpf_bwd_block2_kernel(MpfBwdArgs a, long long n_groups) {
  const int C = a.C, CV = C / 4;
  const int tid = threadIdx.x, cv = tid % CV, sub = tid / CV, nsub = 256 / CV;
  const int Xw = 2 * a.m_c, Yw = 2 * a.m_r;
  const int MM = a.m_r * a.m_c;
  const int MMC = MM * C, mcC = a.m_c * C;
  const int bj_n = (a.gc + 1) / 2, bi_n = (a.gr + 1) / 2;
  const int groups_per_row = (bj_n + nsub - 1) / nsub;
  float bsum[4] = {0.f, 0.f, 0.f, 0.f};
  if (sub < nsub) {
    // (g, bi, gj) of group grp, advanced by gridDim.x with carries instead of divisions
    int gj = (int)(blockIdx.x % groups_per_row), bi, g;
    {
      const long long t = blockIdx.x / groups_per_row;
      bi = (int)(t % bi_n);
      g = (int)(t / bi_n);
    }
    const int st_gj = (int)(gridDim.x % groups_per_row);
    const long long st_t = gridDim.x / groups_per_row;
    const int st_bi = (int)(st_t % bi_n), st_g = (int)(st_t / bi_n);
    for (long long grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
      if (grp != blockIdx.x) {
        gj += st_gj;
        int cb = st_bi;
        if (gj >= groups_per_row) { gj -= groups_per_row; ++cb; }
        bi += cb;
        int cg = st_g;
        if (bi >= bi_n) { bi -= bi_n; ++cg; }
        g += cg;
      }
      const int bj = gj * nsub + sub;
      if (bj >= bj_n) continue;
      const float* dsrc = a.dout + (size_t)g * 4 * MMC + cv * 4;
      const uint8_t* isrc = a.idx + (size_t)g * 4 * MMC + cv * 4;
      // window patch: rows wy = 2bi - 1 + u, columns wx = 2bj - 1 + v (u, v < 3)
      uint32_t id[3][3];
      float4 d[3][3];
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int wy = 2 * bi - 1 + u;
        const bool yok = wy >= 0 && wy < Yw;
        const int rowoff = yok ? ((wy & 1) * 2) * MMC + (wy >> 1) * mcC : 0;
#pragma unroll
        for (int v = 0; v < 3; ++v) {
          const int wx = 2 * bj - 1 + v;
          const bool ok = yok && wx >= 0 && wx < Xw;
          const int off = rowoff + (wx & 1) * MMC + (wx >> 1) * C;
          id[u][v] = ok ? __ldg(reinterpret_cast<const uint32_t*>(isrc + (ok ? off : 0))) : 0xFFFFFFFFu;
          d[u][v] = ok ? __ldg(reinterpret_cast<const float4*>(dsrc + (ok ? off : 0))) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      float* dst = a.din + ((size_t)g * a.gr * a.gc) * C + cv * 4;
#pragma unroll
      for (int ea = 0; ea < 2; ++ea)
#pragma unroll
        for (int eb = 0; eb < 2; ++eb) {
          const int Y = 2 * bi + ea, X = 2 * bj + eb;
          if (Y >= a.gr || X >= a.gc) continue;
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int dy = 0; dy < 2; ++dy)
#pragma unroll
            for (int dx = 0; dx < 2; ++dx) {
              // window (Y - dy, X - dx) = patch (ea - dy + 1, eb - dx + 1)
              const uint32_t x = id[ea - dy + 1][eb - dx + 1] ^ ((uint32_t)(dy * 2 + dx) * 0x01010101u);
              const float4 w = d[ea - dy + 1][eb - dx + 1];
              if (!(x & 0xFFu)) acc[0] += w.x;
              if (!(x & 0xFF00u)) acc[1] += w.y;
              if (!(x & 0xFF0000u)) acc[2] += w.z;
              if (!(x & 0xFF000000u)) acc[3] += w.w;
            }
          float o[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            bsum[q] += acc[q];
            o[q] = a.round_tf32 ? tf32_rn(acc[q]) : acc[q];
          }
          stv<4>(dst + (Y * a.gc + X) * C, o);
        }
    }
  }
  write_bias_rows(a, bsum, sub, nsub, cv);
}

// Band form of the k = 2 gather: a thread walks its 2 x 2 block column down a band of
// `band` block rows.  Block row bi needs window patch rows 2bi-1, 2bi, 2bi+1; the next block
// row's first patch row (2bi+1) is this one's last, so it stays in registers and only two
// new patch rows (6 windows) are loaded per block instead of 9, with row offsets advanced
// by one pooled row per step instead of recomputed.  Same candidates in the same (dy, dx)
// order per element: bitwise the deltas of mpf_bwd_block2_kernel.
__global__ void __launch_bounds__(256, 3) mpf_bwd_band2_kernel(MpfBwdArgs a, long long n_units, int band_rows) {
  const int C = a.C, CV = C / 4;
  const int tid = threadIdx.x, cv = tid % CV, sub = tid / CV, nsub = 256 / CV;
  const int Xw = 2 * a.m_c, Yw = 2 * a.m_r;
  const int MMC = a.m_r * a.m_c * C, mcC = a.m_c * C;
  const int bj_n = (a.gc + 1) / 2, bi_n = (a.gr + 1) / 2;
  const int groups_per_row = (bj_n + nsub - 1) / nsub;
  const int bands = (bi_n + band_rows - 1) / band_rows;
  float bsum[4] = {0.f, 0.f, 0.f, 0.f};
  if (sub < nsub) {
    for (long long unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
      const int gj = (int)(unit % groups_per_row);
      const long long t = unit / groups_per_row;
      const int band = (int)(t % bands);
      const int g = (int)(t / bands);
      const int bj = gj * nsub + sub;
      if (bj >= bj_n) continue;
      const int bi0 = band * band_rows, bi1 = min(bi_n, bi0 + band_rows);
      const float* dsrc = a.dout + (size_t)g * 4 * MMC + cv * 4;
      const uint8_t* isrc = a.idx + (size_t)g * 4 * MMC + cv * 4;
      float* dst = a.din + ((size_t)g * a.gr * a.gc) * C + cv * 4;
      // patch columns wx = 2bj - 1 + v: parity odd, even, odd
      int coff[3];
      bool cok[3];
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        const int wx = 2 * bj - 1 + v;
        cok[v] = wx >= 0 && wx < Xw;
        coff[v] = cok[v] ? (wx & 1) * MMC + (wx >> 1) * C : 0;
      }
      auto load_row = [&](int wy, uint32_t (&ir)[3], float4 (&dr)[3]) {
        const bool yok = wy >= 0 && wy < Yw;
        const int rowoff = yok ? (wy & 1) * 2 * MMC + (wy >> 1) * mcC : 0;
#pragma unroll
        for (int v = 0; v < 3; ++v) {
          const bool ok = yok && cok[v];
          const int off = rowoff + coff[v];
          ir[v] = ok ? __ldg(reinterpret_cast<const uint32_t*>(isrc + off)) : 0xFFFFFFFFu;
          dr[v] = ok ? __ldg(reinterpret_cast<const float4*>(dsrc + off)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      };
      uint32_t id[3][3];
      float4 d[3][3];
      load_row(2 * bi0 - 1, id[0], d[0]);
      for (int bi = bi0; bi < bi1; ++bi) {
        load_row(2 * bi, id[1], d[1]);
        load_row(2 * bi + 1, id[2], d[2]);
#pragma unroll
        for (int ea = 0; ea < 2; ++ea)
#pragma unroll
          for (int eb = 0; eb < 2; ++eb) {
            const int Y = 2 * bi + ea, X = 2 * bj + eb;
            if (Y >= a.gr || X >= a.gc) continue;
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int dy = 0; dy < 2; ++dy)
#pragma unroll
              for (int dx = 0; dx < 2; ++dx) {
                const uint32_t x = id[ea - dy + 1][eb - dx + 1] ^ ((uint32_t)(dy * 2 + dx) * 0x01010101u);
                const float4 w = d[ea - dy + 1][eb - dx + 1];
                if (!(x & 0xFFu)) acc[0] += w.x;
                if (!(x & 0xFF00u)) acc[1] += w.y;
                if (!(x & 0xFF0000u)) acc[2] += w.z;
                if (!(x & 0xFF000000u)) acc[3] += w.w;
              }
            float o[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              bsum[q] += acc[q];
              o[q] = a.round_tf32 ? tf32_rn(acc[q]) : acc[q];
            }
            stv<4>(dst + (Y * a.gc + X) * C, o);
          }
#pragma unroll
        for (int v = 0; v < 3; ++v) {  // the last patch row is the next block row's first
          id[0][v] = id[2][v];
          d[0][v] = d[2][v];
        }
      }
    }
  }
  write_bias_rows(a, bsum, sub, nsub, cv);
}

// Register-blocked gather for k = 3 (premul deltas, 4-channel vectors): a thread owns a 3 x 3
// block of conv-output elements of one channel vector; the candidate windows form the 5 x 5
// patch rows 3i-2 .. 3i+2.  Output row ea needs patch rows ea .. ea+2, so the patch streams
// through a ring of 3 rows: rows 0-2 are loaded up front, row ea+3 after output row ea.  Same
// fixed (dy, dx) order as the other MPF backward kernels.  Against the first form of this
// kernel (bitwise equal deltas, tested before it was removed; cfg5 layer 5 0.86 -> 0.76-0.79 ms,
// profiles/r2/mpf_bwd_k3_lean_ab_cfg5.log) it has
//  - 32-bit work-item decoding (the grid-stride loop decoded a 64-bit group index with three
//    64-bit divisions per block);
//  - window offsets without division: patch column v of block column bj is window column
//    3 bj - 2 + v, i.e. offset fragment (v + 1) % 3, cell bj - 1 + (v + 1) / 3 -- compile-time
//    coefficients times the runtime strides -- and the same for the rows;
//  - no selects on the loads: a window outside the window grid loads from an in-bounds
//    address (its row or column offset is replaced by 0) and its argmax word is OR-ed with
//    0xFFFFFFFF, which no candidate test (byte == dy*3+dx <= 8) accepts, so its delta is
//    never added.
__global__ void __launch_bounds__(256, 2) mpf_bwd_k3_kernel(MpfBwdArgs a, int n_groups) {
  constexpr int K = 3, BW = 3, PW = 5;
  const int C = a.C, CV = C / 4;
  const int tid = threadIdx.x, cv = tid % CV, sub = tid / CV, nsub = 256 / CV;
  const int Xw = K * a.m_c, Yw = K * a.m_r;
  const int MMC = a.m_r * a.m_c * C, mcC = a.m_c * C;
  const int bj_n = (a.gc + BW - 1) / BW, bi_n = (a.gr + K - 1) / K;
  const int groups_per_row = (bj_n + nsub - 1) / nsub;
  float bsum[4] = {0.f, 0.f, 0.f, 0.f};
  if (sub < nsub) {
    for (int grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
      const int t = grp / groups_per_row;
      const int gj = grp - t * groups_per_row;
      const int g = t / bi_n;
      const int bi = t - g * bi_n;
      const int bj = gj * nsub + sub;
      if (bj >= bj_n) continue;
      const size_t fbase = (size_t)g * K * K * MMC + cv * 4;
      const float* dsrc = a.dout + fbase;
      const uint8_t* isrc = a.idx + fbase;
      int coloff[PW];
      uint32_t colbad[PW];
#pragma unroll
      for (int v = 0; v < PW; ++v) {
        const int wx = BW * bj - (K - 1) + v;
        const bool bad = wx < 0 || wx >= Xw;
        coloff[v] = bad ? 0 : ((v + 1) % K) * MMC + (bj - 1 + (v + 1) / K) * C;
        colbad[v] = bad ? 0xFFFFFFFFu : 0u;
      }
      uint32_t id[K][PW];
      float4 d[K][PW];
      auto load_row = [&](int u, uint32_t (&ir)[PW], float4 (&dr)[PW]) {
        const int wy = K * bi - (K - 1) + u;
        const bool bad = wy < 0 || wy >= Yw;
        const int rowoff = bad ? 0 : ((u + 1) % K) * K * MMC + (bi - 1 + (u + 1) / K) * mcC;
        const uint32_t rbad = bad ? 0xFFFFFFFFu : 0u;
        const uint8_t* ip = isrc + rowoff;
        const float* dp = dsrc + rowoff;
#pragma unroll
        for (int v = 0; v < PW; ++v) {
          ir[v] = __ldg(reinterpret_cast<const uint32_t*>(ip + coloff[v])) | rbad | colbad[v];
          dr[v] = __ldg(reinterpret_cast<const float4*>(dp + coloff[v]));
        }
      };
#pragma unroll
      for (int u = 0; u < K; ++u) load_row(u, id[u], d[u]);
      float* dst = a.din + (size_t)g * a.gr * a.gc * C + cv * 4;
      const int gcC = a.gc * C;
      int eoff = K * bi * gcC + BW * bj * C;  // 32-bit element offset inside the fragment
#pragma unroll
      for (int ea = 0; ea < K; ++ea, eoff += gcC) {
        const int Y = K * bi + ea;
#pragma unroll
        for (int eb = 0; eb < BW; ++eb) {
          const int X = BW * bj + eb;
          if (Y >= a.gr || X >= a.gc) continue;
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int dy = 0; dy < K; ++dy)
#pragma unroll
            for (int dx = 0; dx < K; ++dx) {
              const int u = ea - dy + K - 1, v = eb - dx + K - 1;  // patch row / column
              const uint32_t x = id[u % K][v] ^ ((uint32_t)(dy * K + dx) * 0x01010101u);
              const float4 w = d[u % K][v];
              if (!(x & 0xFFu)) acc[0] += w.x;
              if (!(x & 0xFF00u)) acc[1] += w.y;
              if (!(x & 0xFF0000u)) acc[2] += w.z;
              if (!(x & 0xFF000000u)) acc[3] += w.w;
            }
          float o[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            bsum[q] += acc[q];
            o[q] = a.round_tf32 ? tf32_rn(acc[q]) : acc[q];
          }
          stv<4>(dst + eoff + eb * C, o);
        }
        if (ea + K < 2 * K - 1) load_row(ea + K, id[(ea + K) % K], d[(ea + K) % K]);  // replaces patch row ea
      }
    }
  }
  write_bias_rows(a, bsum, sub, nsub, cv);
}

// Scatter form of the MPF backward (k = 3 default; premul deltas).  Alg. 4
// read forwards: every window routes its delta to the one conv-output element its argmax names,
// instead of every element testing its k^2 candidate windows (the gathers above spend k^2
// predicated adds per element and channel; this kernel spends one shared-memory add per window).
// Windows are grouped into k x k blocks (block (B, bx) = window rows kB .. kB+k-1, columns
// kbx .. kbx+k-1); a block's targets lie in rows kB .. kB+2k-2 and columns kbx .. kbx+2k-2, so
// blocks of one block row whose bx differ by 2 never share a target.  A CTA owns an output tile
// (rows [Y0, Y1), columns [X0, X1), a slice of CS channels) of one input fragment and walks its
// block rows top to bottom: per block row, the even-bx blocks and then the odd-bx blocks add
// their deltas into a shared-memory ring of 2k accumulator rows (one thread per (block, channel),
// no two threads of a phase on one element, no atomics), then output rows kB .. kB+k-1 are
// complete (no later block row reaches them) and are written out, zeroed and summed into the
// bias partials.  Windows of the block row above the tile and of the block column left of it
// (halo) are processed too, keeping only targets inside the tile, so every element receives
// all its contributions from one CTA in one fixed order: block row, then bx parity, then window
// (u, v) row-major — deterministic and independent of the tiling.  (The gathers sum in (dy, dx)
// order instead; the two agree to fp32 rounding.)
struct ScatterGeo {
  int CS, n_cs, NBX, n_cx, BR, n_bb, T;  // T = threads = (NBX / 2 + 1) * CS: one block per thread and phase
  size_t smem;
  long long units;  // CTAs / n_cs: rows of bias partials
};
constexpr int kScatterRing = 8;  // accumulator ring rows (a power of two >= 2k - 1)

#ifndef MPF_SCATTER_MAXT
#define MPF_SCATTER_MAXT 1024
#endif
template <int K, int CS>
__global__ void __launch_bounds__(MPF_SCATTER_MAXT, 1024 / MPF_SCATTER_MAXT) mpf_bwd_scatter_kernel(MpfBwdArgs a, ScatterGeo s) {
  // ring of kRing accumulator rows (slot = row mod kRing; rows kB .. kB+2k-2 of one block row
  // are distinct slots), each K*NBX + 2K - 1 columns: K columns left of the tile and K - 1
  // right of it catch the halo blocks' out-of-tile targets (never written out)
  extern __shared__ __align__(16) float acc[];
  constexpr int HL = K, kRing = kScatterRing;
  static_assert(2 * K - 1 <= kRing && (kRing & (kRing - 1)) == 0, "ring too small");
  // byte offset of the target of a window with argmax q, relative to its block's column in
  // ring row K*B + u: tab[B mod 8][u][q] (K*B mod 8 depends on B mod 8 only)
  __shared__ int tab[8 * K * K * K];
  const int T = s.T, tid = threadIdx.x;  // blockDim.x == T, a multiple of CS
  const int C = a.C;
  int u_ = blockIdx.x;
  const int cs = u_ % s.n_cs; u_ /= s.n_cs;
  const int cx = u_ % s.n_cx; u_ /= s.n_cx;
  const int bb = u_ % s.n_bb;
  const int g = u_ / s.n_bb;
  const int ch = tid % CS, sub = tid / CS, nsub = T / CS;
  const int TXo = K * s.NBX, RW = TXo + 2 * K - 1, ROW = RW * CS;  // ring row pitch (floats)
  for (int i = tid; i < 8 * K * K * K; i += T) {
    const int bm = i / (K * K * K), u = (i / (K * K)) % K, q = i % (K * K);
    tab[i] = (((K * bm + u + q / K) & (kRing - 1)) * ROW + (q % K) * CS) * (int)sizeof(float);
  }
  const int X0 = TXo * cx, X1 = min(a.gc, X0 + TXo);
  const int Y0 = K * s.BR * bb, Y1 = min(a.gr, Y0 + K * s.BR);
  // block (B, bx) has all its k x k windows iff B < m_r and bx < m_c
  const int bxa = max(0, s.NBX * cx - 1), bxb = min(a.m_c, s.NBX * (cx + 1));
  const int MMC = a.m_r * a.m_c * C, mcC = a.m_c * C;
  const float* dsrc = a.dout + (size_t)g * K * K * MMC + cs * CS + ch;
  const uint8_t* isrc = a.idx + (size_t)g * K * K * MMC + cs * CS + ch;
  for (int i = tid; i < kRing * ROW; i += T) acc[i] = 0.f;
  const int Bs = bb > 0 ? Y0 / K - 1 : 0, Be = (Y1 + K - 1) / K;
  // this thread's block of phase p (bx parity p) in block row B, or -1
  auto block_of = [&](int B, int p) -> int {
    const int bx = bxa + ((p - bxa) & 1) + 2 * sub;
    return (B < a.m_r && B < Be && bx < bxb) ? bx : -1;
  };
  auto load = [&](int B, int bx, uint32_t (&id)[K][K], float (&d)[K][K]) {
    if (bx < 0) return;
    const int o = B * mcC + bx * C;
    const uint8_t* ip = isrc + o;
    const float* dp = dsrc + o;
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int v = 0; v < K; ++v) {
        id[u][v] = __ldg(ip + (u * K + v) * MMC);
        d[u][v] = __ldg(dp + (u * K + v) * MMC);
      }
  };
  auto scatter = [&](int B, int bx, const uint32_t (&id)[K][K], const float (&d)[K][K]) {
    char* base = reinterpret_cast<char*>(acc + (K * bx - X0 + HL) * CS + ch);
    const int* tb = tab + (B & 7) * K * K * K;
#pragma unroll
    for (int u = 0; u < K; ++u)
#pragma unroll
      for (int v = 0; v < K; ++v) {
        float* e = reinterpret_cast<float*>(base + tb[u * K * K + (int)id[u][v]]) + v * CS;
        *e += d[u][v];
      }
  };
  // write-out mapping: 4-channel vectors, thread (column lane, vector) with a fixed vector
  constexpr int CV = CS / 4;
  const int vq = tid % CV, csub = tid / CV, ncsub = T / CV;
  float bsum[4] = {0.f, 0.f, 0.f, 0.f};
  const int W = X1 - X0;
  float* dst = a.din + ((size_t)g * a.gr * a.gc + X0) * C + cs * CS + vq * 4;
  // rows kB .. kB+k-1 are complete after block row B (no later block row reaches them): write
  // out and zero them (the halo block row above the tile only zeroes: its rows belong to the
  // tile above), bias partials
  auto write_out = [&](int B) {
    for (int r = 0; r < K; ++r) {
      const int rr = K * B + r;
      if (rr >= Y1) break;
      float* q = acc + (rr & (kRing - 1)) * ROW + HL * CS + vq * 4;
      int c0 = 0;
      if (rr >= Y0) {
        float* op = dst + ((size_t)rr * a.gc + csub) * C;
        float* qp = q + csub * CS;
        const size_t ostep = (size_t)ncsub * C;
        const int qstep = ncsub * CS;
        for (int col = csub; col < W; col += ncsub, op += ostep, qp += qstep) {
          const float4 v = *reinterpret_cast<float4*>(qp);
          *reinterpret_cast<float4*>(qp) = make_float4(0.f, 0.f, 0.f, 0.f);
          bsum[0] += v.x; bsum[1] += v.y; bsum[2] += v.z; bsum[3] += v.w;
          float4 w = v;
          if (a.round_tf32) { w.x = tf32_rn(v.x); w.y = tf32_rn(v.y); w.z = tf32_rn(v.z); w.w = tf32_rn(v.w); }
          *reinterpret_cast<float4*>(op) = w;
        }
        c0 = W;
      }
      // the columns not written out (halo; the whole row above the tile): zero for reuse
      for (int j = csub; j < RW - c0; j += ncsub) {
        const int col = j < HL ? j - HL : c0 + j - HL;
        *reinterpret_cast<float4*>(q + col * CS) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
  uint32_t idA[K][K], idB[K][K];
  float dA[K][K], dB[K][K];
  int bxA = block_of(Bs, 0), bxB;
  load(Bs, bxA, idA, dA);
  __syncthreads();
  for (int B = Bs; B < Be; ++B) {
    // phase 0 (even bx) from set A while phase 1's windows load into set B; then phase 1 from
    // set B while the next block row's phase 0 loads into set A
    bxB = block_of(B, 1);
    load(B, bxB, idB, dB);
    if (bxA >= 0) scatter(B, bxA, idA, dA);
    __syncthreads();
    bxA = block_of(B + 1, 0);
    load(B + 1, bxA, idA, dA);
    if (bxB >= 0) scatter(B, bxB, idB, dB);
    __syncthreads();
    write_out(B);
    __syncthreads();
  }
  if (a.bias_part == nullptr) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i * T + tid] = bsum[i];  // fixed-order reduction per channel
  __syncthreads();
  if (tid < CS) {
    const int v = tid / 4, i = tid % 4;
    float t = 0.f;
    for (int j = 0; j < ncsub; ++j) t += acc[i * T + j * CV + v];
    a.bias_part[(size_t)(blockIdx.x / s.n_cs) * C + cs * CS + tid] = t;
  }
}

// ----------------------------------------------------------------------------- channel sums
// Generic per-channel partials of a [P][C] tensor (bias gradient of a conv whose delta
// comes from a dgrad, i.e. a conv followed by another conv).
template <int V>
__global__ void __launch_bounds__(256) channel_partial_kernel(const float* __restrict__ dy, long long P, int C,
                                                              long long rows_per_block, float* part) {
  extern __shared__ float s_red[];
  const int cv = threadIdx.x;
  const long long r0 = (long long)blockIdx.x * rows_per_block;
  const long long r1 = min(P, r0 + rows_per_block);
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) acc[v] = 0.f;
  for (long long r = r0 + threadIdx.y; r < r1; r += blockDim.y) {
    const Vec<V> q = ldv<V>(dy + r * C + cv * V);
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] += q.v[v];
  }
#pragma unroll
  for (int v = 0; v < V; ++v) s_red[threadIdx.y * C + cv * V + v] = acc[v];
  __syncthreads();
  if (threadIdx.y == 0) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float t = 0.f;
      for (int q = 0; q < (int)blockDim.y; ++q) t += s_red[q * C + cv * V + v];
      part[(size_t)blockIdx.x * C + cv * V + v] = t;
    }
  }
}

// dst[e] (+)= sum_b part[b][e] (e >= split_at: dst2[e - split_at]), b in [0, nb), fixed order.
// Grid (column chunks of 32, S row segments): thread (column c, row lane r) sums rows
// seg0 + r, seg0 + r + 8, ... of its segment (four interleaved accumulators) with coalesced 128-byte row reads; the 8 lanes
// meet in shared memory (fixed order) and the block writes tmp[s][e].  The last of the S
// blocks of a column chunk (counted in cnt[chunk], reset afterwards) sums tmp[0..S) in order.
__global__ void __launch_bounds__(256) partial_reduce_kernel(const float* __restrict__ part, int nb, int E,
                                                             float* dst, float* dst2, int split_at, float* tmp,
                                                             unsigned* cnt, int S) {
  __shared__ float red[8][33];
  __shared__ bool last;
  const int c = threadIdx.x & 31, r = threadIdx.x >> 5;
  const int e = blockIdx.x * 32 + c;
  const int seg = blockIdx.y;
  const int rows = (nb + S - 1) / S, b0 = seg * rows, b1 = min(nb, b0 + rows);
  float t = 0.f;
  if (e < E) {  // four independent loads in flight per thread; fixed order
    float t1 = 0.f, t2 = 0.f, t3 = 0.f;
    int b = b0 + r;
    for (; b + 24 < b1; b += 32) {
      t += part[(size_t)b * E + e];
      t1 += part[(size_t)(b + 8) * E + e];
      t2 += part[(size_t)(b + 16) * E + e];
      t3 += part[(size_t)(b + 24) * E + e];
    }
    for (; b < b1; b += 8) t += part[(size_t)b * E + e];
    t = (t + t1) + (t2 + t3);
  }
  red[r][c] = t;
  __syncthreads();
  if (r == 0) {
    float v = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) v += red[q][c];
    if (e < E) tmp[(size_t)seg * E + e] = v;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(cnt + blockIdx.x, 1u) == (unsigned)S - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  float u = 0.f;
  if (e < E)
    for (int q = r; q < S; q += 8) u += __ldcg(tmp + (size_t)q * E + e);
  red[r][c] = u;
  __syncthreads();
  if (r == 0 && e < E) {
    float v = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) v += red[q][c];
    if (e < split_at) dst[e] += v;
    else dst2[e - split_at] += v;
  }
  if (threadIdx.x == 0) cnt[blockIdx.x] = 0u;  // ready for the next launch on this stream
}

}  // namespace

cudaError_t launch_mpf_fwd(const MpfArgs& a, cudaStream_t s) {
  if (a.C % 4 == 0) return fwd_dispatch<4>(a, s);
  return fwd_dispatch<1>(a, s);
}

// k = 2, 3: register-blocked gathers
static bool bwd_block2(const MpfBwdArgs& a) {
  return a.premul && (a.k == 2 || a.k == 3) && a.C % 4 == 0 && a.C <= 1024;
}
static long long block2_groups(const MpfBwdArgs& a) {
  const int nsub = 256 / (a.C / 4);
  const int bw = a.k == 2 ? 2 : 3;
  const long long bj_n = (a.gc + bw - 1) / bw, bi_n = (a.gr + a.k - 1) / a.k;
  return (long long)a.n_frag_in * bi_n * ((bj_n + nsub - 1) / nsub);
}
// block rows per band: long bands (up to 32; measured 8 -> 32: 4.6 -> 4.8-5.2 TB/s on cfg4)
// while the grid keeps about two waves of 3 CTAs per SM
static int band2_rows(const MpfBwdArgs& a) {
  const int nsub = 256 / (a.C / 4);
  const long long bj_n = (a.gc + 1) / 2, bi_n = (a.gr + 1) / 2;
  const long long cols = (long long)a.n_frag_in * ((bj_n + nsub - 1) / nsub);
  long long r = cols * bi_n / (148LL * 6);
  if (r > 32) r = 32;
  if (r < 1) r = 1;
  return (int)r;
}
static long long band2_units(const MpfBwdArgs& a) {
  const int nsub = 256 / (a.C / 4), rows = band2_rows(a);
  const long long bj_n = (a.gc + 1) / 2, bi_n = (a.gr + 1) / 2;
  return (long long)a.n_frag_in * ((bi_n + rows - 1) / rows) * ((bj_n + nsub - 1) / nsub);
}
static bool use_band2(const MpfBwdArgs& a) { return a.k == 2 && !a.block_form; }

static int block2_grid(const MpfBwdArgs& a) {
  const long long g = use_band2(a) ? band2_units(a) : block2_groups(a);
  const long long cap = 148LL * 8;  // 8 CTAs of 256 threads per SM
  return (int)(g < cap ? (g < 1 ? 1 : g) : cap);
}
// k = 4 (and k = 2, 3 with C > 1024): the shared-memory tiled gather
static bool bwd_tile(const MpfBwdArgs& a) {
  return a.premul && a.C % 4 == 0 && a.C <= 1024 && a.k >= 2 && a.k <= 4;
}
constexpr int kTileRows = 64;  // conv-output rows per CTA of the tiled kernel (partials per CTA)

// tile shape (rows x cols of conv-output positions per CTA step); one staging buffer
static int tile_nbuf() { return 1; }
// staging budget per CTA (4 CTAs per SM)
static size_t tile_budget() { return 56 * 1024; }
static size_t tile_bytes(int C, int k, int ty, int tx) {
  const int CV = C / 4, CVP = (CV + 3) & ~3, S = tile_cells_padded(ty + k - 1, tx + k - 1);
  return tile_nbuf() * ((size_t)CVP * S * 4 + (size_t)CV * S * 16) + sizeof(float) * (256 / CV) * C;
}

// Largest tile whose staging fits ~56 KB (4 CTAs per SM): measured best per layer on
// cfg4/cfg5 (A/B over 8x8 .. 16x16).
static void tile_shape(const MpfBwdArgs& a, int* ty, int* tx) {
  *ty = 8;
  *tx = 8;
  const int cand[3][2] = {{16, 16}, {8, 16}, {8, 8}};
  for (int i = 0; i < 3; ++i)
    if (tile_bytes(a.C, a.k, cand[i][0], cand[i][1]) <= tile_budget()) {
      *ty = cand[i][0];
      *tx = cand[i][1];
      break;
    }
}

static size_t tile_smem(const MpfBwdArgs& a) {
  int ty, tx;
  tile_shape(a, &ty, &tx);
  return tile_bytes(a.C, a.k, ty, tx);
}

template <int K>
static cudaError_t launch_tile_k(const MpfBwdArgs& a, dim3 grid, dim3 blk, size_t sm, cudaStream_t s) {
  int ty, tx;
  tile_shape(a, &ty, &tx);
  cudaError_t e = cudaSuccess;
#define MPF_TILE_CASE(TY, TX)                                                                                   \
  if (ty == TY && tx == TX) {                                                                                   \
    e = cudaFuncSetAttribute(mpf_bwd_tile_kernel<K, TY, TX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    if (e != cudaSuccess) return e;                                                                             \
    mpf_bwd_tile_kernel<K, TY, TX><<<grid, blk, sm, s>>>(a, kTileRows, tile_nbuf());                                          \
    return cudaGetLastError();                                                                                  \
  }
  MPF_TILE_CASE(8, 8)
  MPF_TILE_CASE(8, 16)
  MPF_TILE_CASE(16, 8)
  MPF_TILE_CASE(16, 16)
#undef MPF_TILE_CASE
  return cudaErrorInvalidValue;
}

static void bwd_geometry(const MpfBwdArgs& a, int V, dim3* grid, dim3* blk) {
  if (bwd_tile(a)) {
    int ty, tx;
    tile_shape(a, &ty, &tx);
    *blk = dim3(256, 1, 1);
    *grid = dim3((a.gc + tx - 1) / tx, (a.gr + kTileRows - 1) / kTileRows, a.n_frag_in < 65535 ? a.n_frag_in : 65535);
    return;
  }
  const int ty = block_dims(a.C, V, blk);
  const int band = kBand;
  *grid = dim3((a.gc + ty - 1) / ty, (a.gr + band - 1) / band, a.n_frag_in < 65535 ? a.n_frag_in : 65535);
}

// k = 3 (premul, C a multiple of 16, 24 or 32) under MPF_FLAG_MPF_BWD_SCATTER: the scatter
static bool scatter_geo(const MpfBwdArgs& a, ScatterGeo* s) {
  if (!(a.k == 3 && a.premul && a.scatter_form)) return false;
  const int K = a.k, C = a.C;
  // channel slice: 32, 24 or 16 channels (compile-time in the kernel)
  int CS = 0;
  if (C % 32 == 0) CS = 32;
  else if (C % 24 == 0) CS = 24;
  else if (C % 16 == 0) CS = 16;
  else return false;
  s->CS = CS;
  s->n_cs = C / CS;
  // widest tile of NBX blocks whose ring fits ~64 KB (three CTAs per SM) within 1024 threads
#ifndef MPF_SCATTER_BUDGET_KB
#define MPF_SCATTER_BUDGET_KB 32
#endif
  const size_t budget = MPF_SCATTER_BUDGET_KB * 1024 + 512;
  int nbx_max = (int)((budget / ((size_t)kScatterRing * CS * sizeof(float)) - (2 * K - 1)) / K);
  while (nbx_max > 1 && (nbx_max / 2 + 1) * CS > MPF_SCATTER_MAXT) --nbx_max;
  if (nbx_max < 1 || (nbx_max / 2 + 1) * CS > MPF_SCATTER_MAXT) return false;
  const int blk_cols = (a.gc + K - 1) / K, blk_rows = (a.gr + K - 1) / K;
  s->n_cx = (blk_cols + nbx_max - 1) / nbx_max;
  s->NBX = (blk_cols + s->n_cx - 1) / s->n_cx;
  s->T = (s->NBX / 2 + 1) * CS;  // blocks per phase <= NBX / 2 + 1 (the halo block included)
  const long long per_row = (long long)a.n_frag_in * s->n_cx * s->n_cs;
  long long br = (blk_rows * per_row + 148LL * 9 - 1) / (148LL * 9);  // about three waves of 3 CTAs/SM
  if (br < 4) br = 4;
  if (br > blk_rows) br = blk_rows;
  s->n_bb = (int)((blk_rows + br - 1) / br);
  s->BR = (blk_rows + s->n_bb - 1) / s->n_bb;
  s->smem = sizeof(float) * std::max((size_t)kScatterRing * (K * s->NBX + 2 * K - 1) * CS, (size_t)4 * s->T);
  s->units = (long long)a.n_frag_in * s->n_bb * s->n_cx;
  return true;
}

long long mpf_bwd_partials(const MpfBwdArgs& a) {
  ScatterGeo sg;
  if (scatter_geo(a, &sg)) return sg.units;
  if (bwd_block2(a)) return (long long)block2_grid(a) * (a.C / 4 <= 32 ? 8 : 256 / (a.C / 4));
  dim3 g, b;
  bwd_geometry(a, a.C % 4 == 0 ? 4 : 1, &g, &b);
  return (long long)g.x * g.y * g.z;
}

cudaError_t launch_mpf_bwd(const MpfBwdArgs& a, cudaStream_t s) {
  ScatterGeo sg;
  if (scatter_geo(a, &sg)) {
    if (sg.units * sg.n_cs > 0x7fffffffLL) return cudaErrorInvalidValue;
    auto kern = sg.CS == 32 ? mpf_bwd_scatter_kernel<3, 32>
                : sg.CS == 24 ? mpf_bwd_scatter_kernel<3, 24> : mpf_bwd_scatter_kernel<3, 16>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sg.smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)(sg.units * sg.n_cs), sg.T, sg.smem, s>>>(a, sg);
    return cudaGetLastError();
  }
  if (bwd_block2(a)) {
    const size_t smem = 0;
    if (use_band2(a)) mpf_bwd_band2_kernel<<<block2_grid(a), 256, smem, s>>>(a, band2_units(a), band2_rows(a));
    else if (a.k == 2) mpf_bwd_block2_kernel<<<block2_grid(a), 256, smem, s>>>(a, block2_groups(a));
    else {
      if (block2_groups(a) > 0x7fffffffLL) return cudaErrorInvalidValue;
      mpf_bwd_k3_kernel<<<block2_grid(a), 256, smem, s>>>(a, (int)block2_groups(a));
    }
    return cudaGetLastError();
  }
  const int V = a.C % 4 == 0 ? 4 : 1;
  dim3 grid, blk;
  bwd_geometry(a, V, &grid, &blk);
  if (bwd_tile(a)) {
    const size_t sm = tile_smem(a);
    if (a.k == 2) return launch_tile_k<2>(a, grid, blk, sm, s);
    if (a.k == 3) return launch_tile_k<3>(a, grid, blk, sm, s);
    return launch_tile_k<4>(a, grid, blk, sm, s);
  }
  const size_t smem = sizeof(float) * blk.y * a.C;
  if (V == 4)
    mpf_bwd_kernel<4><<<grid, blk, smem, s>>>(a);
  else
    mpf_bwd_kernel<1><<<grid, blk, smem, s>>>(a);
  return cudaGetLastError();
}

long long channel_partials(long long P) {
  long long nb = (P + 4095) / 4096;
  if (nb > 148 * 8) nb = 148 * 8;
  if (nb < 1) nb = 1;
  return nb;
}

cudaError_t launch_channel_partial(const float* dy, long long P, int C, float* part, cudaStream_t s) {
  const long long nb = channel_partials(P);
  const long long rows = (P + nb - 1) / nb;
  const int V = C % 4 == 0 ? 4 : 1;
  dim3 blk;
  block_dims(C, V, &blk);
  const size_t smem = sizeof(float) * blk.y * C;
  if (V == 4)
    channel_partial_kernel<4><<<(unsigned)nb, blk, smem, s>>>(dy, P, C, rows, part);
  else
    channel_partial_kernel<1><<<(unsigned)nb, blk, smem, s>>>(dy, P, C, rows, part);
  return cudaGetLastError();
}

cudaError_t launch_partial_reduce(const float* part, int nb, int E, float* dst, float* dst2, int split_at,
                                  const ReduceScratch& rs, cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  int S = (nb + 63) / 64;  // >= 8 rows per thread; the last block then sums S / 8 per thread
  if (S > kReduceSegments) S = kReduceSegments;
  if (S < 1) S = 1;
  const int chunks = (E + 31) / 32;
  if (chunks > rs.n_cnt || (size_t)S * E > rs.tmp_floats) return cudaErrorInvalidValue;
  partial_reduce_kernel<<<dim3(chunks, S), 256, 0, s>>>(part, nb, E, dst, dst2, split_at, rs.tmp, rs.cnt, S);
  return cudaGetLastError();
}

}  // namespace mpf
