// head_mma.cu — the training softmax head (last FC + per-pixel softmax + class-weighted MCCE +
// dL/dx_hat, and the back-propagation through that FC: "first dL/dx_hat",
// 197 MCCE per pixel, 252 per-class weights; readings R8, R9, R15) with its three small
// contractions on the warp-level tensor cores (mma.sync m16n8k8, TF32 operands, fp32
// accumulate), in one pass over the last hidden activation h:
//
//   GEMM1  z[pos][c]    = sum_ch h[pos][ch] W_L[c][ch]        (+ b_L; softmax; dz)
//   GEMM3  dW_L[c][ch] += sum_pos dz[pos][c] h[pos][ch]        (Alg. 2: sum over all fragments)
//   GEMM2  dh[pos][ch]  = (sum_c dz[pos][c] W_L[c][ch]) act'(h[pos][ch])
//
// with db_L = sum dz and db_prev = sum dh.  Every product is split 3xTF32 (a_hi b_hi +
// a_hi b_lo + a_lo b_hi, x_lo = x - tf32(x)), so the head keeps fp32-level accuracy (its
// FMA form was exact fp32).  The FMA form (head.cu) needs ~3000 FMAs + ~200 other warp
// instructions per position and ran instruction-bound at ~53 % of HBM; here the MMAs take
// ~900 tensor instructions per 64-position tile and the kernel streams h in / dh out.
//
// Schedule (persistent CTAs, one per SM, 8 warps): tiles of 64 positions of one image.  A
// tile of h arrives by TMA as ceil(Ch/32) SWIZZLE_128B boxes [64 positions][32 channels]
// (3-D map [n][per_img][Ch]: rows past the image end and channels past Ch read as zeros and
// are clipped on store), three tiles in flight.  Per tile: labels -> GEMM1 (warp = 16
// positions x half of K, partial logits combined in shared memory) -> softmax / loss / dz
// (warps 0-3) -> GEMM3 (warp = two 16-channel tiles, accumulators live across tiles) ->
// GEMM2 + act' + TF32 rounding written IN PLACE over the h tile -> TMA store of dh.  All
// sums have a fixed order (deterministic; loss and bias partials as in head.cu).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "conv_tc.h"
#include "head_common.cuh"
#include "mpf_internal.h"
#include "numerics.cuh"
#include "tc_ptx.cuh"

namespace mpf {

namespace {

constexpr int kMT = 64;          // positions per tile
constexpr int kMThr = 512;       // 16 warps
constexpr int kMaxStages = 6;    // h tiles in the ring (stages - 1 loads in flight)
constexpr int kBoxBytes = kMT * 128;  // one [64 x 32 fp32] SW128 box
constexpr int kWS = 260;         // row stride of the split W_L copies (conflict-free fragment reads)

struct HeadMmaParams {
  int C, Ch, nchunk, nkt, nmt3;  // classes, channels, 32-ch boxes, 8-ch K/N tiles, 16-ch M tiles
  int tpi;                       // tiles per image
  long long total;               // tiles
  long long per_img;             // positions per image (fragment-major, padded grid)
  const float* wL;               // [C][Ch]
  const float* bL;               // [C]
  const uint8_t* lab_frag;       // [n][per_img] (launch_label_frag)
  const int* nlab;               // [n]
  float cw[16];
  int act;                       // activation of h
  int round;                     // TF32-round dh (operand of the FC1 dgrad / wgrad MMAs)
  float* loss_part;              // [n][tpi][8]
  float* part;                   // [grid][C*Ch + C + Ch]
  float* dh;                     // [n][per_img][Ch]
  int n_stages;                  // h tiles in the ring
};

// byte offset of (row r, channel c) inside a tile: box c/32, TMA SWIZZLE_128B pattern
__device__ __forceinline__ uint32_t swz(int r, int c) {
  return (uint32_t)((c >> 5) * kBoxBytes + r * 128 + ((((c & 31) >> 2) ^ (r & 7)) << 4) + ((c & 3) << 2));
}

// 3xTF32 split: x = hi + lo, hi the TF32 rounding of x (one F2FP), lo = x - hi exactly in
// fp32 (the MMA reads only its top 19 bits: the dropped part is ~2^-22 |x|).  Non-finite
// inputs give non-finite products (NaN stays NaN; Inf becomes MAX_TF32 + Inf in lo).
__device__ __forceinline__ void split3(float x, uint32_t& hi, uint32_t& lo) {
  const float h = tf32_rn_sat(x);
  hi = __float_as_uint(h);
  lo = __float_as_uint(x - h);
}

__device__ __forceinline__ float act_der_m(int act, float y) {
  if (act == MPF_TANH) return fmaf(-y, y, 1.f);
  if (act == MPF_LOGISTIC) return y * (1.f - y);
  return 1.f;
}

template <bool TANH>
__global__ void __launch_bounds__(kMThr, 1) head_mma_kernel(const __grid_constant__ CUtensorMap tmH, HeadMmaParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t s0 = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* g0 = smem_raw + (s0 - ptx::smem_u32(smem_raw));  // generic address of s0
  const uint32_t stage_bytes = (uint32_t)p.nchunk * kBoxBytes;
  // [h stages | W_L hi [8][kWS] | W_L lo [8][kWS] | z partials [4 K-quarters][64][8] | dz [64][8] |
  //  lab [64] | db_L partials [64][8] | cw [16] | nlab | bars]
  const int S = p.n_stages;
  uint32_t* s_whi = reinterpret_cast<uint32_t*>(g0 + S * stage_bytes);
  uint32_t* s_wlo = s_whi + 8 * kWS;
  float* s_zp = reinterpret_cast<float*>(s_wlo + 8 * kWS);
  float* s_dz = s_zp + 4 * kMT * 8;
  int* s_lab = reinterpret_cast<int*>(s_dz + kMT * 8);
  float* s_dbl = reinterpret_cast<float*>(s_lab + kMT);
  float* s_cw = s_dbl + kMT * 8;
  int* s_nl = reinterpret_cast<int*>(s_cw + 16);
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_nl + 2);
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int g = lane >> 2, t = lane & 3;
  const int C = p.C, Ch = p.Ch;

  for (int e = tid; e < 8 * 256; e += kMThr) {
    const int c = e >> 8, ch = e & 255;
    uint32_t hi, lo;
    split3((c < C && ch < Ch) ? p.wL[c * Ch + ch] : 0.f, hi, lo);
    s_whi[c * kWS + ch] = hi;
    s_wlo[c * kWS + ch] = lo;
  }
  if (tid < 16) s_cw[tid] = p.cw[tid];
  if (tid == 0) {
    ptx::prefetch_tmap(&tmH);
    for (int s = 0; s < S; ++s) ptx::mbar_init(ptx::smem_u32(&bars[s]), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](long long tile, int st) {
    const int img = (int)(tile / p.tpi), p0 = (int)(tile % p.tpi) * kMT;
    const uint32_t bar = ptx::smem_u32(&bars[st]);
    ptx::mbar_arrive_expect_tx(bar, stage_bytes);
    for (int c = 0; c < p.nchunk; ++c) ptx::tma_load_3d(s0 + st * stage_bytes + c * kBoxBytes, &tmH, bar, 32 * c, p0, img);
  };
  // label of position tid of a tile (threads 0-63) and the image's labelled-pixel count
  // (thread 64), issued one tile ahead and kept in a register
  auto fetch = [&](long long tile) -> int {
    if (tile >= p.total) return kLabBeyond;
    const int img = (int)(tile / p.tpi);
    if (tid == kMT) return __ldg(p.nlab + img);
    const long long pos = (long long)(tile % p.tpi) * kMT + tid;
    return pos < p.per_img ? (int)__ldg(p.lab_frag + (long long)img * p.per_img + pos) : kLabBeyond;
  };
  if (tid == 0)
    for (int s = 0; s + 1 < S; ++s) {  // S - 1 tiles in flight
      const long long tile = blockIdx.x + (long long)s * gridDim.x;
      if (tile < p.total) issue(tile, s);
    }
  int pre = tid <= kMT ? fetch(blockIdx.x) : 0;

  // GEMM2's B fragments (constant): N-tiles nt = warp + 16 j; b0 = W[t][8 nt + g], b1 = W[t + 4][8 nt + g]
  uint32_t bW[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int ch = 8 * (warp + 16 * j) + g;
    bW[j][0] = s_whi[t * kWS + ch];
    bW[j][1] = s_whi[(t + 4) * kWS + ch];
    bW[j][2] = s_wlo[t * kWS + ch];
    bW[j][3] = s_wlo[(t + 4) * kWS + ch];
  }
  // accumulators living across tiles: dW_L^T of channel tile `warp`, db_prev of the warp's two
  // 8-channel tiles, db_L (threads 0-63: eight classes)
  float accW[4] = {0.f, 0.f, 0.f, 0.f}, accP[2][2] = {{0.f, 0.f}, {0.f, 0.f}}, accL[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) accL[c] = 0.f;
  float blc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) blc[c] = c < C ? p.bL[c] : 0.f;
  const int mt = warp & 3, kq = warp >> 2;  // GEMM1: M tile, K quarter

  int it = 0;
  for (long long tile = blockIdx.x; tile < p.total; tile += gridDim.x, ++it) {
    const int st = it % S;
    const int img = (int)(tile / p.tpi), tt = (int)(tile % p.tpi), p0 = tt * kMT;
    if (tid < kMT) s_lab[tid] = pre == kLabFragPad ? kLabPad : pre;
    if (tid == kMT) s_nl[0] = pre;
    if (tid <= kMT) pre = fetch(tile + gridDim.x);  // in flight during this tile
    ptx::mbar_wait(ptx::smem_u32(&bars[st]), (uint32_t)((it / S) & 1));
    __syncthreads();  // labels and h visible; the previous tile's stage is no longer read
    if (tid == 0) {  // refill that stage with the tile S - 1 ahead
      const long long nt = tile + (long long)(S - 1) * gridDim.x;
      if (nt < p.total) issue(nt, (it + S - 1) % S);
    }
    const uint8_t* hb = g0 + st * stage_bytes;

    // ------------------------------------------------ GEMM1: partial logits (M tile x K quarter)
    {
      float za[4] = {0.f, 0.f, 0.f, 0.f};
      const int r0 = 16 * mt + g, r1 = r0 + 8;
      for (int ks = kq; ks < p.nkt; ks += 4) {
        const int k0 = 8 * ks;
        uint32_t ah[4], al[4];
        split3(*reinterpret_cast<const float*>(hb + swz(r0, k0 + t)), ah[0], al[0]);
        split3(*reinterpret_cast<const float*>(hb + swz(r1, k0 + t)), ah[1], al[1]);
        split3(*reinterpret_cast<const float*>(hb + swz(r0, k0 + t + 4)), ah[2], al[2]);
        split3(*reinterpret_cast<const float*>(hb + swz(r1, k0 + t + 4)), ah[3], al[3]);
        const uint32_t bh0 = s_whi[g * kWS + k0 + t], bh1 = s_whi[g * kWS + k0 + t + 4];
        const uint32_t bo0 = s_wlo[g * kWS + k0 + t], bo1 = s_wlo[g * kWS + k0 + t + 4];
        ptx::mma_m16n8k8_tf32(za, al, bh0, bh1);
        ptx::mma_m16n8k8_tf32(za, ah, bo0, bo1);
        ptx::mma_m16n8k8_tf32(za, ah, bh0, bh1);
      }
      float* zp = s_zp + kq * kMT * 8;
      *reinterpret_cast<float2*>(zp + r0 * 8 + 2 * t) = make_float2(za[0], za[1]);
      *reinterpret_cast<float2*>(zp + r1 * 8 + 2 * t) = make_float2(za[2], za[3]);
    }
    __syncthreads();

    // ------------------------------------------------ softmax, loss, dz (thread = position)
    float lossv = 0.f;
    if (tid < kMT) {
      float z[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) z[c] = blc[c];
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // fixed order over the K quarters
        const float4 a = *reinterpret_cast<const float4*>(s_zp + (q * kMT + tid) * 8);
        const float4 b = *reinterpret_cast<const float4*>(s_zp + (q * kMT + tid) * 8 + 4);
        z[0] += a.x; z[1] += a.y; z[2] += a.z; z[3] += a.w;
        z[4] += b.x; z[5] += b.y; z[6] += b.z; z[7] += b.w;
      }
      float m = -INFINITY;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < C) m = fmaxf(m, z[c]);
      float ex[8], se = 0.f;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        ex[c] = c < C ? expf(z[c] - m) : 0.f;
        se += ex[c];
      }
      const float lse = m + logf(se);
      const int lab = s_lab[tid];
      float d[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) d[c] = 0.f;
      if (lab >= 0 && lab < C) {
        const int nl = s_nl[0];
        const float wt = s_cw[lab];
        const float inv = nl > 0 ? wt / (float)nl : 0.f;
        const float rs = 1.f / se;
        float zt = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c < C) d[c] = inv * (ex[c] * rs - (c == lab ? 1.f : 0.f));
          if (c == lab) zt = z[c];
        }
        lossv = wt * (lse - zt);
      }
      *reinterpret_cast<float4*>(s_dz + tid * 8) = make_float4(d[0], d[1], d[2], d[3]);
      *reinterpret_cast<float4*>(s_dz + tid * 8 + 4) = make_float4(d[4], d[5], d[6], d[7]);
#pragma unroll
      for (int c = 0; c < 8; ++c) accL[c] += d[c];
    }
    if (warp < kMThr / 32 / 2) {  // loss partials: warps 0-1 hold the positions, 2-7 write zeros
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lossv += __shfl_xor_sync(0xffffffffu, lossv, o);
      if (lane == 0) p.loss_part[((long long)img * p.tpi + tt) * 8 + warp] = lossv;
    }
    __syncthreads();  // dz complete

    // ------------------------------------------------ GEMM3 (dW_L^T += h^T dz) and GEMM2 (dh)
    // interleaved: step kst does one K step of GEMM3 for the warp's channel tile and one of
    // the warp's (N-tile, M-tile) units of GEMM2, so independent MMA chains overlap.  dh goes
    // straight to global memory (each fragment row is one full 32-byte sector).
    float* dh_img = p.dh + ((long long)img * p.per_img + p0) * Ch;
    const int nrow = (int)min((long long)kMT, p.per_img - p0);
#pragma unroll
    for (int kst = 0; kst < kMT / 8; ++kst) {
      if (warp < p.nmt3) {  // GEMM3, positions 8 kst .. 8 kst + 7 (warp-uniform)
        const int k0 = 8 * kst;
        uint32_t bh0, bo0, bh1, bo1;
        split3(s_dz[(k0 + t) * 8 + g], bh0, bo0);
        split3(s_dz[(k0 + t + 4) * 8 + g], bh1, bo1);
        const int c0 = 16 * warp + g, c1 = c0 + 8;
        uint32_t ah[4], al[4];
        split3(*reinterpret_cast<const float*>(hb + swz(k0 + t, c0)), ah[0], al[0]);
        split3(*reinterpret_cast<const float*>(hb + swz(k0 + t, c1)), ah[1], al[1]);
        split3(*reinterpret_cast<const float*>(hb + swz(k0 + t + 4, c0)), ah[2], al[2]);
        split3(*reinterpret_cast<const float*>(hb + swz(k0 + t + 4, c1)), ah[3], al[3]);
        ptx::mma_m16n8k8_tf32(accW, al, bh0, bh1);
        ptx::mma_m16n8k8_tf32(accW, ah, bo0, bo1);
        ptx::mma_m16n8k8_tf32(accW, ah, bh0, bh1);
      }
      {  // GEMM2 unit (j, m) = (kst / 4, kst % 4)
        const int j = kst >> 2, m = kst & 3;
        const int nt = warp + 16 * j;
        if (nt < p.nkt) {  // warp-uniform
          const int q0 = 16 * m + g, q1 = q0 + 8;
          uint32_t ah[4], al[4];
          split3(s_dz[q0 * 8 + t], ah[0], al[0]);
          split3(s_dz[q1 * 8 + t], ah[1], al[1]);
          split3(s_dz[q0 * 8 + t + 4], ah[2], al[2]);
          split3(s_dz[q1 * 8 + t + 4], ah[3], al[3]);
          float d[4] = {0.f, 0.f, 0.f, 0.f};
          ptx::mma_m16n8k8_tf32(d, al, bW[j][0], bW[j][1]);
          ptx::mma_m16n8k8_tf32(d, ah, bW[j][2], bW[j][3]);
          ptx::mma_m16n8k8_tf32(d, ah, bW[j][0], bW[j][1]);
          const int ch = 8 * nt + 2 * t;
          const float2 hv0 = *reinterpret_cast<const float2*>(hb + swz(q0, ch));
          const float2 hv1 = *reinterpret_cast<const float2*>(hb + swz(q1, ch));
          const int la = s_lab[q0], lb = s_lab[q1];
          const bool a0 = la >= 0 && la < C, a1 = lb >= 0 && lb < C;
          float e[4];
          e[0] = a0 ? d[0] * (TANH ? fmaf(-hv0.x, hv0.x, 1.f) : act_der_m(p.act, hv0.x)) : 0.f;
          e[1] = a0 ? d[1] * (TANH ? fmaf(-hv0.y, hv0.y, 1.f) : act_der_m(p.act, hv0.y)) : 0.f;
          e[2] = a1 ? d[2] * (TANH ? fmaf(-hv1.x, hv1.x, 1.f) : act_der_m(p.act, hv1.x)) : 0.f;
          e[3] = a1 ? d[3] * (TANH ? fmaf(-hv1.y, hv1.y, 1.f) : act_der_m(p.act, hv1.y)) : 0.f;
          accP[j][0] += e[0] + e[2];
          accP[j][1] += e[1] + e[3];
          if (p.round) {
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] = tf32_rn_sat(e[u]);
          }
          if (ch < Ch) {
            if (q0 < nrow) *reinterpret_cast<float2*>(dh_img + (long long)q0 * Ch + ch) = make_float2(e[0], e[1]);
            if (q1 < nrow) *reinterpret_cast<float2*>(dh_img + (long long)q1 * Ch + ch) = make_float2(e[2], e[3]);
          }
        }
      }
    }
  }

  // ------------------------------------------------------------------ block partials
  const int E = C * Ch + C + Ch;
  float* out = p.part + (size_t)blockIdx.x * E;
  if (warp < p.nmt3) {  // dW_L[c][ch]: each (class, channel) is owned by exactly one thread
    const int c0 = 16 * warp + g, c1 = c0 + 8, ca = 2 * t, cb = 2 * t + 1;
    if (ca < C && c0 < Ch) out[ca * Ch + c0] = accW[0];
    if (cb < C && c0 < Ch) out[cb * Ch + c0] = accW[1];
    if (ca < C && c1 < Ch) out[ca * Ch + c1] = accW[2];
    if (cb < C && c1 < Ch) out[cb * Ch + c1] = accW[3];
  }
  // db_prev[ch]: the 8 lanes of equal t hold channels 8 nt + 2t, + 1 (fixed-order butterfly)
#pragma unroll
  for (int j = 0; j < 2; ++j) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      float v = accP[j][u];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      const int nt = warp + 16 * j, ch = 8 * nt + 2 * t + u;
      if (g == 0 && nt < p.nkt && ch < Ch) out[C * Ch + C + ch] = v;
    }
  }
  // db_L[c]: threads 0-63 hold the eight classes of their positions; fixed-order sum
  if (tid < kMT) {
#pragma unroll
    for (int c = 0; c < 8; ++c) s_dbl[tid * 8 + c] = accL[c];
  }
  __syncthreads();
  if (tid < C) {
    float v = 0.f;
    for (int q = 0; q < kMT; ++q) v += s_dbl[q * 8 + tid];
    out[C * Ch + tid] = v;
  }
}

size_t head_mma_fixed_smem() {
  return 1024 + 2 * 8 * kWS * 4 + 4 * kMT * 8 * 4 + kMT * 8 * 4 + kMT * 4 + kMT * 8 * 4 + 16 * 4 + 8 + kMaxStages * 8 +
         64;
}
// as many h stages as fit (at most kMaxStages): S - 1 tiles of loads in flight per SM
int head_mma_stages(int Ch) {
  const size_t stage = (size_t)((Ch + 31) / 32) * kBoxBytes;
  int s = (int)((225 * 1024 - head_mma_fixed_smem()) / stage);
  return s > kMaxStages ? kMaxStages : s;
}

}  // namespace

bool head_mma_ok(int C, int Ch, bool train) {
  return train && C >= 2 && C <= 8 && Ch >= 4 && Ch <= 256 && Ch % 4 == 0 && head_mma_stages(Ch) >= 3;
}

int head_mma_grid(long long per_img, int n) {
  const long long tiles = (long long)n * ((per_img + kMT - 1) / kMT);
  const long long g = tiles < 148 ? tiles : 148;
  return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_head_mma(const HeadArgs& a, cudaStream_t s) {
  HeadMmaParams p{};
  p.C = a.C;
  p.Ch = a.Ch;
  p.nchunk = (a.Ch + 31) / 32;
  p.nkt = (a.Ch + 7) / 8;
  p.nmt3 = (a.Ch + 15) / 16;
  p.per_img = (long long)a.F * a.gr * a.gc;
  p.tpi = (int)((p.per_img + kMT - 1) / kMT);
  p.total = (long long)a.n * p.tpi;
  p.wL = a.w;
  p.bL = a.b;
  p.lab_frag = a.lab_frag;
  p.nlab = a.nlab;
  for (int c = 0; c < 16; ++c) p.cw[c] = a.cw[c];
  p.act = a.hidden_act;
  p.round = a.round_tf32;
  p.loss_part = a.loss_part;
  p.part = a.part;
  p.dh = a.dh;
  p.n_stages = head_mma_stages(a.Ch);
  if (p.n_stages < 3) return cudaErrorInvalidConfiguration;
  if (a.tiles_per_img != p.tpi || !a.lab_frag) return cudaErrorInvalidValue;
  CUtensorMap H;
  const uint64_t dims[3] = {(uint64_t)a.Ch, (uint64_t)p.per_img, (uint64_t)a.n};
  const uint64_t strides[2] = {(uint64_t)a.Ch * 4, (uint64_t)p.per_img * a.Ch * 4};
  const uint32_t box[3] = {32, kMT, 1};
  cudaError_t e = make_tmap_f32(&H, a.h, 3, dims, strides, box, true);
  if (e != cudaSuccess) return e;
  const size_t smem = head_mma_fixed_smem() + (size_t)p.n_stages * p.nchunk * kBoxBytes;
  const int grid = a.n_blocks;
  auto kern = a.hidden_act == MPF_TANH ? head_mma_kernel<true> : head_mma_kernel<false>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kMThr, smem, s>>>(H, p);
  return cudaGetLastError();
}

}  // namespace mpf
