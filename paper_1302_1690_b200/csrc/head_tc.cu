// head_tc.cu — the softmax head's training pass (readings R8,
// R9, R15) on the tensor cores.  Same contract as head_kernel (head.cu): per position p
//     z = W_L h + b_L,  p = softmax(z),  loss += w_t (lse - z_t)
//     dz = w_t (p - onehot_t) / n_lab(img)
//     dh = (W_L^T dz) * act'(h)                   -> written, TF32-rounded (next consumers)
//     dW_L += dz h^T,  db_L += dz,  db_prev += dh  (per-CTA partials, fixed-order reduction)
// with the two products that touch every channel as tcgen05 MMAs:
//   GEMM1  Z[pos][c]    = H[pos][:] . W_L[c][:]      M = 128 positions, N = 16 classes,
//          K = Ch in 32-channel TMA chunks (SW128, K-major); W_L split hi + lo (two
//          TF32 MMAs per step: h is already TF32, so Z is exact to fp32 rounding).
//   GEMM2  dhT[ch][pos] = W_L^T[ch][:] . dz[pos][:]   M = 128 channels (2 blocks, Ch <= 256),
//          N = 128 positions, K = 8 classes (SW32, K-major); 3xTF32 (hi.hi + hi.lo + lo.hi).
// The transposed GEMM2 puts one channel per TMEM lane, so the epilogue thread of channel
// ch walks the tile's positions: act'(h) (h re-read from L2, coalesced over channels),
// the TF32 rounding, a coalesced store of dh, and the dW_L / db_prev sums in registers
// (dW_L = dz h^T stays on the FMA pipes: 5 FMAs per element against a broadcast dz row).
//
// Roles (persistent, one CTA per SM, 10 warps): warp 0 TMA producer (ring of H chunks),
// warp 1 MMA issuer, warps 2..17 epilogue (2..5 also run the per-position softmax).
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "conv_tc.h"
#include "head_common.cuh"
#include "mpf_internal.h"
#include "tc_ptx.cuh"

namespace mpf {

namespace {

constexpr int kHT = 64;                   // positions per tile
constexpr int kHS = 22;                   // ring stages (one 32-channel chunk of a tile each)
constexpr int kHChunk = kHT * 128;        // bytes per chunk: 64 rows x 128 B
constexpr int kHDh = 16;                  // dh warps (4 lane quarters x 4 slots)
constexpr int kHSm = 4;                   // softmax warps
constexpr int kHThreads = 64 + 32 * (kHDh + kHSm);
constexpr int kHMaxCh = 256;

// TF32 rounding (nearest-even, finite-saturating: one F2FP instruction on sm_100a; the guarded
// cvt.rna form takes four) of an MMA operand
__device__ __forceinline__ float tf32_rna_h(float x) {
  uint32_t r;
  asm("cvt.rn.satfinite.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// K-major, 32-byte swizzle (rows of 32 B = 8 tf32, 8-row groups 256 B apart)
__device__ __forceinline__ uint64_t sdesc_k_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256u >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;  // SWIZZLE_32B
  return d;
}
// byte offset of element (row r, k) in a K-major SW32 tile (8 fp32 per row)
__device__ __forceinline__ uint32_t sw32_off(int r, int k) {
  return (uint32_t)(r * 32 + ((((k >> 2) ^ (r >> 2)) & 1) << 4) + (k & 3) * 4);
}
// byte offset of element (row r, k < 32) in a K-major SW128 chunk (32 fp32 per row)
__device__ __forceinline__ uint32_t sw128_off(int r, int k) {
  return (uint32_t)(r * 128 + ((((k >> 2) ^ r) & 7) << 4) + (k & 3) * 4);
}

struct HtcLayout {  // shared-memory offsets from the 1024-aligned base
  uint32_t ring, w1, w2, dl, dlp, red, bar;
};
__host__ __device__ inline HtcLayout htc_layout(int n_chunks) {
  HtcLayout L;
  L.ring = 0;
  L.w1 = L.ring + kHS * kHChunk;              // [hi|lo][chunk][16 rows][128 B]
  L.w2 = L.w1 + n_chunks * 16 * 128;          // [chunk][16 rows][128 B] (TF32-rounded W_L)
  L.dl = L.w2 + 2 * 2 * 128 * 32;             // [buf][hi|lo][64 rows][32 B]
  L.dlp = L.dl + 2 * 2 * kHT * 32;            // [buf][64][8] fp32, plain
  L.red = L.dlp + 2 * kHT * 8 * 4;            // [4 warps][8] fp32 (db_L) + [16] bias
  L.bar = L.red + (4 * 8 + 16) * 4;
  L.bar = (L.bar + 7) & ~7u;
  return L;
}
// full/empty[kHS], zfull/zempty[2], dlfull/dlempty[2], dhfull/dhempty[2], tmem slot
constexpr int kHBars = 2 * kHS + 6 * 2 + 1;

// mbarrier wait that adds its duration to prof[slot] when profiling (MPF_HEAD_PROF=1)
__device__ __forceinline__ void pwait(uint32_t bar, uint32_t parity, unsigned long long* prof, int slot) {
  if (!prof) {
    ptx::mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  ptx::mbar_wait(bar, parity);
  if ((threadIdx.x & 31) == 0) atomicAdd(prof + slot, (unsigned long long)(clock64() - t0));
}

// Schedule (i = this CTA's i-th tile of 64 positions, b = i & 1):
//   producer  H(i) chunks -> ring (a slot is free once GEMM1 and the dh warps are done)
//   MMA       GEMM1(i+1) -> Z[b^1] (M = 64) ; GEMM2(i) -> dhT[b] (M = 128 channels, N = 64)
//   softmax   Z[b] -> dz(i) into dl[b] / dlp[b]        (runs one tile ahead of dh)
//   dh        dhT[b] + h (from the ring) -> dh, dW_L, db_prev
// M = 64 accumulators occupy lanes 0..15 of each 32-lane TMEM sub-partition: row r of Z
// is lane 32 (r / 16) + r % 16.
template <int NC>  // classes rounded up to a kernel variant (dz FMAs per element)
__global__ void __launch_bounds__(kHThreads, 1)
    head_tc_kernel(const __grid_constant__ CUtensorMap tmH, HeadArgs a, int tiles_per_img64, int n_chunks,
                   unsigned long long* prof) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (sbase - ptx::smem_u32(smem_raw));
  const HtcLayout L = htc_layout(n_chunks);
  const uint32_t bFull = sbase + L.bar, bEmpty = bFull + 8 * kHS, bZfull = bEmpty + 8 * kHS, bZempty = bZfull + 16,
                 bDlfull = bZempty + 16, bDlempty = bDlfull + 16, bDhfull = bDlempty + 16, bDhempty = bDhfull + 16,
                 sTmemSlot = bDhempty + 16;
  float* s_red = reinterpret_cast<float*>(gbase + L.red);
  float* s_b = s_red + 32;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const int C = a.C, Ch = a.Ch;
  const long long per_img = (long long)a.F * a.gr * a.gc;
  const int frag_sz = a.gr * a.gc;
  const long long total = (long long)a.n * tiles_per_img64;
  const int n_my = blockIdx.x < total ? (int)((total - 1 - blockIdx.x) / gridDim.x) + 1 : 0;  // tiles of this CTA

  // ---- W_L operands (hi / lo TF32 split), written once in the swizzled MMA layouts
  for (int e = tid; e < 16 * n_chunks * 32; e += kHThreads) {  // GEMM1 B: [c][ch]
    const int c = e / (n_chunks * 32), ch = e % (n_chunks * 32);
    const float w = (c < C && ch < Ch) ? a.w[c * Ch + ch] : 0.f;
    const float hi = tf32_rna_h(w), lo = w - hi;
    const uint32_t o = (uint32_t)(ch >> 5) * 2048u + sw128_off(c, ch & 31);
    *reinterpret_cast<float*>(gbase + L.w1 + o) = hi;
    (void)lo;
  }
  for (int e = tid; e < 256 * 8; e += kHThreads) {  // GEMM2 A: [ch][c]
    const int ch = e >> 3, c = e & 7;
    const float w = (c < C && ch < Ch) ? a.w[c * Ch + ch] : 0.f;
    const float hi = tf32_rna_h(w), lo = w - hi;
    const uint32_t o = (uint32_t)(ch >> 7) * 4096u + sw32_off(ch & 127, c);
    *reinterpret_cast<float*>(gbase + L.w2 + o) = hi;
    *reinterpret_cast<float*>(gbase + L.w2 + 2 * 4096 + o) = lo;
  }
  if (tid < 16) s_b[tid] = tid < C ? a.b[tid] : 0.f;
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmH);
    for (int i = 0; i < kHS; ++i) {
      ptx::mbar_init(bFull + 8 * i, 1);
      ptx::mbar_init(bEmpty + 8 * i, 1 + kHDh);  // GEMM1's commit + every dh warp
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(bZfull + 8 * i, 1);
      ptx::mbar_init(bZempty + 8 * i, kHSm);
      ptx::mbar_init(bDlfull + 8 * i, kHSm);
      ptx::mbar_init(bDlempty + 8 * i, kHDh);
      ptx::mbar_init(bDhfull + 8 * i, 1);
      ptx::mbar_init(bDhempty + 8 * i, kHDh);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(sTmemSlot, 512);
  ptx::fence_proxy_async();  // the operand writes above -> async proxy (tensor core)
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(gbase + (sTmemSlot - sbase));
  auto tile_of = [&](int i) { return (long long)blockIdx.x + (long long)i * gridDim.x; };

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int q = 0;
      for (int i = 0; i < n_my; ++i) {
        const long long tile = tile_of(i);
        const int img = (int)(tile / tiles_per_img64), tt = (int)(tile % tiles_per_img64);
        const int row0 = (int)((long long)img * per_img + (long long)tt * kHT);
        for (int j = 0; j < n_chunks; ++j, ++q) {
          const int s = q % kHS;
          pwait(bEmpty + 8 * s, ((q / kHS) & 1) ^ 1, prof, 8);
          ptx::mbar_arrive_expect_tx(bFull + 8 * s, kHChunk);
          ptx::tma_load_2d(sbase + L.ring + s * kHChunk, &tmH, bFull + 8 * s, j * 32, row0);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t id1 = ptx::idesc_tf32(64, 16), id2 = ptx::idesc_tf32(128, 64);
    const int n_blk = (Ch + 127) / 128;
    auto gemm1 = [&](int i) {  // Z[i&1] = H W_L^T  (W_L = hi + lo)
      const int b = i & 1;
      pwait(bZempty + 8 * b, ((i >> 1) & 1) ^ 1, prof, 3);
      ptx::tc_fence_after();
      for (int j = 0; j < n_chunks; ++j) {
        const int q = i * n_chunks + j, s = q % kHS;
        pwait(bFull + 8 * s, (q / kHS) & 1, prof, 1);
        ptx::tc_fence_after();
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          const uint64_t ad = ptx::sdesc_k_sw128(sbase + L.ring + s * kHChunk + k8 * 32, 0);
          const uint64_t bd = ptx::sdesc_k_sw128(sbase + L.w1 + j * 2048 + k8 * 32, 0);
          ptx::mma_tf32_elect(tmem + b * 16, ad, bd, id1, (j | k8) != 0);
        }
        ptx::mma_commit_elect(bEmpty + 8 * s);
      }
      ptx::mma_commit_elect(bZfull + 8 * b);
    };
    const long long t_start = clock64();
    if (n_my > 0) gemm1(0);
    for (int i = 0; i < n_my; ++i) {
      if (i + 1 < n_my) gemm1(i + 1);
      // GEMM2(i): dhT[b][ch][pos] = W_L^T dz^T (3xTF32)
      const int b = i & 1;
      pwait(bDlfull + 8 * b, (i >> 1) & 1, prof, 0);
      pwait(bDhempty + 8 * b, ((i >> 1) & 1) ^ 1, prof, 2);
      ptx::tc_fence_after();
      const uint32_t dlb = sbase + L.dl + b * (2 * kHT * 32);
      for (int m = 0; m < n_blk; ++m) {
        const uint32_t d = tmem + 32 + b * 128 + m * 64;
        const uint64_t a_hi = sdesc_k_sw32(sbase + L.w2 + m * 4096), a_lo = sdesc_k_sw32(sbase + L.w2 + (2 + m) * 4096);
        const uint64_t b_hi = sdesc_k_sw32(dlb), b_lo = sdesc_k_sw32(dlb + kHT * 32);
        ptx::mma_tf32_elect(d, a_hi, b_hi, id2, 0u);
        ptx::mma_tf32_elect(d, a_hi, b_lo, id2, 1u);
        ptx::mma_tf32_elect(d, a_lo, b_hi, id2, 1u);
      }
      ptx::mma_commit_elect(bDhfull + 8 * b);
    }
    if (prof && lane == 0) atomicAdd(prof + 9, (unsigned long long)(clock64() - t_start));
  } else if (warp >= 2 + kHDh) {
    // ------------------------------------------------------------------ softmax warps
    // lanes 0..15 of warp q: position 16 q + lane (the M = 64 accumulator layout)
    const int q = warp & 3, sw = warp - 2 - kHDh;
    const bool on = lane < 16;
    const int pos = q * 16 + (lane & 15);
    float accL[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) accL[c] = 0.f;
    // labels (and the image's label count) run one tile ahead: their loads stay in
    // flight (unconsumed) while the previous tile is processed
    HeadLabel lq{kLabBeyond, 255};
    int nq = 0;
    auto issue = [&](int i) {
      if (i < n_my && on) {
        const long long tile = tile_of(i);
        const int img = (int)(tile / tiles_per_img64);
        lq = head_label_issue(a, img, (tile % tiles_per_img64) * kHT + pos, per_img, frag_sz);
        nq = __ldg(a.nlab + img);
      }
    };
    issue(0);
    for (int i = 0; i < n_my; ++i) {
      const int b = i & 1;
      const long long tile = tile_of(i);
      const int img = (int)(tile / tiles_per_img64), tt = (int)(tile % tiles_per_img64);
      const int lab = on ? head_label_finish(a, lq) : kLabBeyond;
      const int nl = nq;
      issue(i + 1);
      pwait(bZfull + 8 * b, (i >> 1) & 1, prof, 4);
      ptx::tc_fence_after();
      float z[16];
      ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + b * 16, z);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bZempty + 8 * b);
      float dl[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) dl[c] = 0.f;
      float lossv = 0.f;
      if (on && lab >= 0 && lab < C) {
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < C) {
            z[c] += s_b[c];
            mx = fmaxf(mx, z[c]);
          }
        float se = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < C) se += expf(z[c] - mx);
        const float lse = mx + logf(se);
        const float wt = a.cw[lab];
        float zt = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c == lab) zt = z[c];
        lossv = wt * (lse - zt);
        const float inv = nl > 0 ? wt / (float)nl : 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < C) dl[c] = inv * (expf(z[c] - lse) - (c == lab ? 1.f : 0.f));
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) accL[c] += dl[c];
      // dz rows: hi / lo TF32 split in the SW32 operand tile, fp32 copy for the FMAs;
      // buffer b was last read by GEMM2(i - 2) and the dh warps of tile i - 2
      pwait(bDlempty + 8 * b, ((i >> 1) & 1) ^ 1, prof, 5);
      if (on) {
        uint8_t* dlt = gbase + L.dl + b * (2 * kHT * 32);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float hi = tf32_rna_h(dl[c]);
          *reinterpret_cast<float*>(dlt + sw32_off(pos, c)) = hi;
          *reinterpret_cast<float*>(dlt + kHT * 32 + sw32_off(pos, c)) = dl[c] - hi;
        }
        float* dlp = reinterpret_cast<float*>(gbase + L.dlp) + b * (kHT * 8);
        reinterpret_cast<float4*>(dlp + pos * 8)[0] = make_float4(dl[0], dl[1], dl[2], dl[3]);
        reinterpret_cast<float4*>(dlp + pos * 8)[1] = make_float4(dl[4], dl[5], dl[6], dl[7]);
      }
      ptx::fence_proxy_async();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bDlfull + 8 * b);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lossv += __shfl_xor_sync(0xffffffffu, lossv, o);
      if (lane == 0) {  // per-(tile, warp) loss, the layout of head.cu (8 parts per tile)
        const long long base = ((long long)img * a.tiles_per_img + tt) * 8;
        a.loss_part[base + sw] = lossv;
        a.loss_part[base + kHSm + sw] = 0.f;
      }
    }
    // db_L: warp sums, then (after the barrier) a fixed-order sum of the 4 warps
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) accL[c] += __shfl_xor_sync(0xffffffffu, accL[c], o);
    if (lane == 0)
#pragma unroll
      for (int c = 0; c < 8; ++c) s_red[sw * 8 + c] = accL[c];
    named_bar(1, 32 * (kHDh + kHSm));
  } else {
    // ------------------------------------------------------------------ dh warps
    // lane quarter q = warp & 3, slot sl = (warp - 2) / 4: channel block sl % n_blk and
    // the sl / n_blk-th share of the tile's 64 positions.  h comes from the ring chunk
    // that GEMM1 read (conflict-free: a warp reads one 128-byte row per position).
    const int dw = warp - 2, q = warp & 3, sl = dw >> 2;
    const int n_blk = (Ch + 127) / 128, n_parts = (kHDh / 4) / n_blk;
    const int blk = sl % n_blk, part = sl / n_blk, pw = kHT / n_parts;
    const int ch = blk * 128 + q * 32 + lane;
    const bool ch_ok = ch < Ch;
    const int jc = min(ch, Ch - 1) >> 5;  // this channel's chunk
    float accW[8], accP = 0.f;
#pragma unroll
    for (int c = 0; c < 8; ++c) accW[c] = 0.f;
    const int act = a.hidden_act;
    for (int i = 0; i < n_my; ++i) {
      const int b = i & 1;
      const long long tile = tile_of(i);
      const int img = (int)(tile / tiles_per_img64), tt = (int)(tile % tiles_per_img64);
      const long long p0 = (long long)tt * kHT;
      const int np = (int)min((long long)kHT, per_img - p0);
      float* drow = a.dh + ((long long)img * per_img + p0) * Ch + ch;
      const float* dlp = reinterpret_cast<const float*>(gbase + L.dlp) + b * (kHT * 8);
      const int qc = i * n_chunks + jc, s = qc % kHS;
      pwait(bFull + 8 * s, (qc / kHS) & 1, prof, 7);  // (complete: GEMM1 read it) orders the TMA writes
      const uint8_t* hch = gbase + L.ring + s * kHChunk;
      pwait(bDhfull + 8 * b, (i >> 1) & 1, prof, 6);
      ptx::tc_fence_after();
      const int pbeg = part * pw, pend = min(pbeg + pw, np);
      for (int pc = pbeg; pc < pend; pc += 8) {  // warp-uniform
        float v[8];
        ptx::tmem_ld8(tmem + ((uint32_t)(q * 32) << 16) + 32 + b * 128 + blk * 64 + pc, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int pos = pc + j;
          if (pos < pend && ch_ok) {
            const float hh = *reinterpret_cast<const float*>(hch + sw128_off(pos, ch & 31));
            const float der = act == MPF_TANH ? fmaf(-hh, hh, 1.f) : (act == MPF_LOGISTIC ? hh * (1.f - hh) : 1.f);
            const float d = v[j] * der;
            accP += d;
            drow[(long long)pos * Ch] = a.round_tf32 ? tf32_rna_h(d) : d;
            const float4 d0 = reinterpret_cast<const float4*>(dlp + pos * 8)[0];
            accW[0] = fmaf(d0.x, hh, accW[0]);
            accW[1] = fmaf(d0.y, hh, accW[1]);
            if (NC > 2) accW[2] = fmaf(d0.z, hh, accW[2]);
            if (NC > 3) accW[3] = fmaf(d0.w, hh, accW[3]);
            if (NC > 4) {
              const float4 d1 = reinterpret_cast<const float4*>(dlp + pos * 8)[1];
              accW[4] = fmaf(d1.x, hh, accW[4]);
              if (NC > 5) accW[5] = fmaf(d1.y, hh, accW[5]);
              if (NC > 6) accW[6] = fmaf(d1.z, hh, accW[6]);
              if (NC > 7) accW[7] = fmaf(d1.w, hh, accW[7]);
            }
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        ptx::mbar_arrive(bDhempty + 8 * b);
        ptx::mbar_arrive(bDlempty + 8 * b);
        for (int j = 0; j < n_chunks; ++j) ptx::mbar_arrive(bEmpty + 8 * ((i * n_chunks + j) % kHS));
      }
    }
    // ---- block partials: [dW_L (C x Ch) | db_L (C) | db_prev (Ch)]; a channel's sums
    // are split over the n_parts slots of its block: fixed-order sum through smem
    const int E = C * Ch + C + Ch;
    float* out = a.part + (size_t)blockIdx.x * E;
    named_bar(2, 32 * kHDh);  // every dh warp is past its last ring read
    float* s_acc = reinterpret_cast<float*>(gbase + L.ring);  // the ring is idle now
    if (ch_ok) {
#pragma unroll
      for (int c = 0; c < 8; ++c)  // constant indices keep accW in registers
        if (c < C) s_acc[(part * (C + 1) + c) * kHMaxCh + ch] = accW[c];
      s_acc[(part * (C + 1) + C) * kHMaxCh + ch] = accP;
    }
    named_bar(1, 32 * (kHDh + kHSm));
    if (part == 0 && ch_ok) {
      for (int c = 0; c <= C; ++c) {
        float t = 0.f;
        for (int pp = 0; pp < n_parts; ++pp) t += s_acc[(pp * (C + 1) + c) * kHMaxCh + ch];
        if (c < C) out[c * Ch + ch] = t;
        else out[C * Ch + C + ch] = t;
      }
    }
    if (dw == 0 && lane < C) out[C * Ch + lane] = ((s_red[lane] + s_red[8 + lane]) + s_red[16 + lane]) + s_red[24 + lane];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

size_t htc_smem(int Ch) {
  const int n_chunks = (Ch + 31) / 32;
  const HtcLayout L = htc_layout(n_chunks);
  return 1024 + L.bar + 8 * kHBars + 16;
}

}  // namespace

// Training head on the tensor cores: TF32 mode (h arrives TF32-rounded from the layer
// below), C <= 8 classes, Ch <= 256 channels in 16-byte rows.  Opt-in (MPF_HEAD_TC=1):
// correct (GPU parity suite) but measured slower than the CUDA-core head (head.cu) on
// cfg4 (4.74 vs 4.68 ms) and cfg5 (1.46 vs 1.05 ms); its epilogue pipeline is
// latency-bound.
bool head_tc_ok(int C, int Ch, bool train, bool tf32) {
  const char* e = getenv("MPF_HEAD_TC");
  if (!train || !tf32 || !e || atoi(e) == 0) return false;
  return C >= 2 && C <= 8 && Ch >= 8 && Ch <= kHMaxCh && Ch % 4 == 0 && htc_smem(Ch) <= 227 * 1024;
}

int head_tc_grid(long long per_img, int n) {
  const long long tiles = (long long)n * ((per_img + kHT - 1) / kHT);
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  return (int)(tiles < sms ? (tiles < 1 ? 1 : tiles) : sms);
}

cudaError_t launch_head_tc(const HeadArgs& a, cudaStream_t s) {
  const long long per_img = (long long)a.F * a.gr * a.gc;
  const int tpi = (int)((per_img + kHT - 1) / kHT);
  const int n_chunks = (a.Ch + 31) / 32;
  CUtensorMap tm;
  cudaError_t e = make_tmap_sw128(&tm, a.h, (uint64_t)a.Ch, (uint64_t)(a.n * per_img), (uint32_t)kHT);
  if (tpi != a.tiles_per_img) return cudaErrorInvalidValue;  // loss parts use head.cu's tiling
  if (e != cudaSuccess) return e;
  const size_t smem = htc_smem(a.Ch);
  auto kern = a.C == 2 ? head_tc_kernel<2> : a.C == 3 ? head_tc_kernel<3> : a.C == 4 ? head_tc_kernel<4>
            : a.C == 5 ? head_tc_kernel<5> : head_tc_kernel<8>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  static unsigned long long* prof = nullptr;
  const bool do_prof = getenv("MPF_HEAD_PROF") != nullptr;
  if (do_prof && !prof) cudaMalloc(&prof, 16 * sizeof(unsigned long long));
  if (do_prof) cudaMemsetAsync(prof, 0, 16 * sizeof(unsigned long long), s);
  kern<<<a.n_blocks, kHThreads, smem, s>>>(tm, a, tpi, n_chunks, do_prof ? prof : nullptr);
  if (do_prof) {
    unsigned long long h[16];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double cta = a.n_blocks;
    fprintf(stderr,
            "[head-prof] per CTA Mcyc: total(mma warp) %.3f | mma wait dlfull %.3f full %.3f dhempty %.3f zempty %.3f | "
            "softmax(per warp) zfull %.3f dlempty %.3f | dh(per warp) dhfull %.3f full %.3f | producer empty %.3f\n",
            h[9] / cta / 1e6, h[0] / cta / 1e6, h[1] / cta / 1e6, h[2] / cta / 1e6, h[3] / cta / 1e6,
            h[4] / cta / kHSm / 1e6, h[5] / cta / kHSm / 1e6, h[6] / cta / kHDh / 1e6, h[7] / cta / kHDh / 1e6,
            h[8] / cta / 1e6);
  }
  return cudaGetLastError();
}

}  // namespace mpf
