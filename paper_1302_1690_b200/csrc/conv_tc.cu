// conv_tc.cu — tcgen05 (kind::tf32, TMEM accumulators, TMA-fed) implicit-GEMM
// convolution over all fragments at once: forward of C/FC layers (Alg. 1 applied to
// every fragment) and the delta propagation (dgrad) of the backward.
//
// GEMM view.  Positions are flattened over (image, fragment, row, col) of the storage
// grid (row pitch gc): p = ((f * gr) + y) * gc + x.  A valid k x k correlation is a
// sum over k^2 taps t = (ky, kx) of a position shift:
//     D[p, co] = sum_t sum_ci X[p + base + ky*gc + kx, ci] * W[co, t, ci]
// with base = 0 (forward) or -(k-1)(gc+1) (dgrad, rotated weights).  Positions whose
// window leaves the fragment are garbage and are written as 0.  Reads outside the
// tensor are zero-filled by TMA.  Delta tensors are zero outside their valid region,
// which makes the dgrad "full correlation" exact with the same 1-D formulation.
//
// Kernel (persistent, one CTA per SM).  A tile is M_cta = NACC x 128 consecutive
// positions x all output channels (N = cout padded to 16) held in NACC TMEM
// accumulators of 128 x N fp32; two such accumulator sets alternate so the epilogue
// of tile i overlaps the MMAs of tile i+1.  K loop over stages (ky, 32-channel chunk):
// one TMA "slab" of M_cta + k - 1 input rows (128 B = 32 fp32 per row, SWIZZLE_128B)
// serves all k taps kx of that row — each tap only offsets the UMMA descriptor start
// by kx rows; the weights of each tap are a separate TMA tile [N x 32].
// Warp roles: warp 0 TMA producer, warp 1 TMEM allocator + single-thread MMA issuer,
// warps 2-5 epilogue: TMEM -> registers -> bias/act/act'/tf32 rounding -> swizzled
// shared staging -> TMA tile store (the output tile rows are consecutive positions,
// so every store is a dense [32 rows x 32 channels] box).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include <mutex>

#include "conv_tc.h"
#include "tc_ptx.cuh"
#include "mpf_internal.h"
#include "numerics.cuh"

namespace mpf {

namespace {

constexpr int kEpiWarps = 8;   // two per TMEM lane quarter, splitting the column chunks
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kKC = 32;        // fp32 channels per 128-byte row
constexpr uint32_t kStageBytes = 32 * 128;  // one epilogue store box: 32 rows x 32 fp32

struct ConvTcParams {
  int P_tot, gr, gc, out_vr, out_vc;
  int cin, cout, npad, k, shift_rows, n_cc;
  int last_k8;  // k8 steps of the last channel chunk that hold real channels (1..4)
  int act, round_out, dact;
  const float* bias;
  const float* mul_dact;
  int box_rows, nbox;
  uint32_t a_slot_bytes, b_slot_bytes;  // per stage: one A slab + k weight taps of b_slot_bytes
  uint32_t stage_bytes;
  int n_stages;
  int n_stage;  // epilogue staging boxes per warp (1 or 2)
  int base_mode;
  uint32_t tmem_cols;
  int n_tiles;   // tiles of M_CTA (single) or 2 x M_CTA (pair) positions
  int b_rows;    // weight rows per B slot (npad, or npad/2 per CTA of a pair)
  unsigned long long* prof;  // optional role-timing counters (MPF_FLAG_ROLE_TIMERS)
  // logits of the softmax FC in the epilogue (forward of the last hidden layer, head_z set):
  // z[p][c] = sum_ch W_L[c][ch] h[p][ch] over the stored (rounded) h, bias excluded
  const float* head_w;  // canonical W_L [head_C][cout]
  float* head_z;        // [P_tot][head_C]
  int head_C;
};
constexpr int kMaxHeadC = 16;
// row stride of W_L in shared memory: whole 32-channel chunks, zero beyond cout (the last
// chunk of an npad % 32 == 16 layer reads 32 weights; its channels past cout hold act(0))
__host__ __device__ inline int head_w_ld(int npad) { return (npad + 31) / 32 * 32; }
// shared bytes of the logits epilogue: W_L [head_C][ld] + two exchange slots [4][32][head_C]
__host__ __device__ inline uint32_t head_epi_bytes(int head_C, int npad) {
  return head_C > 0 ? (uint32_t)(4 * head_C * head_w_ld(npad) + 2 * 4 * 32 * 4 * head_C) : 0u;
}

// mbarrier wait that adds the cycles spent waiting to a counter when profiling
__device__ __forceinline__ void twait(uint32_t bar, uint32_t parity, unsigned long long& acc, bool on) {
  if (!on) {
    ptx::mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  ptx::mbar_wait(bar, parity);
  acc += (unsigned long long)(clock64() - t0);
}


__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// PAIR: a cluster of two CTAs on one TPC runs tcgen05 cta_group::2 MMAs (M = 256):
// each CTA stages its own positions (A) and HALF of every weight tile (B), the leader
// issues the MMAs, every accumulator lands in the TMEM of the CTA that owns its rows.
// MC (single-CTA tiles only): a cluster of two CTAs runs tiles 2u and 2u + 1 in lockstep;
// each loads half of the k weight taps of a stage and multicasts them to both (the weight
// stream from L2 per SM halves), and a stage slot is refilled only when both CTAs' MMAs
// have released it.
template <int NACC, bool PAIR, bool MC = false>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmO, ConvTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B aligned carve-up
  const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  // stage s: [A slab | k weight taps], one full/empty barrier pair per stage
  const uint32_t sS = sbase;
  const uint32_t sC = sS + p.n_stages * p.stage_bytes;         // epilogue staging boxes
  const uint32_t sBias = sC + p.n_stage * kEpiWarps * kStageBytes;  // [npad] fp32
  const uint32_t sBar = sBias + 4 * 256;
  const uint32_t barFull = sBar, barEmpty = barFull + 8 * p.n_stages;
  const uint32_t barTfull = barEmpty + 8 * p.n_stages, barTempty = barTfull + 16;
  const uint32_t sTmemSlot = barTempty + 16;
  uint8_t* gen = smem_raw - ptx::smem_u32(smem_raw);  // generic pointer of shared address 0
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(gen + sTmemSlot);
  float* s_bias = reinterpret_cast<float*>(gen + sBias);
  const int HC = p.head_z ? p.head_C : 0;  // logits epilogue (0: off)
  const int hw_ld = head_w_ld(p.npad);
  float* s_hw = reinterpret_cast<float*>(gen + sBar + 512);  // W_L [HC][hw_ld], zero-padded
  float* s_zx = s_hw + HC * hw_ld;                           // [2][4][32][HC] half-1 partials

  // warp index via a shuffle: provably warp-uniform, so role branches stay convergent and
  // the MMA warp's descriptor arithmetic lives in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  constexpr int M_CTA = NACC * 128;
  const uint32_t rank = PAIR ? ptx::cluster_rank() : 0u;
  const bool leader = rank == 0;
  static_assert(!(PAIR && MC), "multicast is for single-CTA tiles");
  const int mrank = MC ? (int)ptx::cluster_rank() : 0;
  // tiles: one per CTA, or one per pair (2 x M_CTA positions, CTA r owns the r-th half); MC:
  // both CTAs of a cluster iterate over the same number of tiles (tile 2u + 1 may lie past
  // the end: its loads read zeros and its stores are clipped)
  const int unit0 = PAIR ? (int)(blockIdx.x >> 1) : (MC ? (int)(blockIdx.x >> 1) * 2 + mrank : (int)blockIdx.x);
  const int n_units = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int tile_end = MC ? (p.n_tiles + 1) / 2 * 2 : p.n_tiles;
  const int tile_pos = PAIR ? 2 * M_CTA : M_CTA;
  const int my_off = (int)rank * M_CTA;
  // the pair's full barriers and the TMEM-empty barriers live in the leader
  const uint32_t barFullL = PAIR ? ptx::mapa(barFull, 0) : barFull;
  const uint32_t barTemptyL = PAIR ? ptx::mapa(barTempty, 0) : barTempty;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    ptx::prefetch_tmap(&tmO);
    for (int i = 0; i < p.n_stages; ++i) {
      ptx::mbar_init(barFull + 8 * i, 1);
      ptx::mbar_init(barEmpty + 8 * i, MC ? 2 : 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(barTfull + 8 * i, 1);
      ptx::mbar_init(barTempty + 8 * i, (PAIR ? 2 : 1) * kEpiWarps);  // one arrive per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) {
    if (PAIR) ptx::tmem_alloc_pair(sTmemSlot, p.tmem_cols);
    else ptx::tmem_alloc(sTmemSlot, p.tmem_cols);
  }
  for (int c = threadIdx.x; c < 256; c += kThreads) s_bias[c] = (p.bias && c < p.cout) ? p.bias[c] : 0.f;
  for (int e = threadIdx.x; e < HC * hw_ld; e += kThreads) {
    const int c = e / hw_ld, ch = e - c * hw_ld;
    s_hw[e] = ch < p.cout ? p.head_w[c * p.cout + ch] : 0.f;
  }
  ptx::tc_fence_before();
  if (PAIR || MC) ptx::cluster_sync_all();  // barrier inits and TMEM allocation visible to the peer
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;

  const int k = p.k;
  const bool prof_on = p.prof != nullptr;
  unsigned long long pc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      const uint32_t npair = PAIR ? 2u : 1u;
      for (int tile = unit0; tile < tile_end; tile += n_units) {
        const int p0 = tile * tile_pos + my_off;
        for (int ky = 0; ky < k; ++ky) {
          for (int cc = 0; cc < p.n_cc; ++cc, ++it) {
            const int st = it % p.n_stages;
            twait(barEmpty + 8 * st, ((it / p.n_stages) & 1) ^ 1, pc[0], prof_on);
            if (leader) ptx::mbar_arrive_expect_tx(barFull + 8 * st, npair * (p.a_slot_bytes + k * p.b_slot_bytes));
            const uint32_t bar = (PAIR ? barFullL : barFull) + 8 * st;
            const uint32_t sa = sS + st * p.stage_bytes;
            const int row0 = p0 + p.shift_rows + ky * p.gc;
            for (int b = 0; b < p.nbox; ++b) {
              if (PAIR) ptx::tma_load_2d_pair(sa + b * p.box_rows * 128, &tmA, bar, cc * kKC, row0 + b * p.box_rows);
              else ptx::tma_load_2d(sa + b * p.box_rows * 128, &tmA, bar, cc * kKC, row0 + b * p.box_rows);
            }
            for (int kx = 0; kx < k; ++kx) {
              const uint32_t sb = sa + p.a_slot_bytes + kx * p.b_slot_bytes;
              const int c0 = (ky * k + kx) * p.cin + cc * kKC;
              if (PAIR) ptx::tma_load_2d_pair(sb, &tmB, bar, c0, (int)rank * p.b_rows);
              else if (MC) {
                if ((kx & 1) == mrank) ptx::tma_load_2d_mc(sb, &tmB, bar, c0, 0, (uint16_t)3);
              } else ptx::tma_load_2d(sb, &tmB, bar, c0, 0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    const uint32_t idesc = ptx::idesc_tf32(PAIR ? 256 : 128, p.npad);
    int it = 0, lt = 0;
    for (int tile = unit0; leader && tile < tile_end; tile += n_units, ++lt) {
      const int buf = lt & 1;
      twait(barTempty + 8 * buf, ((lt >> 1) & 1) ^ 1, pc[3], prof_on);  // the epilogue drained this set
      ptx::tc_fence_after();
      const uint32_t dbase = tmem + buf * (NACC * p.npad);
      for (int ky = 0; ky < k; ++ky) {
        for (int cc = 0; cc < p.n_cc; ++cc, ++it) {
          const int st = it % p.n_stages;
          twait(barFull + 8 * st, (it / p.n_stages) & 1, pc[4], prof_on);
          ptx::tc_fence_after();
          const uint32_t sa = sS + st * p.stage_bytes;
          const uint64_t adesc0 = ptx::sdesc_k_sw128(sa, p.base_mode);
          const uint64_t bdesc0 = ptx::sdesc_k_sw128(sa + p.a_slot_bytes, p.base_mode);
          // the last channel chunk skips its all-zero k8 steps (e.g. C_in = 200: 7 chunks of
          // 32, the last holding 8 real channels)
          const int nk8 = cc == p.n_cc - 1 ? p.last_k8 : 4;
          for (int kx = 0; kx < k; ++kx) {
#pragma unroll
            for (int acc = 0; acc < NACC; ++acc) {
#pragma unroll
              for (int k8 = 0; k8 < 4; ++k8) {
                if (k8 >= nk8) break;  // warp-uniform
                // descriptor start-address field is (addr >> 4) in the low bits
                const uint64_t ad = adesc0 + (uint64_t)((((acc * 128 + kx) * 128) + k8 * 32) >> 4);
                const uint64_t bd = bdesc0 + (uint64_t)((kx * p.b_slot_bytes + k8 * 32) >> 4);
                const uint32_t accum = (ky | cc | kx | k8) != 0;
                if (PAIR) ptx::mma_tf32_pair_elect(dbase + acc * p.npad, ad, bd, idesc, accum);
                else ptx::mma_tf32_elect(dbase + acc * p.npad, ad, bd, idesc, accum);
              }
            }
          }
          if (PAIR) ptx::mma_commit_pair_elect(barEmpty + 8 * st, 3);  // frees the stage in both CTAs
          else if (MC) ptx::mma_commit_mc_elect(barEmpty + 8 * st, (uint16_t)3);
          else ptx::mma_commit_elect(barEmpty + 8 * st);
        }
      }
      if (PAIR) ptx::mma_commit_pair_elect(barTfull + 8 * buf, 3);
      else ptx::mma_commit_elect(barTfull + 8 * buf);
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;  // which alternate 32-column chunks this warp stores
    const int ew = warp - 2;
    const int per_frag = p.gr * p.gc;
    int lt = 0, sb = 0, zslot = 0;
    for (int tile = unit0; tile < tile_end; tile += n_units, ++lt) {
      const int buf = lt & 1;
      twait(barTfull + 8 * buf, (lt >> 1) & 1, pc[7], prof_on);
      ptx::tc_fence_after();
      const int p0 = tile * tile_pos + my_off;
      for (int acc = 0; acc < NACC; ++acc) {
        float zc[kMaxHeadC];  // this half's logit partials of position row0 + lane
#pragma unroll
        for (int c = 0; c < kMaxHeadC; ++c) zc[c] = 0.f;
        const int row0 = p0 + acc * 128 + q * 32;
        const int pos = row0 + lane;
        bool valid = false;
        if (pos < p.P_tot) {
          const int r = pos % per_frag;
          const int y = r / p.gc, x = r - (r / p.gc) * p.gc;
          valid = y < p.out_vr && x < p.out_vc;
        }
        const float* md = (p.mul_dact && valid) ? p.mul_dact + (size_t)pos * p.cout : nullptr;
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + buf * (NACC * p.npad) + acc * p.npad;
        for (int c0 = 32 * half; c0 < p.npad; c0 += 64) {
          const long long e0 = prof_on ? clock64() : 0;
          uint32_t r[32];
          const bool two = c0 + 16 < p.npad;
          {
            uint32_t* r0 = r;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r0[0]), "=r"(r0[1]), "=r"(r0[2]), "=r"(r0[3]), "=r"(r0[4]), "=r"(r0[5]), "=r"(r0[6]),
                  "=r"(r0[7]), "=r"(r0[8]), "=r"(r0[9]), "=r"(r0[10]), "=r"(r0[11]), "=r"(r0[12]), "=r"(r0[13]),
                  "=r"(r0[14]), "=r"(r0[15])
                : "r"(taddr + c0));
          }
          if (two) {
            uint32_t* r1 = r + 16;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r1[0]), "=r"(r1[1]), "=r"(r1[2]), "=r"(r1[3]), "=r"(r1[4]), "=r"(r1[5]), "=r"(r1[6]),
                  "=r"(r1[7]), "=r"(r1[8]), "=r"(r1[9]), "=r"(r1[10]), "=r"(r1[11]), "=r"(r1[12]), "=r"(r1[13]),
                  "=r"(r1[14]), "=r"(r1[15])
                : "r"(taddr + c0 + 16));
          } else {
#pragma unroll
            for (int j = 16; j < 32; ++j) r[j] = 0u;
          }
          // operand of the act' multiply (dgrad), 32 contiguous floats of this row
          float mdv[32];
          if (md) {
            if (c0 + 32 <= p.cout) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 t = __ldg(reinterpret_cast<const float4*>(md + c0) + j);
                mdv[4 * j] = t.x; mdv[4 * j + 1] = t.y; mdv[4 * j + 2] = t.z; mdv[4 * j + 3] = t.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) mdv[j] = (c0 + j < p.cout) ? __ldg(md + c0 + j) : 0.f;
            }
          }
          ptx::tmem_ld_wait();
          const long long e1 = prof_on ? clock64() : 0;
          // every branch below is warp-uniform (kernel parameters) except `valid`, taken
          // once per row: no per-element control flow
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) + s_bias[c0 + j];
          if (p.act == MPF_TANH) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fast_tanh(v[j]);
          } else if (p.act == MPF_LOGISTIC) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = fast_logistic(v[j]);
          }
          if (md) {
            if (p.dact == MPF_TANH) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] *= fmaf(-mdv[j], mdv[j], 1.f);
            } else if (p.dact == MPF_LOGISTIC) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] *= mdv[j] * (1.f - mdv[j]);
            }
          }
          if (p.round_out) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = tf32_rn(v[j]);
          }
          if (!valid) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = 0.f;
          }
          if (HC) {  // logits: W_L rows of this chunk are broadcast reads (same address per warp)
#pragma unroll
            for (int c = 0; c < kMaxHeadC; ++c) {
              if (c >= HC) break;
              const float4* w4 = reinterpret_cast<const float4*>(s_hw + c * hw_ld + c0);
              float t = zc[c];
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 w = w4[j];
                t = fmaf(w.x, v[4 * j], t);
                t = fmaf(w.y, v[4 * j + 1], t);
                t = fmaf(w.z, v[4 * j + 2], t);
                t = fmaf(w.w, v[4 * j + 3], t);
              }
              zc[c] = t;
            }
          }
          // staging box (swizzled like the TMA SWIZZLE_128B pattern): 16-B chunk jj of
          // row `lane` lives at lane*128 + ((jj ^ (lane & 7)) * 16)
          const uint32_t sbuf = sC + (ew * p.n_stage + sb) * kStageBytes;
          const long long e2 = prof_on ? clock64() : 0;
          if (lane == 0) {  // the store that last used this box has finished reading it
            if (p.n_stage == 2) ptx::bulk_wait_read<1>();
            else ptx::bulk_wait_read<0>();
          }
          __syncwarp();
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const uint32_t a = sbuf + lane * 128 + ((jj ^ (lane & 7)) * 16);
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v[4 * jj]), "f"(v[4 * jj + 1]),
                         "f"(v[4 * jj + 2]), "f"(v[4 * jj + 3])
                         : "memory");
          }
          ptx::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            ptx::tma_store_2d(&tmO, sbuf, c0, row0);
            ptx::bulk_commit();
          }
          sb = (sb + 1 == p.n_stage) ? 0 : sb + 1;
          if (prof_on) {
            const long long e3 = clock64();
            pc[1] += (unsigned long long)(e1 - e0);   // TMEM loads (+ act' operand loads)
            pc[5] += (unsigned long long)(e2 - e1);   // epilogue math
            pc[9] += (unsigned long long)(e3 - e2);   // staging wait + st.shared + fence + store issue
          }
        }
        if (HC) {  // z = half-0 partial + half-1 partial (fixed order), written by half 0
          float* slot = s_zx + ((zslot * 4 + q) * 32 + lane) * HC;
          if (half) {
#pragma unroll
            for (int c = 0; c < kMaxHeadC; ++c)
              if (c < HC) slot[c] = zc[c];
          }
          named_bar(1 + q, 64);
          if (!half && row0 + lane < p.P_tot) {
            float* zo = p.head_z + (size_t)(row0 + lane) * HC;
#pragma unroll
            for (int c = 0; c < kMaxHeadC; ++c)
              if (c < HC) zo[c] = zc[c] + slot[c];
          }
          zslot ^= 1;
        }
      }
      // every TMEM read of this accumulator set is complete: hand it back to the MMA warp
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (PAIR) ptx::mbar_arrive_cluster(barTemptyL + 8 * buf);
        else ptx::mbar_arrive(barTempty + 8 * buf);
      }
    }
    if (lane == 0) ptx::bulk_wait<0>();
  }
  if (prof_on && (warp >= 2 || lane == 0)) {
    const int slot_total = warp == 0 ? 2 : (warp == 1 ? 6 : 8);
    pc[slot_total] = (unsigned long long)(clock64() - t_start);
    for (int i = 0; i < 12; ++i)
      if (pc[i]) atomicAdd(p.prof + i, pc[i]);
  }
  ptx::tc_fence_before();
  if (PAIR || MC) ptx::cluster_sync_all();  // the peer may still signal our barriers until here
  else __syncthreads();
  if (warp == 1) {
    if (PAIR) ptx::tmem_dealloc_pair(tmem, p.tmem_cols);
    else ptx::tmem_dealloc(tmem, p.tmem_cols);
  }
}

// Narrow layers (k * npad <= 256, e.g. the dgrad into a 16/24/32-map layer): the k taps of a
// slab row go into ONE MMA of N = k * npad, D_kx[r] = sum_c A[p0 + r][c] W_kx[c] over the
// 128 slab rows r, instead of k MMAs of N = npad on A shifted by kx rows.  The A operand
// (4 KB per K step, the shared-memory-bound part of a narrow MMA) is then read
// once per K step instead of k times.  The shift moves to the epilogue:
// out[p0 + r] = sum_kx D_kx[r + kx], a sum over TMEM rows r .. r + k - 1 (lane shuffles; rows
// of the next lane quarter through a small shared exchange), so a tile of 128 accumulator
// rows yields TR = 128 - (k - 1) outputs and tiles overlap by k - 1 rows.  The last quarter
// stores its 32 - (k - 1) rows through a second tensor map with that box height, so a tile
// never writes its neighbour's rows.
// MC: a cluster of two CTAs runs tiles 2u and 2u + 1 in lockstep; each CTA loads half of the
// k weight taps of a stage and multicasts them to both, halving the weight stream from L2
// (the k = 5 dgrad was starved by it: 20 of its 36 KB per stage are weights, re-read for
// every 124-row tile).  A stage slot is refilled only after BOTH CTAs' MMAs released it.
template <int K, bool MC>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_ntap_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmO3,
                        ConvTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sS = sbase;
  const uint32_t sC = sS + p.n_stages * p.stage_bytes;
  const uint32_t sX = sC + p.n_stage * kEpiWarps * kStageBytes;  // [2 halves][4 q][7 taps][8 lanes][16]
  const uint32_t sBias = sX + 2 * 4 * 7 * 8 * 16 * 4;
  const uint32_t sBar = sBias + 4 * 256;
  const uint32_t barFull = sBar, barEmpty = barFull + 8 * p.n_stages;
  const uint32_t barTfull = barEmpty + 8 * p.n_stages, barTempty = barTfull + 16;
  const uint32_t sTmemSlot = barTempty + 16;
  uint8_t* gen = smem_raw - ptx::smem_u32(smem_raw);
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(gen + sTmemSlot);
  float* s_bias = reinterpret_cast<float*>(gen + sBias);
  float* s_x = reinterpret_cast<float*>(gen + sX);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  constexpr int k = K;
  const int TR = 128 - (k - 1), N = k * p.npad;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    ptx::prefetch_tmap(&tmO);
    ptx::prefetch_tmap(&tmO3);
    for (int i = 0; i < p.n_stages; ++i) {
      ptx::mbar_init(barFull + 8 * i, 1);
      ptx::mbar_init(barEmpty + 8 * i, MC ? 2 : 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(barTfull + 8 * i, 1);
      ptx::mbar_init(barTempty + 8 * i, kEpiWarps);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(sTmemSlot, p.tmem_cols);
  for (int c = threadIdx.x; c < 256; c += kThreads) s_bias[c] = (p.bias && c < p.cout) ? p.bias[c] : 0.f;
  ptx::tc_fence_before();
  if (MC) ptx::cluster_sync_all();  // the peer's barriers exist before anything is multicast
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  const int rank = MC ? (int)ptx::cluster_rank() : 0;
  const int first = MC ? (int)(blockIdx.x >> 1) * 2 + rank : (int)blockIdx.x;
  const int stride = MC ? (int)(gridDim.x >> 1) * 2 : (int)gridDim.x;
  // MC: both CTAs of the cluster run the same number of units (tile 2u + 1 may lie past the
  // end: its loads read zeros and its stores are clipped)
  const int n_iter_tiles = MC ? (p.n_tiles + 1) / 2 * 2 : p.n_tiles;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      for (int tile = first; tile < n_iter_tiles; tile += stride) {
        const int p0 = tile * TR;
        for (int ky = 0; ky < k; ++ky) {
          for (int cc = 0; cc < p.n_cc; ++cc, ++it) {
            const int st = it % p.n_stages;
            ptx::mbar_wait(barEmpty + 8 * st, ((it / p.n_stages) & 1) ^ 1);
            ptx::mbar_arrive_expect_tx(barFull + 8 * st, p.a_slot_bytes + k * p.b_slot_bytes);
            const uint32_t sa = sS + st * p.stage_bytes;
            ptx::tma_load_2d(sa, &tmA, barFull + 8 * st, cc * kKC, p0 + p.shift_rows + ky * p.gc);
            for (int kx = 0; kx < k; ++kx) {
              if (MC) {
                if ((kx & 1) == rank)
                  ptx::tma_load_2d_mc(sa + p.a_slot_bytes + kx * p.b_slot_bytes, &tmB, barFull + 8 * st,
                                      (ky * k + kx) * p.cin + cc * kKC, 0, (uint16_t)3);
              } else {
                ptx::tma_load_2d(sa + p.a_slot_bytes + kx * p.b_slot_bytes, &tmB, barFull + 8 * st,
                                 (ky * k + kx) * p.cin + cc * kKC, 0);
              }
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    const uint32_t idesc = ptx::idesc_tf32(128, N);
    int it = 0, lt = 0;
    for (int tile = first; tile < n_iter_tiles; tile += stride, ++lt) {
      const int buf = lt & 1;
      ptx::mbar_wait(barTempty + 8 * buf, ((lt >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t dbase = tmem + buf * N;
      for (int ky = 0; ky < k; ++ky) {
        for (int cc = 0; cc < p.n_cc; ++cc, ++it) {
          const int st = it % p.n_stages;
          ptx::mbar_wait(barFull + 8 * st, (it / p.n_stages) & 1);
          ptx::tc_fence_after();
          const uint32_t sa = sS + st * p.stage_bytes;
          const uint64_t adesc0 = ptx::sdesc_k_sw128(sa, p.base_mode);
          const uint64_t bdesc0 = ptx::sdesc_k_sw128(sa + p.a_slot_bytes, p.base_mode);
          const int nk8 = cc == p.n_cc - 1 ? p.last_k8 : 4;
#pragma unroll
          for (int k8 = 0; k8 < 4; ++k8) {
            if (k8 >= nk8) break;
            const uint64_t ad = adesc0 + (uint64_t)((k8 * 32) >> 4);
            const uint64_t bd = bdesc0 + (uint64_t)((k8 * 32) >> 4);
            ptx::mma_tf32_elect(dbase, ad, bd, idesc, (ky | cc | k8) != 0);
          }
          if (MC) ptx::mma_commit_mc_elect(barEmpty + 8 * st, (uint16_t)3);  // frees the slot in both CTAs
          else ptx::mma_commit_elect(barEmpty + 8 * st);
        }
      }
      ptx::mma_commit_elect(barTfull + 8 * buf);
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9)
    // The two warps of a lane quarter take alternate 16-column slices of every 32-column
    // chunk and share one swizzled staging box per chunk; the four warps of a half exchange
    // the first k - 1 rows of their quarter (taps 1 .. k-1) for the previous quarter.
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int per_frag = p.gr * p.gc;
    float* xq = s_x + ((half * 4 + q) * 7) * 8 * 16;
    const float* xn = s_x + ((half * 4 + q + 1) * 7) * 8 * 16;
    int lt = 0, sb = 0;
    for (int tile = first; tile < n_iter_tiles; tile += stride, ++lt) {
      const int buf = lt & 1;
      ptx::mbar_wait(barTfull + 8 * buf, (lt >> 1) & 1);
      ptx::tc_fence_after();
      const int p0 = tile * TR;
      const int r = q * 32 + lane;  // accumulator row = output row of this thread
      const int pos = p0 + r;
      bool valid = false;
      if (r < TR && pos < p.P_tot) {
        const int rr = pos % per_frag;
        const int y = rr / p.gc, x = rr - (rr / p.gc) * p.gc;
        valid = y < p.out_vr && x < p.out_vc;
      }
      const float* md = (p.mul_dact && valid) ? p.mul_dact + (size_t)pos * p.cout : nullptr;
      const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16) + buf * N;
      for (int c0 = 0; c0 < p.npad; c0 += 32) {
        const int cs = c0 + 16 * half;
        // the act' operand (a global load) is issued first so it lands while TMEM is read
        float mdv[16];
        if (md) {
          if (cs + 16 <= p.cout) {
#pragma unroll
            for (int j4 = 0; j4 < 4; ++j4) {
              const float4 t = __ldg(reinterpret_cast<const float4*>(md + cs) + j4);
              mdv[4 * j4] = t.x; mdv[4 * j4 + 1] = t.y; mdv[4 * j4 + 2] = t.z; mdv[4 * j4 + 3] = t.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) mdv[j] = (cs + j < p.cout) ? __ldg(md + cs + j) : 0.f;
          }
        }
        float o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = 0.f;
        if (cs < p.npad) {
          uint32_t v[K][16];
#pragma unroll
          for (int kx = 0; kx < K; ++kx)
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(v[kx][0]), "=r"(v[kx][1]), "=r"(v[kx][2]), "=r"(v[kx][3]), "=r"(v[kx][4]), "=r"(v[kx][5]),
                  "=r"(v[kx][6]), "=r"(v[kx][7]), "=r"(v[kx][8]), "=r"(v[kx][9]), "=r"(v[kx][10]), "=r"(v[kx][11]),
                  "=r"(v[kx][12]), "=r"(v[kx][13]), "=r"(v[kx][14]), "=r"(v[kx][15])
                : "r"(trow + kx * p.npad + cs));
          ptx::tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = __uint_as_float(v[0][j]);
#pragma unroll
          for (int kx = 1; kx < K; ++kx) {
            // rows 0 .. kx-1 of this quarter serve the previous quarter's last lanes
            if (lane < kx && q > 0) {
#pragma unroll
              for (int j4 = 0; j4 < 4; ++j4)
                *reinterpret_cast<float4*>(xq + ((kx - 1) * 8 + lane) * 16 + 4 * j4) =
                    make_float4(__uint_as_float(v[kx][4 * j4]), __uint_as_float(v[kx][4 * j4 + 1]),
                                __uint_as_float(v[kx][4 * j4 + 2]), __uint_as_float(v[kx][4 * j4 + 3]));
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float t = __shfl_down_sync(0xffffffffu, __uint_as_float(v[kx][j]), kx);
              if (lane + kx < 32) o[j] += t;
            }
          }
        }
        named_bar(1 + half, 128);  // every quarter's exchange rows are written
        if (cs < p.npad && q < 3) {
#pragma unroll
          for (int kx = 1; kx < K; ++kx) {
            if (lane + kx >= 32) {
              const float* src = xn + ((kx - 1) * 8 + (lane + kx - 32)) * 16;
#pragma unroll
              for (int j4 = 0; j4 < 4; ++j4) {
                const float4 t = *reinterpret_cast<const float4*>(src + 4 * j4);
                o[4 * j4] += t.x; o[4 * j4 + 1] += t.y; o[4 * j4 + 2] += t.z; o[4 * j4 + 3] += t.w;
              }
            }
          }
        }
        // the rest of the epilogue on this warp's 16 columns
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] += s_bias[(cs + j) & 255];
        if (p.act == MPF_TANH) {
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = fast_tanh(o[j]);
        } else if (p.act == MPF_LOGISTIC) {
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = fast_logistic(o[j]);
        }
        if (md) {
          if (p.dact == MPF_TANH) {
#pragma unroll
            for (int j = 0; j < 16; ++j) o[j] *= fmaf(-mdv[j], mdv[j], 1.f);
          } else if (p.dact == MPF_LOGISTIC) {
#pragma unroll
            for (int j = 0; j < 16; ++j) o[j] *= mdv[j] * (1.f - mdv[j]);
          }
        }
        if (p.round_out) {
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = tf32_rn(o[j]);
        }
        if (!valid) {
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = 0.f;
        }
        // shared staging box of the quarter (half 0's slot): half h fills columns 16h..16h+15
        const uint32_t sbuf = sC + (q * p.n_stage + sb) * kStageBytes;
        if (half == 0 && lane == 0) {  // the store that last used this box has read it
          if (p.n_stage == 2) ptx::bulk_wait_read<1>();
          else ptx::bulk_wait_read<0>();
        }
        named_bar(3 + q, 64);
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int chunk = half * 4 + jj;
          const uint32_t a = sbuf + lane * 128 + ((chunk ^ (lane & 7)) * 16);
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(o[4 * jj]), "f"(o[4 * jj + 1]),
                       "f"(o[4 * jj + 2]), "f"(o[4 * jj + 3])
                       : "memory");
        }
        ptx::fence_proxy_async();
        named_bar(3 + q, 64);
        if (half == 0 && lane == 0) {
          if (q < 3) ptx::tma_store_2d(&tmO, sbuf, c0, p0 + q * 32);
          else ptx::tma_store_2d(&tmO3, sbuf, c0, p0 + 96);  // rows 96 .. TR-1 only
          ptx::bulk_commit();
        }
        sb = (sb + 1 == p.n_stage) ? 0 : sb + 1;
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(barTempty + 8 * buf);
    }
    if (lane == 0) ptx::bulk_wait<0>();
  }
  ptx::tc_fence_before();
  if (MC) ptx::cluster_sync_all();  // the peer may still multicast into / arrive on our smem
  else __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, p.tmem_cols);
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_once;

cudaError_t get_encoder() {
  cudaError_t err = cudaSuccess;
  std::call_once(g_once, [&]() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (err == cudaSuccess && q == cudaDriverEntryPointSuccess) g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  });
  if (!g_encode) return cudaErrorNotSupported;
  return cudaSuccess;
}

// 2-D fp32 tensor [rows][cols] (cols contiguous), box {32 cols, box_rows}, SW128.
cudaError_t make_map(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint32_t box_rows,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  cudaError_t e = get_encoder();
  if (e != cudaSuccess) return e;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 4};
  cuuint32_t box[2] = {(cuuint32_t)kKC, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// UMMA descriptor base-offset mode: measured, the swizzle is address-based, base offset 0
int base_mode() { return 0; }

int g_num_sms = 0;
int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

unsigned long long* g_prof = nullptr;
unsigned long long* prof_counters(uint32_t flags) {
  if (!(flags & MPF_FLAG_ROLE_TIMERS)) return nullptr;
  if (!g_prof && cudaMalloc(&g_prof, 16 * sizeof(unsigned long long)) != cudaSuccess) g_prof = nullptr;
  if (g_prof) cudaMemset(g_prof, 0, 16 * sizeof(unsigned long long));
  return g_prof;
}
void prof_report(const ConvTcParams& p, int nacc, bool pair, int grid) {
  if (!p.prof) return;
  unsigned long long h[16];
  cudaDeviceSynchronize();
  cudaMemcpy(h, p.prof, sizeof(h), cudaMemcpyDeviceToHost);
  const double ctas = grid;
  fprintf(stderr,
          "[tc-prof] cin=%d cout=%d k=%d nacc=%d pair=%d tiles=%d grid=%d | per CTA Mcyc: prod total %.2f wAempty %.2f "
          "wBempty %.2f | mma total %.2f wTempty %.2f wAfull %.2f wBfull %.2f | epi(sum of %d warps) total %.2f wTfull %.2f\n",
          p.cin, p.cout, p.k, nacc, pair ? 1 : 0, p.n_tiles, grid, h[2] / ctas / 1e6, h[0] / ctas / 1e6,
          h[1] / ctas / 1e6, h[6] / ctas / 1e6, h[3] / ctas / 1e6, h[4] / ctas / 1e6, h[5] / ctas / 1e6, kEpiWarps,
          h[8] / ctas / 1e6, h[7] / ctas / 1e6);
  fprintf(stderr, "[tc-prof]   epi per thread Mcyc: tmem-ld %.2f math %.2f stage+store %.2f (of total %.2f)\n",
          h[1] / ctas / 256e6, h[5] / ctas / 256e6, h[9] / ctas / 256e6, h[8] / ctas / 256e6);
}

template <int NACC, bool PAIR, bool MC = false>
cudaError_t launch_nacc(const CUtensorMap& A, const CUtensorMap& B, const CUtensorMap& O, ConvTcParams& p,
                        size_t smem, cudaStream_t s) {
  auto kern = conv_tc_kernel<NACC, PAIR, MC>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (!PAIR && !MC) {
    const int grid = p.n_tiles < num_sms() ? p.n_tiles : num_sms();
    kern<<<grid, kThreads, smem, s>>>(A, B, O, p);
    prof_report(p, NACC, PAIR, grid);
    return cudaGetLastError();
  }
  // pairs of CTAs: a cta_group::2 pair per tile, or (MC) two single-CTA tiles in lockstep
  const int units = MC ? (p.n_tiles + 1) / 2 : p.n_tiles;
  const int pairs = units < num_sms() / 2 ? units : num_sms() / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, A, B, O, p);
  if (e != cudaSuccess) return e;
  prof_report(p, NACC, PAIR, 2 * pairs);
  return cudaGetLastError();
}

// CTA-pair policy: the pair halves the weight stream per SM, which pays only for wide,
// deep layers (N >= 192, or N >= 128 with K >= 1536); everywhere else the single-CTA MMA
// measured as fast or faster (per-layer A/B on cfg4/cfg5).
// MPF_FLAG_TC_PAIR / MPF_FLAG_TC_SINGLE force a mode.
bool want_pair(int npad, int K, uint32_t flags) {
  if (flags & MPF_FLAG_TC_SINGLE) return false;
  if (flags & MPF_FLAG_TC_PAIR) return true;
  return npad >= 192 || (npad >= 128 && K >= 1536);
}

}  // namespace

bool tc_supported(int cin, int cout, int k) {
  return cin % 4 == 0 && cin >= 16 && cout % 4 == 0 && cout >= 4 && cout <= 256 && k >= 1 && k <= 8;
}

// The multi-tap kernel for narrow layers (k * npad <= 256, npad <= 64) with k >= 5: measured
// 2.06 vs 2.58 ms on the cfg4 C5x5 dgrad (N = 32), but slower for k <= 4 (cfg5: 1.01 vs
// 0.75 ms), where the cross-row epilogue outweighs the A reads it saves.
// MPF_FLAG_NTAP_ON uses it for every eligible layer, MPF_FLAG_NTAP_OFF for none.
static bool use_ntap(const TcConvArgs& a) {
  const int npad = (a.cout + 15) / 16 * 16;
  const bool ok = a.k >= 2 && a.k <= 8 && a.k * npad <= 256 && npad <= 64;
  if (a.flags & MPF_FLAG_NTAP_OFF) return false;
  if (a.flags & MPF_FLAG_NTAP_ON) return ok;
  return ok && a.k >= 5;
}

static cudaError_t launch_conv_ntap(const TcConvArgs& a, cudaStream_t s, int* grid_out) {
  ConvTcParams p{};
  p.P_tot = a.n_frag * a.gr * a.gc;
  p.gr = a.gr;
  p.gc = a.gc;
  p.out_vr = a.out_vr;
  p.out_vc = a.out_vc;
  p.cin = a.cin;
  p.cout = a.cout;
  p.npad = (a.cout + 15) / 16 * 16;
  p.k = a.k;
  p.shift_rows = a.shift * (a.gc + 1);
  p.n_cc = (a.cin + kKC - 1) / kKC;
  p.last_k8 = (a.cin - (p.n_cc - 1) * kKC + 7) / 8;
  p.act = a.act;
  p.round_out = a.round_out;
  p.dact = a.dact;
  p.bias = a.bias;
  p.mul_dact = a.mul_dact;
  p.base_mode = base_mode();
  p.nbox = 1;
  p.box_rows = 128;
  p.a_slot_bytes = 128 * 128;
  p.b_rows = p.npad;
  p.b_slot_bytes = (uint32_t)(p.npad * 128);
  p.stage_bytes = p.a_slot_bytes + (uint32_t)a.k * p.b_slot_bytes;
  const size_t xbytes = 2 * 4 * 7 * 8 * 16 * 4;
  const size_t base_fixed = 1024 + xbytes + 4 * 256 + 512;
  const size_t total = 227 * 1024;
  int ns = 0, nst = 0;
  for (int cand_ns = 2; cand_ns >= 1 && !ns; --cand_ns) {
    const size_t budget = total - base_fixed - (size_t)cand_ns * kEpiWarps * kStageBytes;
    int cand = (int)(budget / p.stage_bytes);
    if (cand > 6) cand = 6;
    if (cand >= 3 || (cand_ns == 1 && cand >= 2)) {
      ns = cand_ns;
      nst = cand;
    }
  }
  if (!ns) return cudaErrorInvalidConfiguration;
  p.n_stage = ns;
  p.n_stages = nst;
  const int N = a.k * p.npad;
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * N)) cols <<= 1;
  p.tmem_cols = cols;
  const int TR = 128 - (a.k - 1);
  p.n_tiles = (p.P_tot + TR - 1) / TR;
  const size_t smem = base_fixed + (size_t)ns * kEpiWarps * kStageBytes + (size_t)nst * p.stage_bytes;
  const int grid = p.n_tiles < num_sms() ? p.n_tiles : num_sms();
  if (grid_out) *grid_out = grid;
  CUtensorMap A, B, O, O3;
  cudaError_t e = make_map(&A, a.x, (uint64_t)a.cin, (uint64_t)p.P_tot, 128u);
  if (e != cudaSuccess) return e;
  e = make_map(&B, a.w, (uint64_t)a.k * a.k * a.cin, (uint64_t)a.cout, (uint32_t)p.b_rows);
  if (e != cudaSuccess) return e;
  e = make_map(&O, a.out, (uint64_t)a.cout, (uint64_t)p.P_tot, 32u);
  if (e != cudaSuccess) return e;
  e = make_map(&O3, a.out, (uint64_t)a.cout, (uint64_t)p.P_tot, (uint32_t)(32 - (a.k - 1)));
  if (e != cudaSuccess) return e;
  // weight multicast across a cluster of two (MPF_FLAG_NTAP_NO_MC turns it off)
  const bool mc = !(a.flags & MPF_FLAG_NTAP_NO_MC) && p.n_tiles >= 2;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e2 != cudaSuccess) return e2;
    if (!mc) {
      kern<<<grid, kThreads, smem, s>>>(A, B, O, O3, p);
    } else {
      const int units = (p.n_tiles + 1) / 2;
      const int pairs = units < num_sms() / 2 ? units : num_sms() / 2;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * pairs, 1, 1);
      cfg.blockDim = dim3(kThreads, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = s;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      e2 = cudaLaunchKernelEx(&cfg, kern, A, B, O, O3, p);
      if (e2 != cudaSuccess) return e2;
    }
    return cudaGetLastError();
  };
#define MPF_NTAP_CASE(KK) \
  case KK: return mc ? go(conv_tc_ntap_kernel<KK, true>) : go(conv_tc_ntap_kernel<KK, false>);
  switch (a.k) {
    MPF_NTAP_CASE(2)
    MPF_NTAP_CASE(3)
    MPF_NTAP_CASE(4)
    MPF_NTAP_CASE(5)
    MPF_NTAP_CASE(6)
    MPF_NTAP_CASE(7)
    default: return mc ? go(conv_tc_ntap_kernel<8, true>) : go(conv_tc_ntap_kernel<8, false>);
  }
#undef MPF_NTAP_CASE
}

cudaError_t launch_conv_tc(const TcConvArgs& a, cudaStream_t s, int* grid_out) {
  if (use_ntap(a)) return launch_conv_ntap(a, s, grid_out);
  ConvTcParams p{};
  p.P_tot = a.n_frag * a.gr * a.gc;
  p.gr = a.gr;
  p.gc = a.gc;
  p.out_vr = a.out_vr;
  p.out_vc = a.out_vc;
  p.cin = a.cin;
  p.cout = a.cout;
  p.npad = (a.cout + 15) / 16 * 16;
  p.k = a.k;
  p.shift_rows = a.shift * (a.gc + 1);
  p.n_cc = (a.cin + kKC - 1) / kKC;
  p.last_k8 = (a.cin - (p.n_cc - 1) * kKC + 7) / 8;
  p.act = a.act;
  p.round_out = a.round_out;
  p.dact = a.dact;
  p.bias = a.bias;
  p.mul_dact = a.mul_dact;
  p.base_mode = base_mode();
  p.prof = prof_counters(a.flags);
  if (a.head_z) {
    if (a.head_C < 1 || a.head_C > kMaxHeadC || !a.head_w) return cudaErrorInvalidValue;
    p.head_w = a.head_w;
    p.head_z = a.head_z;
    p.head_C = a.head_C;
  }
  int nacc = 256 / p.npad;  // two accumulator sets in 512 TMEM columns
  if (nacc > 4) nacc = 4;
  if (nacc < 1) nacc = 1;
  auto set_nacc = [&](int na) {
    const int rows_needed = na * 128 + a.k - 1;
    p.nbox = (rows_needed + 255) / 256;
    p.box_rows = ((rows_needed + p.nbox - 1) / p.nbox + 7) / 8 * 8;
    p.a_slot_bytes = (uint32_t)(p.nbox * p.box_rows * 128);
  };
  set_nacc(nacc);
  // shared memory: stages of [A slab | k weight taps] (2..4, as many as fit), epilogue
  // staging (two boxes per warp when 3 stages still fit, else one)
  const size_t base_fixed = 1024 + 4 * 256 + 512 + head_epi_bytes(p.head_z ? p.head_C : 0, p.npad);
  const size_t total = 227 * 1024;
  int ns = 0, nst = 0;
  auto plan_smem = [&](bool pr) {
    p.b_rows = pr ? p.npad / 2 : p.npad;  // a CTA of a pair stages half of every weight tile
    p.b_slot_bytes = (uint32_t)(p.b_rows * 128);
    p.stage_bytes = p.a_slot_bytes + (uint32_t)a.k * p.b_slot_bytes;
    ns = nst = 0;
    for (int cand_ns = 2; cand_ns >= 1 && !ns; --cand_ns) {
      const size_t budget = total - base_fixed - (size_t)cand_ns * kEpiWarps * kStageBytes;
      int cand = (int)(budget / p.stage_bytes);
      if (cand > 4) cand = 4;
      if (cand >= 3 || (cand_ns == 1 && cand >= 2)) {
        ns = cand_ns;
        nst = cand;
      }
    }
    return ns != 0;
  };
  // keep the preferred mode and give up accumulator depth first (a smaller A slab lets two
  // stages fit: measured faster than switching mode); then try the other mode
  bool pair = want_pair(p.npad, a.k * a.k * a.cin, a.flags);
  bool ok = false;
  for (int na = nacc; na >= 1 && !ok; --na) {
    set_nacc(na);
    if (plan_smem(pair)) {
      nacc = na;
      ok = true;
    }
  }
  for (int na = nacc; na >= 1 && !ok; --na) {
    set_nacc(na);
    if (plan_smem(!pair)) {
      nacc = na;
      pair = !pair;
      ok = true;
    }
  }
  if (!ok) return cudaErrorInvalidConfiguration;
  const int m_cta = nacc * 128;
  const size_t fixed = base_fixed + (size_t)ns * kEpiWarps * kStageBytes;
  p.n_stage = ns;
  p.n_stages = nst;
  uint32_t cols = 32;
  while (cols < (uint32_t)(2 * nacc * p.npad)) cols <<= 1;
  p.tmem_cols = cols;
  p.n_tiles = (p.P_tot + (pair ? 2 : 1) * m_cta - 1) / ((pair ? 2 : 1) * m_cta);
  const size_t smem = fixed + (size_t)nst * p.stage_bytes;
  const int pairs = p.n_tiles < num_sms() / 2 ? p.n_tiles : num_sms() / 2;
  if (grid_out) *grid_out = pair ? 2 * pairs : (p.n_tiles < num_sms() ? p.n_tiles : num_sms());
  CUtensorMap A, B, O;
  cudaError_t e = make_map(&A, a.x, (uint64_t)a.cin, (uint64_t)p.P_tot, (uint32_t)p.box_rows);
  if (e != cudaSuccess) return e;
  e = make_map(&B, a.w, (uint64_t)a.k * a.k * a.cin, (uint64_t)a.cout, (uint32_t)p.b_rows);
  if (e != cudaSuccess) return e;
  e = make_map(&O, a.out, (uint64_t)a.cout, (uint64_t)p.P_tot, 32u);
  if (e != cudaSuccess) return e;
  if (pair) {
    switch (nacc) {
      case 1: return launch_nacc<1, true>(A, B, O, p, smem, s);
      case 2: return launch_nacc<2, true>(A, B, O, p, smem, s);
      case 3: return launch_nacc<3, true>(A, B, O, p, smem, s);
      default: return launch_nacc<4, true>(A, B, O, p, smem, s);
    }
  }
  if (!(a.flags & MPF_FLAG_NTAP_NO_MC) && a.k >= 2 && p.n_tiles >= 2) {  // weight taps multicast over two CTAs
    switch (nacc) {
      case 1: return launch_nacc<1, false, true>(A, B, O, p, smem, s);
      case 2: return launch_nacc<2, false, true>(A, B, O, p, smem, s);
      case 3: return launch_nacc<3, false, true>(A, B, O, p, smem, s);
      default: return launch_nacc<4, false, true>(A, B, O, p, smem, s);
    }
  }
  switch (nacc) {
    case 1: return launch_nacc<1, false>(A, B, O, p, smem, s);
    case 2: return launch_nacc<2, false>(A, B, O, p, smem, s);
    case 3: return launch_nacc<3, false>(A, B, O, p, smem, s);
    default: return launch_nacc<4, false>(A, B, O, p, smem, s);
  }
}

// ============================================================================ wgrad
// dW[co][(ky,kx,ci)] = sum_p dY[p][co] * X[p + ky*gc + kx][ci]  (Alg. 2: the sum over
// every fragment and position is the K-reduction of this GEMM).
//
// M = 128 output channels (A = dY tile, MN-major: co contiguous, one TMA box of 32 co x R
// positions per 32-channel atom), N = 32 k (B = one X "slab" of R + 8 positions x 32
// input channels for one (ky, ci chunk); the k taps kx are k MN-atoms of that same slab,
// one row (128 B) apart: LBO = 128 B), K = positions, 8 per instruction.  A CTA owns G
// such (ky, ci-chunk) groups (G * 32k <= 512 TMEM columns) of one 128-channel tile, and
// one contiguous split of the positions; its partial sums go to part[split] and a
// fixed-order reduction adds them to the gradient (deterministic, no atomics).
namespace {

constexpr int kWR = 64;  // positions per stage

struct WgTcParams {
  int P_tot, gc, cin, cout, k, n_cc, n_groups, G, n_sets, m_tiles;
  int chunk_stages;      // stages (of kWR positions) per split
  float* part;           // [splits][cout][k*k*cin]
  uint32_t a_bytes, b_bytes, stage_bytes;
  int n_stages_ring;
  uint32_t tmem_cols;
};

// CS > 1: the CS group sets of one split run as a cluster; each CTA loads 1/CS of the dY
// tile and multicasts it to all of them (the tile is read from L2 once per split instead of
// CS times), and a stage slot is refilled only when every CTA's MMAs have released it.
template <int MT, int CS>  // MT: output channels per tile, 128, or 64 (M = 64 MMA) when C_out <= 64
__global__ void __launch_bounds__(kThreads, 1)
    wgrad_tc_kernel(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX, WgTcParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sBar = sbase + p.n_stages_ring * p.stage_bytes;
  const uint32_t barFull = sBar, barEmpty = sBar + 8 * p.n_stages_ring, barT = sBar + 16 * p.n_stages_ring;
  const uint32_t sTmemSlot = barT + 8;
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (sTmemSlot - ptx::smem_u32(smem_raw)));
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  // block -> (m tile, group set, split); neighbouring blocks share a split (L2 reuse)
  const int mt = blockIdx.x % p.m_tiles;
  const int set = (blockIdx.x / p.m_tiles) % p.n_sets;
  const int split = blockIdx.x / (p.m_tiles * p.n_sets);
  // groups are spread evenly over the sets (equal MMA work per CTA keeps the sets of a
  // split in lockstep, so their shared dY / X tiles are L2 hits)
  const int g0 = (int)((long long)set * p.n_groups / p.n_sets);
  const int G = (int)((long long)(set + 1) * p.n_groups / p.n_sets) - g0;
  const int N = 32 * p.k;
  const long long pbeg = (long long)split * p.chunk_stages * kWR;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmD);
    ptx::prefetch_tmap(&tmX);
    for (int i = 0; i < p.n_stages_ring; ++i) {
      ptx::mbar_init(barFull + 8 * i, 1);
      ptx::mbar_init(barEmpty + 8 * i, CS);
    }
    ptx::mbar_init(barT, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(sTmemSlot, p.tmem_cols);
  ptx::tc_fence_before();
  if (CS > 1) ptx::cluster_sync_all();  // every CTA's barriers exist before anything is multicast
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  const int n_st = p.chunk_stages;
  const int rank = CS > 1 ? (int)ptx::cluster_rank() : 0;

  if (warp == 0) {
    if (lane == 0) {
      for (int st = 0; st < n_st; ++st) {
        const int slot = st % p.n_stages_ring;
        ptx::mbar_wait(barEmpty + 8 * slot, ((st / p.n_stages_ring) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(barFull + 8 * slot, p.a_bytes + G * p.b_bytes);
        const uint32_t sa = sbase + slot * p.stage_bytes;
        const int row = (int)(pbeg + (long long)st * kWR);
        for (int j = 0; j < MT / 32; ++j) {  // atoms of 32 output channels
          if (CS > 1) {
            if (j % CS == rank)
              ptx::tma_load_2d_mc(sa + j * kWR * 128, &tmD, barFull + 8 * slot, mt * MT + j * 32, row,
                                  (uint16_t)((1u << CS) - 1u));
          } else {
            ptx::tma_load_2d(sa + j * kWR * 128, &tmD, barFull + 8 * slot, mt * MT + j * 32, row);
          }
        }
        for (int g = 0; g < G; ++g) {
          const int ng = g0 + g, ky = ng / p.n_cc, cc = ng % p.n_cc;
          ptx::tma_load_2d(sa + p.a_bytes + g * p.b_bytes, &tmX, barFull + 8 * slot, cc * kKC, row + ky * p.gc);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = ptx::idesc_tf32_mn(MT, N);
    for (int st = 0; st < n_st; ++st) {
      const int slot = st % p.n_stages_ring;
      ptx::mbar_wait(barFull + 8 * slot, (st / p.n_stages_ring) & 1);
      ptx::tc_fence_after();
      const uint32_t sa = sbase + slot * p.stage_bytes;
      const uint64_t ad0 = ptx::sdesc_mn_sw128_32b(sa, kWR * 128, 512);
      const uint64_t bd0 = ptx::sdesc_mn_sw128_32b(sa + p.a_bytes, 128, 512);
      for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int r8 = 0; r8 < kWR / 8; ++r8) {
          const uint64_t ad = ad0 + (uint64_t)((r8 * 1024) >> 4);
          const uint64_t bd = bd0 + (uint64_t)((g * p.b_bytes + r8 * 1024) >> 4);
          ptx::mma_tf32_elect(tmem + g * N, ad, bd, idesc, (st | r8) != 0);
        }
      }
      if (CS > 1) ptx::mma_commit_mc_elect(barEmpty + 8 * slot, (uint16_t)((1u << CS) - 1u));  // frees the slot in every CTA
      else ptx::mma_commit_elect(barEmpty + 8 * slot);
    }
    ptx::mma_commit_elect(barT);
  } else {
    // TMEM lane quarter q; with M = 64 the accumulator rows sit in lanes 0-15 of each
    // quarter (row r -> lane 32 (r / 16) + r % 16).  The two warps of a quarter split the
    // 16-column chunks.
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int co = MT == 128 ? mt * 128 + q * 32 + lane : mt * 64 + q * 16 + lane;
    const bool row_ok = (MT == 128 || lane < 16) && co < p.cout;
    ptx::mbar_wait(barT, 0);
    ptx::tc_fence_after();
    const int K = p.k * p.k * p.cin;
    float* dst = p.part + ((long long)split * p.cout + (row_ok ? co : 0)) * K;
    for (int g = 0; g < G; ++g) {
      const int ng = g0 + g, ky = ng / p.n_cc, cc = ng % p.n_cc;
      for (int c0 = half * 16; c0 < N; c0 += 32) {
        float v[16];
        ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + g * N + c0, v);
        if (row_ok) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = c0 + j, kx = n / 32, ci = cc * kKC + (n % 32);
            if (ci < p.cin) dst[(ky * p.k + kx) * p.cin + ci] = n_st > 0 ? v[j] : 0.f;
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  if (CS > 1) ptx::cluster_sync_all();  // peers may still multicast into / arrive on our smem
  else __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, p.tmem_cols);
}


// The weight gradient of a layer with 128 < C_out <= 256 (FC1 of the cfg4 net, C_out = 200)
// on CTA pairs: tcgen05.mma.cta_group::2 with M = 256 output channels (CTA r stages the dY
// tile of channels 128 r .. 128 r + 127) and N = 2 x 32 k: the two halves of N come from the
// two CTAs' shared memory at the same offset, so each CTA stages the X slab of ONE group
// (ky, channel chunk) and one MMA covers the taps of two groups.  Against two M = 128 CTAs
// (one per channel half) this reads each X slab once per pair instead of twice and doubles
// the work per A fetch (N 96 -> 192 for k = 3), so the shared-memory port feeds a fuller
// tensor pipe.  Same sums per group as wgrad_tc_kernel in the same K order.
struct WgPairParams {
  int P_tot, gc, cin, cout, k, n_cc, n_groups, n_pairs, G2, n_sets;
  int chunk_stages;
  float* part;
  uint32_t a_bytes, b_bytes, stage_bytes;
  int n_stages_ring;
  uint32_t tmem_cols;
};

__global__ void __launch_bounds__(kThreads, 1)
    wgrad_tc_pair_kernel(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX,
                         WgPairParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sBar = sbase + p.n_stages_ring * p.stage_bytes;
  const uint32_t barFull = sBar, barEmpty = sBar + 8 * p.n_stages_ring, barT = sBar + 16 * p.n_stages_ring;
  const uint32_t sTmemSlot = barT + 8;
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (sTmemSlot - ptx::smem_u32(smem_raw)));
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_rank();
  const bool leader = rank == 0;
  // cluster -> (group-pair set, split); neighbouring clusters share a split (L2 reuse)
  const int cl = (int)(blockIdx.x >> 1);
  const int set = cl % p.n_sets, split = cl / p.n_sets;
  const int q0 = (int)((long long)set * p.n_pairs / p.n_sets);
  const int G2 = (int)((long long)(set + 1) * p.n_pairs / p.n_sets) - q0;
  const int N = 32 * p.k, N2 = 2 * N;
  const long long pbeg = (long long)split * p.chunk_stages * kWR;
  const uint32_t barFullL = ptx::mapa(barFull, 0);

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmD);
    ptx::prefetch_tmap(&tmX);
    for (int i = 0; i < p.n_stages_ring; ++i) {
      ptx::mbar_init(barFull + 8 * i, 1);
      ptx::mbar_init(barEmpty + 8 * i, 1);
    }
    ptx::mbar_init(barT, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc_pair(sTmemSlot, p.tmem_cols);
  ptx::tc_fence_before();
  ptx::cluster_sync_all();  // barrier inits and TMEM allocation visible to the peer
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  const int n_st = p.chunk_stages;

  if (warp == 0) {
    if (lane == 0) {
      for (int st = 0; st < n_st; ++st) {
        const int slot = st % p.n_stages_ring;
        ptx::mbar_wait(barEmpty + 8 * slot, ((st / p.n_stages_ring) & 1) ^ 1);
        if (leader) ptx::mbar_arrive_expect_tx(barFull + 8 * slot, 2u * (p.a_bytes + G2 * p.b_bytes));
        const uint32_t sa = sbase + slot * p.stage_bytes;
        const uint32_t bar = barFullL + 8 * slot;
        const int row = (int)(pbeg + (long long)st * kWR);
        for (int j = 0; j < 4; ++j)  // this CTA's 128 output channels: 4 atoms of 32
          ptx::tma_load_2d_pair(sa + j * kWR * 128, &tmD, bar, 128 * (int)rank + 32 * j, row);
        for (int gp = 0; gp < G2; ++gp) {
          int ng = 2 * (q0 + gp) + (int)rank;
          if (ng >= p.n_groups) ng = 0;  // odd group count: the pair's second half is discarded
          const int ky = ng / p.n_cc, cc = ng % p.n_cc;
          ptx::tma_load_2d_pair(sa + p.a_bytes + gp * p.b_bytes, &tmX, bar, cc * kKC, row + ky * p.gc);
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = ptx::idesc_tf32_mn(256, N2);
    for (int st = 0; leader && st < n_st; ++st) {
      const int slot = st % p.n_stages_ring;
      ptx::mbar_wait(barFull + 8 * slot, (st / p.n_stages_ring) & 1);
      ptx::tc_fence_after();
      const uint32_t sa = sbase + slot * p.stage_bytes;
      const uint64_t ad0 = ptx::sdesc_mn_sw128_32b(sa, kWR * 128, 512);
      const uint64_t bd0 = ptx::sdesc_mn_sw128_32b(sa + p.a_bytes, 128, 512);
      for (int gp = 0; gp < G2; ++gp) {
#pragma unroll
        for (int r8 = 0; r8 < kWR / 8; ++r8) {
          const uint64_t ad = ad0 + (uint64_t)((r8 * 1024) >> 4);
          const uint64_t bd = bd0 + (uint64_t)((gp * p.b_bytes + r8 * 1024) >> 4);
          ptx::mma_tf32_pair_elect(tmem + gp * N2, ad, bd, idesc, (st | r8) != 0);
        }
      }
      ptx::mma_commit_pair_elect(barEmpty + 8 * slot, 3);  // frees the slot in both CTAs
    }
    if (leader) ptx::mma_commit_pair_elect(barT, 3);
  } else {
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int co = 128 * (int)rank + q * 32 + lane;
    const bool row_ok = co < p.cout;
    ptx::mbar_wait(barT, 0);
    ptx::tc_fence_after();
    const int K = p.k * p.k * p.cin;
    float* dst = p.part + ((long long)split * p.cout + (row_ok ? co : 0)) * K;
    for (int gp = 0; gp < G2; ++gp) {
      for (int c0 = half * 16; c0 < N2; c0 += 32) {
        float v[16];
        ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + gp * N2 + c0, v);
        const int ng = 2 * (q0 + gp) + (c0 >= N ? 1 : 0);
        if (row_ok && ng < p.n_groups) {
          const int ky = ng / p.n_cc, cc = ng % p.n_cc;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int n = (c0 % N) + j, kx = n / 32, ci = cc * kKC + (n % 32);
            if (ci < p.cin) dst[(ky * p.k + kx) * p.cin + ci] = n_st > 0 ? v[j] : 0.f;
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync_all();  // the peer may still signal our barriers until here
  if (warp == 1) ptx::tmem_dealloc_pair(tmem, p.tmem_cols);
}


// The weight gradient of a narrow layer (C_out <= 64) with the roles swapped: M = 128 rows
// = 4 "atoms" of 32 input channels, each atom one tap (ky, kx) of one channel chunk, read
// straight out of the X slab of its (ky, chunk) group (an atom is the slab shifted by kx
// rows: the slab trick on the M side), N = C_out (the dY tile, MN-major), K = positions.
// With C_out on M (wgrad_tc_kernel<64>) an M = 64 MMA uses half of the tensor datapath;
// here every MMA has M = 128 and the whole tap set of a position split fits in TMEM
// (T M-tiles x N <= 512 columns), so one CTA per split reads dY and X once.  M-tiles: for
// every group, runs of 4 consecutive taps (LBO = one 128-B row); the k mod 4 remaining taps
// are tiled across groups (LBO = one slab), the last tile possibly partial (its phantom
// atoms read other shared memory and are discarded).  Same products as wgrad_tc_kernel,
// summed in the same K order per split.
constexpr int kSwapMaxTiles = 16;
constexpr int kSwapMaxPass = 4;
struct WgSwapParams {
  int P_tot, gc, cin, cout, npad, k, n_cc;
  int n_pass;  // passes over disjoint (ky, channel chunk) group ranges; CTA = (split, pass)
  int chunk_stages;
  float* part;
  uint32_t a_bytes, b_bytes, stage_bytes;  // a = the dY tile, b = one X slab; stage: the largest pass's
  int n_stages_ring;
  uint32_t tmem_cols;  // the largest pass's
  // per pass: first group (its slabs are groups g_lo .. g_lo + n_groups - 1) and its M-tiles:
  // first atom (local group, tap) and the atom stride (0: taps of one group, 1: groups)
  int g_lo[kSwapMaxPass], n_groups[kSwapMaxPass], n_tiles[kSwapMaxPass];
  int t_group[kSwapMaxPass][kSwapMaxTiles], t_tap[kSwapMaxPass][kSwapMaxTiles], t_across[kSwapMaxPass][kSwapMaxTiles];
};

__global__ void __launch_bounds__(kThreads, 1)
    wgrad_tc_swap_kernel(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX,
                         WgSwapParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  // ring of stages [X slabs of every group | dY tile], then 3 spare slabs (phantom atoms of a
  // partial M-tile read there), then the barriers
  const uint32_t sBar = sbase + p.n_stages_ring * p.stage_bytes + 3 * p.b_bytes;
  const uint32_t barFull = sBar, barEmpty = sBar + 8 * p.n_stages_ring, barT = sBar + 16 * p.n_stages_ring;
  const uint32_t sTmemSlot = barT + 8;
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (sTmemSlot - ptx::smem_u32(smem_raw)));
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  // the passes of one position split are adjacent CTAs: they stream the same dY / X rows at
  // about the same time, so a pass's re-read of dY is served by L2
  const int pass = blockIdx.x % p.n_pass, split = blockIdx.x / p.n_pass;
  const int g_lo = p.g_lo[pass], n_groups = p.n_groups[pass], n_tiles = p.n_tiles[pass];
  const long long pbeg = (long long)split * p.chunk_stages * kWR;
  const uint32_t slabs_bytes = (uint32_t)n_groups * p.b_bytes;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmD);
    ptx::prefetch_tmap(&tmX);
    for (int i = 0; i < p.n_stages_ring; ++i) {
      ptx::mbar_init(barFull + 8 * i, 1);
      ptx::mbar_init(barEmpty + 8 * i, 1);
    }
    ptx::mbar_init(barT, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(sTmemSlot, p.tmem_cols);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  const int n_st = p.chunk_stages;
  const int n_datoms = (p.npad + 31) / 32;

  if (warp == 0) {
    if (lane == 0) {
      for (int st = 0; st < n_st; ++st) {
        const int slot = st % p.n_stages_ring;
        ptx::mbar_wait(barEmpty + 8 * slot, ((st / p.n_stages_ring) & 1) ^ 1);
        ptx::mbar_arrive_expect_tx(barFull + 8 * slot, p.a_bytes + slabs_bytes);
        const uint32_t sa = sbase + slot * p.stage_bytes;
        const int row = (int)(pbeg + (long long)st * kWR);
        for (int g = 0; g < n_groups; ++g) {
          const int ky = (g_lo + g) / p.n_cc, cc = (g_lo + g) % p.n_cc;
          ptx::tma_load_2d(sa + g * p.b_bytes, &tmX, barFull + 8 * slot, cc * kKC, row + ky * p.gc);
        }
        for (int j = 0; j < n_datoms; ++j)
          ptx::tma_load_2d(sa + slabs_bytes + j * kWR * 128, &tmD, barFull + 8 * slot, j * 32, row);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = ptx::idesc_tf32_mn(128, p.npad);
    for (int st = 0; st < n_st; ++st) {
      const int slot = st % p.n_stages_ring;
      ptx::mbar_wait(barFull + 8 * slot, (st / p.n_stages_ring) & 1);
      ptx::tc_fence_after();
      const uint32_t sa = sbase + slot * p.stage_bytes;
      const uint64_t bd0 = ptx::sdesc_mn_sw128_32b(sa + slabs_bytes, kWR * 128, 512);
      for (int t = 0; t < n_tiles; ++t) {
        const uint32_t a0 = sa + p.t_group[pass][t] * p.b_bytes + p.t_tap[pass][t] * 128;
        const uint64_t ad0 = ptx::sdesc_mn_sw128_32b(a0, p.t_across[pass][t] ? p.b_bytes : 128u, 512);
#pragma unroll
        for (int r8 = 0; r8 < kWR / 8; ++r8) {
          const uint64_t ad = ad0 + (uint64_t)((r8 * 1024) >> 4);
          const uint64_t bd = bd0 + (uint64_t)((r8 * 1024) >> 4);
          ptx::mma_tf32_elect(tmem + t * p.npad, ad, bd, idesc, (st | r8) != 0);
        }
      }
      ptx::mma_commit_elect(barEmpty + 8 * slot);
    }
    ptx::mma_commit_elect(barT);
  } else {
    // TMEM lane quarter q = atom q of every M-tile; lane = input channel within the atom's chunk;
    // the two warps of a quarter split the C_out columns in 16-column halves
    const int q = warp & 3, half = (warp - 2) >> 2;
    ptx::mbar_wait(barT, 0);
    ptx::tc_fence_after();
    const int K = p.k * p.k * p.cin;
    for (int t = 0; t < n_tiles; ++t) {
      const int g = p.t_across[pass][t] ? p.t_group[pass][t] + q : p.t_group[pass][t];
      const int kx = p.t_across[pass][t] ? p.t_tap[pass][t] : p.t_tap[pass][t] + q;
      const bool atom_ok = g < n_groups && kx < p.k;  // warp-uniform
      const int ky = atom_ok ? (g_lo + g) / p.n_cc : 0, cc = atom_ok ? (g_lo + g) % p.n_cc : 0;
      const int ci = cc * kKC + lane;
      const bool ok = atom_ok && ci < p.cin;
      float* dst = p.part + (long long)split * p.cout * K + (ky * p.k + kx) * p.cin + (ok ? ci : 0);
      for (int c0 = half * 16; c0 < p.npad; c0 += 32) {
        float v[16];
        ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + t * p.npad + c0, v);
        if (ok) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int co = c0 + j;
            if (co < p.cout) dst[(long long)co * K] = n_st > 0 ? v[j] : 0.f;
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, p.tmem_cols);
}

}  // namespace

cudaError_t make_tmap_f32(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                          const uint32_t* box, bool sw128) {
  cudaError_t e = get_encoder();
  if (e != cudaSuccess) return e;
  cuuint64_t d[5], st[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    bx[i] = box[i];
    es[i] = 1;
    if (i + 1 < rank) st[i] = strides[i];
  }
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), d, st, bx, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

bool tc_wgrad_supported(int cin, int cout, int k) {
  return cin % 4 == 0 && cin >= 8 && cout % 4 == 0 && cout <= 256 && k >= 1 && k <= 8;
}

static bool wgrad_pair_ok(const TcWgradArgs& a) {
  return !(a.flags & MPF_FLAG_TC_SINGLE) && a.cout > 128 && a.cout <= 256 && 64 * a.k <= 256 && a.k * a.cin > 32;
}

// Split-K count of a tensor-core weight gradient.  The tensor core adds every K step's
// products into the fp32 accumulator without rounding to nearest, so the error of a sum grows
// with the length of the accumulation chain: on cfg4's FC1 weight gradient (7.1 M positions)
// one wave of 24 splits (296 K positions per chain) is 2.06e-3 from the fp64 oracle, 48 / 96 /
// 192 splits are 1.03e-3 / 5.3e-4 / 3.1e-4 (profiles/r2/wgrad_chain_length_cfg4.log), at
// 5.07 / 5.05 / 5.11 / 5.29 ms.  Chains are therefore capped at kMaxChain positions: whole
// extra waves of splits (each ends in an fp32 partial; the fixed-order reduction adds the
// partials in round-to-nearest fp32), which also keeps the error independent of the batch size.
// 160 K positions (FC1 of cfg4: 48 splits, 1.03e-3) cost nothing in the overlapped step; 80 K
// (96 splits, 5.3e-4) cost 0.4-0.7 ms of its 54 (three interleaved bench runs each).
constexpr long long kMaxChain = 160 * 1024;
static int wgrad_splits(int one_wave, long long P_tot) {
  if (one_wave < 1) one_wave = 1;
  long long s = one_wave;
  const long long need = (P_tot + kMaxChain - 1) / kMaxChain;
  if (need > s) s = (need + one_wave - 1) / one_wave * one_wave;
  if (s > kMaxSplits) s = one_wave <= kMaxSplits ? (long long)(kMaxSplits / one_wave) * one_wave : kMaxSplits;
  return (int)s;
}

static cudaError_t launch_wgrad_pair(const TcWgradArgs& a, int* splits_out, cudaStream_t s) {
  WgPairParams p{};
  p.P_tot = a.n_frag * a.gr * a.gc;
  p.gc = a.gc;
  p.cin = a.cin;
  p.cout = a.cout;
  p.k = a.k;
  p.n_cc = (a.cin + kKC - 1) / kKC;
  p.n_groups = a.k * p.n_cc;
  p.n_pairs = (p.n_groups + 1) / 2;
  const int N2 = 64 * a.k;
  p.G2 = 512 / N2;
  if (p.G2 > p.n_pairs) p.G2 = p.n_pairs;
  p.n_sets = (p.n_pairs + p.G2 - 1) / p.G2;
  p.a_bytes = 4 * kWR * 128;
  p.b_bytes = (kWR + 8) * 128;
  p.stage_bytes = p.a_bytes + p.G2 * p.b_bytes;
  const size_t budget = 225 * 1024 - 1024 - 256;
  p.n_stages_ring = (int)(budget / p.stage_bytes);
  if (p.n_stages_ring > 4) p.n_stages_ring = 4;
  if (p.n_stages_ring < 2) return cudaErrorInvalidConfiguration;
  uint32_t cols = 32;
  while (cols < (uint32_t)(p.G2 * N2)) cols <<= 1;
  p.tmem_cols = cols;
  const long long total_stages = (p.P_tot + kWR - 1) / kWR;
  int splits = wgrad_splits(num_sms() / (2 * p.n_sets), p.P_tot);  // whole waves of co-resident CTA pairs
  const size_t K = (size_t)a.k * a.k * a.cin;
  while (splits > 1 && (size_t)splits * (a.cout * K + a.cout) > a.part_cap_floats) --splits;
  if (splits > total_stages) splits = (int)total_stages;
  p.chunk_stages = (int)((total_stages + splits - 1) / splits);
  splits = (int)((total_stages + p.chunk_stages - 1) / p.chunk_stages);
  p.part = a.part;
  *splits_out = splits;
  CUtensorMap D, X;
  cudaError_t e = make_map(&D, a.dy, (uint64_t)a.cout, (uint64_t)p.P_tot, (uint32_t)kWR,
                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (e != cudaSuccess) return e;
  e = make_map(&X, a.x, (uint64_t)a.cin, (uint64_t)p.P_tot, (uint32_t)(kWR + 8), CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (e != cudaSuccess) return e;
  const size_t smem = 1024 + (size_t)p.n_stages_ring * p.stage_bytes + 256;
  e = cudaFuncSetAttribute(wgrad_tc_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * splits * p.n_sets, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, wgrad_tc_pair_kernel, D, X, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// the M-tiles of the swapped-role plan over G groups (local group indices); returns the tile
// count, or -1 when more than kSwapMaxTiles
static int swap_tiles(int k, int G, WgSwapParams* p, int pass = 0) {
  int T = 0;
  for (int g = 0; g < G; ++g)
    for (int t0 = 0; t0 + 4 <= k; t0 += 4) {
      if (T == kSwapMaxTiles) return -1;
      if (p) { p->t_group[pass][T] = g; p->t_tap[pass][T] = t0; p->t_across[pass][T] = 0; }
      ++T;
    }
  for (int kx = k / 4 * 4; kx < k; ++kx)
    for (int g0 = 0; g0 < G; g0 += 4) {
      if (T == kSwapMaxTiles) return -1;
      if (p) { p->t_group[pass][T] = g0; p->t_tap[pass][T] = kx; p->t_across[pass][T] = 1; }
      ++T;
    }
  return T;
}

static uint32_t swap_stage_bytes(int G, int npad) {
  return (uint32_t)G * (kWR + 8) * 128 + (uint32_t)((npad + 31) / 32) * kWR * 128;
}
static size_t swap_budget() { return 225 * 1024 - 1024 - 256 - 3 * (kWR + 8) * 128; }

// The swapped-role plan: C_out <= 64, or 64 < C_out <= 96 where C_out on M would leave at least
// a quarter of every M = 128 tile empty.  A pass's tiles must fit TMEM (tiles x npad <= 512
// columns) with >= 2 pipeline stages of slabs; when all groups' tiles do not, the groups are
// split into passes (one launch each over the same position splits, with its own slabs and
// tiles, writing its own (tap, channel) columns of the partials; dY is re-read per pass).
// Narrow layers (C_out <= 64) keep the single pass.  Returns the groups per pass (0 = not
// applicable).
static int wgrad_swap_plan(const TcWgradArgs& a, WgSwapParams* p) {
  if ((a.flags & MPF_FLAG_WGRAD_M128) || a.cout > 96) return 0;
  const int n_cc = (a.cin + kKC - 1) / kKC, G = a.k * n_cc, npad = (a.cout + 15) / 16 * 16;
  int GP = 0;
  for (int gp = G; gp >= 1 && !GP; --gp) {
    const int T = swap_tiles(a.k, gp, nullptr);
    if (T < 1 || T * npad > 512) continue;
    if (swap_budget() / swap_stage_bytes(gp, npad) < 2) continue;
    GP = gp;
  }
  if (!GP) return 0;
  if (GP < G && a.cout <= 64) return 0;
  if ((G + GP - 1) / GP > kSwapMaxPass) return 0;
  p->npad = npad;
  p->n_cc = n_cc;
  return GP;
}

static cudaError_t launch_wgrad_swap(const TcWgradArgs& a, WgSwapParams& p, int GP, int* splits_out, cudaStream_t s) {
  p.P_tot = a.n_frag * a.gr * a.gc;
  p.gc = a.gc;
  p.cin = a.cin;
  p.cout = a.cout;
  p.k = a.k;
  const int G = a.k * p.n_cc;
  p.a_bytes = (uint32_t)((p.npad + 31) / 32) * kWR * 128;
  p.b_bytes = (kWR + 8) * 128;
  const long long total_stages = (p.P_tot + kWR - 1) / kWR;
  int splits = wgrad_splits(num_sms(), p.P_tot);
  const size_t K = (size_t)a.k * a.k * a.cin;
  while (splits > 1 && (size_t)splits * (a.cout * K + a.cout) > a.part_cap_floats) --splits;
  if (splits > total_stages) splits = (int)total_stages;
  p.chunk_stages = (int)((total_stages + splits - 1) / splits);
  splits = (int)((total_stages + p.chunk_stages - 1) / p.chunk_stages);
  p.part = a.part;
  *splits_out = splits;
  CUtensorMap D, X;
  cudaError_t e = make_map(&D, a.dy, (uint64_t)a.cout, (uint64_t)p.P_tot, (uint32_t)kWR,
                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (e != cudaSuccess) return e;
  e = make_map(&X, a.x, (uint64_t)a.cin, (uint64_t)p.P_tot, (uint32_t)(kWR + 8), CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (e != cudaSuccess) return e;
  // passes over disjoint groups (disjoint partial columns), launched together
  p.n_pass = 0;
  int max_tiles = 0;
  for (int g_lo = 0; g_lo < G; g_lo += GP) {
    const int q = p.n_pass++;
    p.g_lo[q] = g_lo;
    p.n_groups[q] = std::min(GP, G - g_lo);
    p.n_tiles[q] = swap_tiles(a.k, p.n_groups[q], &p, q);
    if (p.n_tiles[q] < 1) return cudaErrorInvalidConfiguration;
    max_tiles = std::max(max_tiles, p.n_tiles[q]);
  }
  p.stage_bytes = swap_stage_bytes(std::min(GP, G), p.npad);
  p.n_stages_ring = (int)(swap_budget() / p.stage_bytes);
  if (p.n_stages_ring > 4) p.n_stages_ring = 4;
  if (p.n_stages_ring < 2) return cudaErrorInvalidConfiguration;
  uint32_t cols = 32;
  while (cols < (uint32_t)(max_tiles * p.npad)) cols <<= 1;
  p.tmem_cols = cols;
  const size_t smem = 1024 + (size_t)p.n_stages_ring * p.stage_bytes + 3 * p.b_bytes + 256;
  e = cudaFuncSetAttribute(wgrad_tc_swap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  wgrad_tc_swap_kernel<<<splits * p.n_pass, kThreads, smem, s>>>(D, X, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return cudaSuccess;
}

cudaError_t launch_wgrad_tc(const TcWgradArgs& a, int* splits_out, cudaStream_t s) {
  if (wgrad_pair_ok(a)) return launch_wgrad_pair(a, splits_out, s);
  {
    WgSwapParams sp{};
    if (const int GP = wgrad_swap_plan(a, &sp)) return launch_wgrad_swap(a, sp, GP, splits_out, s);
  }
  WgTcParams p{};
  p.P_tot = a.n_frag * a.gr * a.gc;
  p.gc = a.gc;
  p.cin = a.cin;
  p.cout = a.cout;
  p.k = a.k;
  p.n_cc = (a.cin + kKC - 1) / kKC;
  p.n_groups = a.k * p.n_cc;
  const int N = 32 * a.k;
  p.G = 512 / N;
  if (p.G > p.n_groups) p.G = p.n_groups;
  p.n_sets = (p.n_groups + p.G - 1) / p.G;
  const int MT = (a.cout <= 64 && !(a.flags & MPF_FLAG_WGRAD_M128)) ? 64 : 128;
  p.m_tiles = (a.cout + MT - 1) / MT;
  p.a_bytes = (MT / 32) * kWR * 128;
  p.b_bytes = (kWR + 8) * 128;
  p.stage_bytes = p.a_bytes + p.G * p.b_bytes;
  const size_t budget = 225 * 1024 - 1024 - 256;
  p.n_stages_ring = (int)(budget / p.stage_bytes);
  if (p.n_stages_ring > 4) p.n_stages_ring = 4;
  if (p.n_stages_ring < 2) {  // shrink G until two stages fit
    while (p.G > 1 && 2 * (p.a_bytes + p.G * p.b_bytes) > budget) --p.G;
    p.n_sets = (p.n_groups + p.G - 1) / p.G;
    p.stage_bytes = p.a_bytes + p.G * p.b_bytes;
    p.n_stages_ring = 2;
  }
  uint32_t cols = 32;
  while (cols < (uint32_t)(p.G * N)) cols <<= 1;
  p.tmem_cols = cols;
  const long long total_stages = (p.P_tot + kWR - 1) / kWR;
  const int per_split_blocks = p.m_tiles * p.n_sets;
  int splits = wgrad_splits(num_sms() / per_split_blocks, p.P_tot);  // whole waves of co-resident CTAs
  const size_t K = (size_t)a.k * a.k * a.cin;
  while (splits > 1 && (size_t)splits * (a.cout * K + a.cout) > a.part_cap_floats) --splits;
  if (splits > total_stages) splits = (int)total_stages;
  p.chunk_stages = (int)((total_stages + splits - 1) / splits);
  splits = (int)((total_stages + p.chunk_stages - 1) / p.chunk_stages);
  p.part = a.part;
  *splits_out = splits;
  CUtensorMap D, X;
  cudaError_t e = make_map(&D, a.dy, (uint64_t)a.cout, (uint64_t)p.P_tot, (uint32_t)kWR,
                           CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (e != cudaSuccess) return e;
  e = make_map(&X, a.x, (uint64_t)a.cin, (uint64_t)p.P_tot, (uint32_t)(kWR + 8), CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  if (e != cudaSuccess) return e;
  const size_t smem = 1024 + (size_t)p.n_stages_ring * p.stage_bytes + 256;
  // pairs of group sets of a split share the dY tile through a cluster multicast (m_tiles == 1):
  // measured on cfg4's C3x3 96->128 weight gradient 2.96 -> 2.65 ms; one cluster of all four
  // sets of C5x5 64->96 was slower (5.0 -> 9.2 ms: four-way lockstep of uneven sets)
  const int cs = (p.m_tiles == 1 && p.n_sets % 2 == 0 && !(a.flags & MPF_FLAG_NTAP_NO_MC)) ? 2 : 1;
  auto pick = [&]() {
    if (MT == 64) return cs == 2 ? wgrad_tc_kernel<64, 2> : cs == 3 ? wgrad_tc_kernel<64, 3> : cs == 4 ? wgrad_tc_kernel<64, 4> : wgrad_tc_kernel<64, 1>;
    return cs == 2 ? wgrad_tc_kernel<128, 2> : cs == 3 ? wgrad_tc_kernel<128, 3> : cs == 4 ? wgrad_tc_kernel<128, 4> : wgrad_tc_kernel<128, 1>;
  };
  auto kern = pick();
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (cs == 1) {
    kern<<<splits * per_split_blocks, kThreads, smem, s>>>(D, X, p);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(splits * per_split_blocks, 1, 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, D, X, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace mpf
