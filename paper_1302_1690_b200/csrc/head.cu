// head.cu — the softmax FC (1x1, linear) + per-pixel softmax + class-weighted MCCE +
// dL/dx_hat, and the whole back-propagation through that layer, in one pass over the
// last hidden activation h ("first dL/dx_hat", 197 MCCE per pixel,
// 252 per-class weights; readings R8, R9, R15).
//
// Per position p (fragment-major; the label is fetched through the fragment -> pixel
// map, R2/R7; positions outside the O_H x O_W output grid and label 255 are ignored):
//     z = W_L h + b_L,  p = softmax(z),  loss += w_t (lse - z_t)
//     dz = w_t (p - onehot_t) / n_lab(img)
//     dh = (W_L^T dz) * act'(h)                 -> written (delta of the previous layer)
//     dW_L += dz h^T,  db_L += dz,  db_prev += dh   (Alg. 2: sums over all fragments)
// The three sums are per-block register partials finished by a fixed-order reduction,
// so the softmax layer needs no separate weight-gradient pass and the previous layer
// needs no separate bias pass.
//
// Schedule: persistent CTAs walk tiles of TP = 64 positions.  A tile of h is TP*Ch
// contiguous floats: one TMA bulk copy into a double-buffered shared buffer, issued one
// tile ahead; the labels of the tile are gathered while it lands.  Phase A: a warp
// computes 8 positions at once (4 lanes per position split the Ch-long dot products,
// rotated per position so the 8 rows hit distinct banks, and combine them with an xor
// butterfly that is bit-identical on the 4 lanes).  Phase B: thread = (channel ch,
// position stream); W_L[:, ch] sits in registers, dh is written coalesced and the
// dW/db partials accumulate in registers.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "head_common.cuh"
#include "mpf_internal.h"
#include "numerics.cuh"
#include "tc_ptx.cuh"

namespace mpf {

namespace {

constexpr int kTP = 64;  // positions per tile
constexpr int kThr = 256;
constexpr int kMaxC = 16;


__device__ __forceinline__ float act_der(int act, float y) {
  if (act == MPF_TANH) return 1.f - y * y;
  if (act == MPF_LOGISTIC) return y * (1.f - y);
  return 1.f;
}

__device__ __forceinline__ void named_bar_h(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// bytes of region0: two h tiles, or the end-of-kernel reduction area if larger
__host__ __device__ inline size_t head_region0(int C, int Ch) {
  const int nw = kThr / 32;
  const size_t red = sizeof(float) * ((size_t)nw * Ch * (C + 1) + (size_t)nw * kMaxC);
  const size_t tiles = 2 * (size_t)kTP * Ch * sizeof(float);
  return ((red > tiles ? red : tiles) + 127) / 128 * 128;
}

// VEC (Ch % 4 == 0): both phases work on float4 channel groups (LDS.128 / STG.128, one
// W_L row fetch per 4 channels), which halves the instruction count per element.
template <int NC, bool TRAIN, bool TANH, bool VEC>
__global__ void __launch_bounds__(kThr, 2) head_kernel(HeadArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int C = a.C, Ch = a.Ch;
  const size_t tile_bytes = (size_t)kTP * Ch * sizeof(float);
  // [2 mbarriers | pad | region0: two h tiles, later the reduction area | W | b | dl | lab]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  float* hb0 = reinterpret_cast<float*>(smem_raw + 128);
  float* hb1 = reinterpret_cast<float*>(smem_raw + 128 + tile_bytes);
  // W_L [C][Ch] (canonical): phase A reads it with 4 distinct addresses per warp, phase B
  // with consecutive channels per lane (conflict-free)
  float* s_w2 = reinterpret_cast<float*>(smem_raw + 128 + head_region0(C, Ch));
  float* s_b = s_w2 + ((C * Ch + 3) & ~3);  // 16-byte aligned (s_dl is read as float4)
  float* s_dl = s_b + kMaxC;                                  // [kTP][kNCP]
  int* s_lab = reinterpret_cast<int*>(s_dl + kTP * kMaxC);     // [kTP]
  const uint32_t bar0 = ptx::smem_u32(&bars[0]), bar1 = ptx::smem_u32(&bars[1]);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int e = tid; e < C * Ch; e += kThr) s_w2[e] = a.w[e];
  for (int e = tid; e < C; e += kThr) s_b[e] = a.b[e];
  const long long per_img = (long long)a.F * a.gr * a.gc;
  const int frag_sz = a.gr * a.gc;
  const int tpi = a.tiles_per_img;
  const long long total = (long long)a.n * tpi;
  if (tid == 0) {
    ptx::mbar_init(bar0, 1);
    ptx::mbar_init(bar1, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();

  auto issue = [&](long long tile, int buf) {
    const int img = (int)(tile / tpi), tt = (int)(tile % tpi);
    const long long p0 = (long long)tt * kTP;
    const long long np = min((long long)kTP, per_img - p0);
    const uint32_t bytes = (uint32_t)(np * Ch * sizeof(float));
    const uint32_t bar = buf ? bar1 : bar0;
    ptx::mbar_arrive_expect_tx(bar, bytes);
    ptx::bulk_load(ptx::smem_u32(buf ? hb1 : hb0), a.h + ((long long)img * per_img + p0) * Ch, bytes, bar);
  };

  // Every warp owns 8 positions of a tile: phase A maps 4 lanes to a position, phase B
  // maps lanes to channels; only the tile-buffer hand-off needs the whole block.
  const int pw0 = warp * 8;                       // first position of this warp
  const int pa = pw0 + (lane >> 2), qa = lane & 3;
  const int M = Ch >> 2;  // channels per lane in phase A (Ch % 4 == 0 path)
  const int rot = pa % (M > 0 ? M : 1);
  constexpr int kMC = 8;  // channel slots per lane in phase B (Ch <= 256)
  // VEC phase B: one float4 channel group per lane.  Ch > 128 (more than 32 groups): the
  // warps pair up — both warps of a pair walk the pair's 16 positions, warp w & 1 taking
  // channel groups 32 (w & 1) + lane (keeps the accumulators in registers).
  constexpr int kMG = 1;
  const bool pairB = VEC && Ch > 128;
  // dz rows in shared memory are padded to kNCP classes (float4 reads in phase B)
  constexpr int kNCP = (NC + 3) & ~3;
  float accW[VEC ? 1 : kMC][NC], accP[VEC ? 1 : kMC], accL[NC];
  float accW4[VEC ? kMG : 1][NC][4], accP4[VEC ? kMG : 1][4];
#pragma unroll
  for (int m = 0; m < (VEC ? kMG : 1); ++m)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      accP4[m][u] = 0.f;
#pragma unroll
      for (int c = 0; c < NC; ++c) accW4[m][c][u] = 0.f;
    }
  // W_L[:, ch] of this lane's phase-B channels, held in registers (constant over tiles)
  constexpr bool kWReg = !VEC && NC <= 4;
  float wreg[kWReg ? kMC : 1][kWReg ? NC : 1];
#pragma unroll
  for (int m = 0; m < (VEC ? 1 : kMC); ++m) {
    accP[m] = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) accW[m][c] = 0.f;
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) accL[c] = 0.f;
  __syncthreads();  // s_w is filled (the barrier init sync above precedes nothing else)
  // VEC: W_L[:, 4g..4g+3] of this lane's phase-B channel group, held in registers
  constexpr bool kW4Reg = VEC && NC <= 8;
  float4 w4reg[kW4Reg ? NC : 1];
  if constexpr (kW4Reg) {
    const int g = lane + (pairB ? 32 * (warp & 1) : 0);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      w4reg[c] = 4 * g < Ch ? reinterpret_cast<const float4*>(s_w2 + c * Ch)[g] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if constexpr (kWReg) {
#pragma unroll
    for (int m = 0; m < kMC; ++m) {
      const int ch = lane + 32 * m;
#pragma unroll
      for (int c = 0; c < NC; ++c) wreg[m][c] = ch < Ch ? s_w2[c * Ch + ch] : 0.f;
    }
  }

  // TMA bulk copies need 16-byte granules: Ch % 4 == 0; otherwise a plain cooperative copy
  const bool bulk = (Ch % 4) == 0;
  if (bulk && tid == 0 && blockIdx.x < total) issue(blockIdx.x, 0);
  int it = 0;
  for (long long tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
    const int cur = it & 1;
    const int img = (int)(tile / tpi), tt = (int)(tile % tpi);
    const long long p0 = (long long)tt * kTP;
    // ---------------------------------------------------------- phase 0: labels (lanes 0..7)
    if (lane < 8) {
      int lab;
      if (TRAIN && a.lab_frag) {  // pre-gathered in head-position order (launch_label_frag)
        const long long pos = p0 + pw0 + lane;
        lab = kLabBeyond;
        if (pos < per_img) {
          lab = a.lab_frag[(long long)img * per_img + pos];
          if (lab == kLabFragPad) lab = kLabPad;
        }
      } else {
        lab = head_label(a, img, p0 + pw0 + lane, per_img, frag_sz, TRAIN);
      }
      s_lab[pw0 + lane] = lab;
    }
    if (bulk) {
      ptx::mbar_wait(cur ? bar1 : bar0, (it >> 1) & 1);
      if (tid == 0 && tile + gridDim.x < total) issue(tile + gridDim.x, cur ^ 1);
    } else {
      float* dst = (cur ? hb1 : hb0) + pw0 * Ch;
      const long long np = min(8LL, per_img - p0 - pw0);
      const float* src = a.h + ((long long)img * per_img + p0 + pw0) * Ch;
      for (int e = lane; e < np * Ch; e += 32) dst[e] = src[e];
    }
    __syncwarp();
    const float* hs = cur ? hb1 : hb0;
    float lossv = 0.f;
    // ---------------------------------------------------------------- phase A
    {
      const int lab = s_lab[pa];
      const bool need = lab >= 0 && lab < C;
      float z[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) z[c] = 0.f;
      if (a.zpre) {  // logits from the last hidden layer's epilogue: every lane of the position loads them
        if (need) {
          const float* zr = a.zpre + ((long long)img * per_img + p0 + pa) * C;
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (c < C) z[c] = __ldg(zr + c);
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) z[c] += (c < C) ? s_b[c] : 0.f;
      } else {  // the logits from h: 4 lanes per position, each over a quarter of the channels
        if (need && VEC) {  // float4 channel groups g = qa, qa + 4, ...
          const float4* hrow4 = reinterpret_cast<const float4*>(hs + pa * Ch);
          const int G4 = Ch >> 2;
          for (int g = qa; g < G4; g += 4) {
            const float4 hv = hrow4[g];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const float4 w = reinterpret_cast<const float4*>(s_w2 + c * Ch)[g];
              z[c] = fmaf(w.x, hv.x, fmaf(w.y, hv.y, fmaf(w.z, hv.z, fmaf(w.w, hv.w, z[c]))));
            }
          }
        } else if (need) {  // uniform over the 4 lanes of a position
          const float* hrow = hs + pa * Ch;
          if (bulk) {
            for (int m = 0; m < M; ++m) {
              int mm = m + rot;
              if (mm >= M) mm -= M;
              const int ch = qa + 4 * mm;
              const float hv = hrow[ch];
#pragma unroll
              for (int c = 0; c < NC; ++c) z[c] = fmaf(s_w2[c * Ch + ch], hv, z[c]);
            }
          } else {
            for (int ch = qa; ch < Ch; ch += 4) {
              const float hv = hrow[ch];
#pragma unroll
              for (int c = 0; c < NC; ++c) z[c] = fmaf(s_w2[c * Ch + ch], hv, z[c]);
            }
          }
        }
        // 4-lane butterfly (the lanes of one position are lane^1, lane^2: same group);
        // executed by every lane of the warp
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          z[c] += __shfl_xor_sync(0xffffffffu, z[c], 1);
          z[c] += __shfl_xor_sync(0xffffffffu, z[c], 2);
          z[c] += (c < C) ? s_b[c] : 0.f;
        }
      }
      if (need) {
        float mx = z[0];
#pragma unroll
        for (int c = 1; c < NC; ++c)
          if (c < C) mx = fmaxf(mx, z[c]);
        float se = 0.f;
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if (c < C) se += expf(z[c] - mx);
        const float lse = mx + logf(se);
        if (!TRAIN) {
          const long long pos = p0 + pa;
          const int gl = (int)(pos / frag_sz);
          const int rem = (int)(pos - (long long)gl * frag_sz);
          const int i = rem / a.gc, j = rem - (rem / a.gc) * a.gc;
          const long long g = (long long)img * a.F + gl;
          float* pr = a.probs + ((g * a.vr + i) * a.vc + j) * C;
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (c < C && (c & 3) == qa) pr[c] = expf(z[c] - lse);
        } else {
          const int nl = a.nlab[img];
          const float wt = a.cw[lab];
          float zt = 0.f;
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (c == lab) zt = z[c];
          if (qa == 0) lossv = wt * (lse - zt);
          const float inv = nl > 0 ? wt / (float)nl : 0.f;
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if ((c & 3) == qa) {
              const float dz = (c < C) ? inv * (expf(z[c] - lse) - (c == lab ? 1.f : 0.f)) : 0.f;
              s_dl[pa * kNCP + c] = dz;
              accL[c] += dz;  // db_L: this lane owns class c of its positions
            }
        }
      }
    }
    if (TRAIN) {
      // per-(tile, warp) loss: fixed-order warp sum
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) lossv += __shfl_xor_sync(0xffffffffu, lossv, o);
      if (lane == 0) a.loss_part[((long long)img * tpi + tt) * (kThr / 32) + warp] = lossv;
      __syncwarp();
      // -------------------------------------------------------------- phase B
      float* dh_img = a.dh + ((long long)img * per_img + p0) * Ch;
      if (pairB) named_bar_h(1 + (warp >> 1), 64);  // the partner warp's dz rows are in s_dl
      const int pb0 = pairB ? (warp & ~1) * 8 : pw0;
      const int npb = pairB ? 16 : 8;
      const int gB = VEC ? lane + (pairB ? 32 * (warp & 1) : 0) : 0;  // this lane's float4 group
      if constexpr (VEC) {
        // float4 channel group gB per lane; lanes past the last group (Ch < 4 * 64) compute on
        // group 0 and skip their stores, so the loop body has no divergent branch; their
        // accumulators are never written out (the partials below test 4 * g < Ch).  Row
        // pointers advance by one position per iteration (no per-position address math).
        const bool lane_on = 4 * gB < Ch;
        const int stride4 = Ch >> 2;
        float4* dh4 = reinterpret_cast<float4*>(dh_img + pb0 * Ch) + (lane_on ? gB : 0);
        const float4* h4 = reinterpret_cast<const float4*>(hs + pb0 * Ch) + (lane_on ? gB : 0);
        const float4* w4s = reinterpret_cast<const float4*>(s_w2) + (lane_on ? gB : 0);
        // which of the npb positions are labelled (bit q) and how many lie before the end of
        // the image: one shared load and two ballots instead of a load and tests per position
        unsigned act_mask, in_mask;
        {
          const int lq = lane < npb ? s_lab[pb0 + lane] : kLabBeyond;
          act_mask = __ballot_sync(0xffffffffu, lq >= 0 && lq < C);
          in_mask = __ballot_sync(0xffffffffu, lq != kLabBeyond);
        }
        const int nq = __popc(in_mask);  // positions past the image end come last
        for (int q = 0; q < nq; ++q, dh4 += stride4, h4 += stride4) {
          if (!((act_mask >> q) & 1u)) {  // padding position or ignored label -> zero delta
            if (lane_on) *dh4 = make_float4(0.f, 0.f, 0.f, 0.f);
            continue;
          }
          float dl[NC];
          {  // the row of dz: kNCP / 4 broadcast LDS.128
            const float4* r4 = reinterpret_cast<const float4*>(s_dl + (pb0 + q) * kNCP);
#pragma unroll
            for (int j = 0; j < kNCP / 4; ++j) {
              const float4 v = r4[j];
              const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (4 * j + u < NC) dl[4 * j + u] = vv[u];
            }
          }
          const float4 hv = *h4;
          const float hh[4] = {hv.x, hv.y, hv.z, hv.w};
          float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const float4 w = kW4Reg ? w4reg[kW4Reg ? c : 0] : w4s[c * stride4];
            const float ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              sacc[u] = fmaf(ww[u], dl[c], sacc[u]);
              accW4[0][c][u] = fmaf(dl[c], hh[u], accW4[0][c][u]);
            }
          }
          float d[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            d[u] = sacc[u] * (TANH ? fmaf(-hh[u], hh[u], 1.f) : act_der(a.hidden_act, hh[u]));
            accP4[0][u] += d[u];
            if (a.round_tf32) d[u] = tf32_rn_sat(d[u]);
          }
          if (lane_on) *dh4 = make_float4(d[0], d[1], d[2], d[3]);
        }
      } else
      for (int q = 0; q < npb; ++q) {
        const int p = pb0 + q;
        const int lab = s_lab[p];  // warp-uniform
        if (lab == kLabBeyond) break;  // past the end of the image (and so are the rest)
        const bool act = lab >= 0 && lab < C;
        float dl[NC];
        if (act) {  // the row of dz: kNCP / 4 broadcast LDS.128
          const float4* r4 = reinterpret_cast<const float4*>(s_dl + p * kNCP);
#pragma unroll
          for (int j = 0; j < kNCP / 4; ++j) {
            const float4 v = r4[j];
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (4 * j + u < NC) dl[4 * j + u] = vv[u];
          }
        } else {
#pragma unroll
          for (int c = 0; c < NC; ++c) dl[c] = 0.f;
        }
        float* dh_row = dh_img + p * Ch;  // 32-bit offset: a tile is far below 2^31 elements
        if (!act) {  // warp-uniform: padding position or ignored label -> zero delta
          if (VEC) {
            if (4 * gB < Ch) reinterpret_cast<float4*>(dh_row)[gB] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
#pragma unroll
            for (int m = 0; m < kMC; ++m)
              if (lane + 32 * m < Ch) dh_row[lane + 32 * m] = 0.f;
          }
          continue;
        }
        if constexpr (VEC) {
#pragma unroll
          for (int m = 0; m < kMG; ++m) {
            const int g = gB;
            if (4 * g < Ch) {
              const float4 hv = reinterpret_cast<const float4*>(hs + p * Ch)[g];
              const float hh[4] = {hv.x, hv.y, hv.z, hv.w};
              float sacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
              for (int c = 0; c < NC; ++c) {
                const float4 w = kW4Reg ? w4reg[kW4Reg ? c : 0] : reinterpret_cast<const float4*>(s_w2 + c * Ch)[g];
                const float ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  sacc[u] = fmaf(ww[u], dl[c], sacc[u]);
                  accW4[m][c][u] = fmaf(dl[c], hh[u], accW4[m][c][u]);
                }
              }
              float d[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                d[u] = sacc[u] * (TANH ? fmaf(-hh[u], hh[u], 1.f) : act_der(a.hidden_act, hh[u]));
                accP4[m][u] += d[u];
                if (a.round_tf32) d[u] = tf32_rn_sat(d[u]);
              }
              reinterpret_cast<float4*>(dh_row)[g] = make_float4(d[0], d[1], d[2], d[3]);
            }
          }
          continue;
        }
#pragma unroll
        for (int m = 0; m < kMC; ++m) {
          const int ch = lane + 32 * m;
          if (ch < Ch) {
            const float hv = hs[p * Ch + ch];
            float sacc = 0.f;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const float w = kWReg ? wreg[kWReg ? m : 0][kWReg ? c : 0] : s_w2[c * Ch + ch];
              sacc = fmaf(w, dl[c], sacc);
              accW[VEC ? 0 : m][c] = fmaf(dl[c], hv, accW[VEC ? 0 : m][c]);
            }
            const float d = sacc * (TANH ? fmaf(-hv, hv, 1.f) : act_der(a.hidden_act, hv));
            accP[VEC ? 0 : m] += d;
            dh_row[ch] = a.round_tf32 ? tf32_rn_sat(d) : d;
          }
        }
      }
    }
    __syncthreads();  // every warp is done with this tile buffer before it is refilled
  }
  if (!TRAIN) return;
  // ------------------------------------------------------------------ block partials
  // red[warp][ch][0..C) = accW, red[warp][ch][C] = accP; redL[warp][c] = accL (lane 0)
  float* red = hb0;  // tiles are no longer needed
  const int RW = C + 1;
  if constexpr (VEC) {
#pragma unroll
    for (int m = 0; m < kMG; ++m) {
      const int g = lane + (pairB ? 32 * (warp & 1) : 0);
      if (4 * g < Ch) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (c < C) red[(warp * Ch + 4 * g + u) * RW + c] = accW4[m][c][u];
          red[(warp * Ch + 4 * g + u) * RW + C] = accP4[m][u];
        }
      }
    }
  } else {
#pragma unroll
    for (int m = 0; m < kMC; ++m) {
      const int ch = lane + 32 * m;
      if (ch < Ch) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if (c < C) red[(warp * Ch + ch) * RW + c] = accW[m][c];
        red[(warp * Ch + ch) * RW + C] = accP[m];
      }
    }
  }
  float* redL = red + (kThr / 32) * Ch * RW;
  // db_L: class c was accumulated by the lanes with (lane & 3) == (c & 3); fixed-order
  // butterfly over the lanes (the other lanes hold zeros for c)
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) accL[c] += __shfl_xor_sync(0xffffffffu, accL[c], o);
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c < C) redL[warp * kMaxC + c] = accL[c];
  }
  __syncthreads();
  const int E = C * Ch + C + Ch;
  float* out = a.part + (size_t)blockIdx.x * E;
  for (int e = tid; e < E; e += kThr) {
    float s = 0.f;
    // with paired warps, channel group g was accumulated only by the warps w with
    // (w & 1) == g / 32, and db_L only by even warps
    if (e < C * Ch) {
      const int c = e / Ch, ch = e % Ch;
      const int own = pairB ? (ch / 4) / 32 : -1;
      for (int q = 0; q < kThr / 32; ++q)
        if (own < 0 || (q & 1) == own) s += red[(q * Ch + ch) * RW + c];
    } else if (e < C * Ch + C) {
      const int c = e - C * Ch;
      for (int q = 0; q < kThr / 32; ++q) s += redL[q * kMaxC + c];
    } else {
      const int ch = e - C * Ch - C;
      const int own = pairB ? (ch / 4) / 32 : -1;
      for (int q = 0; q < kThr / 32; ++q)
        if (own < 0 || (q & 1) == own) s += red[(q * Ch + ch) * RW + C];
    }
    out[e] = s;
  }
}

size_t head_smem(int C, int Ch) {
  return 128 + head_region0(C, Ch) + sizeof(float) * (((C * Ch + 3) & ~3) + kMaxC + kTP * kMaxC) + sizeof(int) * kTP;
}

template <int NC, bool TRAIN, bool TANH>
cudaError_t launch_k(const HeadArgs& a, size_t smem, cudaStream_t s) {
  auto kern = (a.Ch % 4 == 0) ? head_kernel<NC, TRAIN, TANH, true> : head_kernel<NC, TRAIN, TANH, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<a.n_blocks, kThr, smem, s>>>(a);
  return cudaGetLastError();
}

template <int NC>
cudaError_t launch_nc(const HeadArgs& a, size_t smem, cudaStream_t s) {
  if (a.probs) return launch_k<NC, false, true>(a, smem, s);  // forward: activation unused
  if (a.hidden_act == MPF_TANH) return launch_k<NC, true, true>(a, smem, s);
  return launch_k<NC, true, false>(a, smem, s);
}

// The label of every head position, gathered once per step in position order through
// the fragment -> pixel map (head_label; R2, R7), so the head reads 64 contiguous bytes
// per tile instead of decoding the mixed-radix index per position.
__global__ void label_frag_kernel(HeadArgs a, uint8_t* __restrict__ out, long long per_img, int frag_sz) {
  const long long total = (long long)a.n * per_img;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int img = (int)(e / per_img);
    const int lab = head_label(a, img, e - (long long)img * per_img, per_img, frag_sz, true);
    out[e] = (uint8_t)(lab == kLabPad ? kLabFragPad : lab);
  }
}

}  // namespace

int head_tiles_per_image(long long per_img) { return (int)((per_img + kTP - 1) / kTP); }
int head_loss_parts_per_tile() { return kThr / 32; }

int head_blocks(long long total_tiles) {
  long long nb = 148LL * 2;
  if (nb > total_tiles) nb = total_tiles;
  return (int)(nb < 1 ? 1 : nb);
}

bool head_supported(int C, int Ch) {
  return C >= 2 && C <= kMaxC && Ch >= 1 && Ch <= kThr && head_smem(C, Ch) <= 200 * 1024;
}

cudaError_t launch_head2(const HeadArgs& a, cudaStream_t s) {
  const size_t smem = head_smem(a.C, a.Ch);
  switch (a.C) {  // exact class counts of the common heads; padded beyond
    case 2: return launch_nc<2>(a, smem, s);
    case 3: return launch_nc<3>(a, smem, s);
    case 4: return launch_nc<4>(a, smem, s);
    case 5: return launch_nc<5>(a, smem, s);
    default: return a.C <= 8 ? launch_nc<8>(a, smem, s) : launch_nc<16>(a, smem, s);
  }
}

cudaError_t launch_label_frag(const HeadArgs& a, uint8_t* out, cudaStream_t s) {
  const long long per_img = (long long)a.F * a.gr * a.gc;
  const long long total = (long long)a.n * per_img;
  const long long blocks = (total + 255) / 256 < 148 * 16 ? (total + 255) / 256 : 148 * 16;
  label_frag_kernel<<<(unsigned)(blocks < 1 ? 1 : blocks), 256, 0, s>>>(a, out, per_img, a.gr * a.gc);
  return cudaGetLastError();
}

}  // namespace mpf
