// conv_first_tc.cu — the first convolution layer's forward pass (one input map: the raw
// image; Alg. 1, readings R7, R10) on the tensor cores.
//
// With C_in = 1 the implicit GEMM's K dimension is the k x k window itself.  A column slab
// turns it into the slab trick of the wide convolutions: for an output row y and 128
// consecutive outputs x0 .. x0+127, the slab S[r][ky] = img[y + ky][x0 + r]
// (r < 128 + k - 1, ky < 8, zero beyond k) holds, in row r + kx, exactly the k values that
// output x0 + r needs from column kx of its window.  So
//     out[x0 + r][co] = sum_kx  S[r + kx][:] . W[co][:][kx]
// is k MMAs (M = 128 outputs, N = C_out, K = 8 "channels" = ky) whose A operand is the
// same slab with its start moved by kx rows (K-major, 32-byte swizzle).  3xTF32 (image and
// weights split hi + lo): the first layer feeds a max pool, whose argmax must see the
// same fp32-accurate values as the CUDA-core kernel (R16).
//
// Roles (persistent, one CTA per SM): 8 warps build slabs (ring of 4), 1 warp issues the
// MMAs, 8 warps drain the double-buffered TMEM accumulator (bias, activation) into
// staging boxes (ring of 4), 4 warps copy the boxes out with coalesced 16-byte stores.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "conv_tc.h"
#include "mpf_internal.h"
#include "tc_ptx.cuh"

namespace mpf {

namespace {

constexpr int kFT = 128;                     // outputs per tile (one output row segment)
constexpr int kFRing = 4;                    // slab ring
constexpr int kFSlabRows = kFT + 8;          // >= 128 + k - 1 for k <= 8 (17 SW32 atoms)
constexpr int kFSlabBytes = kFSlabRows * 32; // one of hi / lo
constexpr int kFBld = 8;                     // slab builder warps
constexpr int kFEpi = 8;                     // epilogue warps: 4 lane quarters x 2 groups of 16 maps
constexpr int kFStage = 4;                   // output staging boxes
constexpr int kFSt = 4;                      // store warps
constexpr int kFW0 = kFBld, kFE0 = kFBld + 1, kFS0 = kFE0 + kFEpi;  // MMA warp, first epilogue / store warp
constexpr int kFThreads = 32 * (kFS0 + kFSt);
constexpr int kFRaw = 4, kFPre = 3;          // raw image ring, prefetch distance (tiles)

// TF32 rounding (nearest-even, finite-saturating: one F2FP instruction on sm_100a; the guarded
// cvt.rna form takes four) of an MMA operand
__device__ __forceinline__ float tf32_rna_f(float x) {
  uint32_t r;
  asm("cvt.rn.satfinite.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ float ex2a(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpa(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// tanh(v) = 1 - 2 / (2^(2 v log2 e) + 1) (absolute error ~1e-7, as the wide convolutions)
__device__ __forceinline__ float act_f(int act, float v) {
  if (act == MPF_TANH) return fmaf(-2.f, rcpa(ex2a(2.8853900817779268f * v) + 1.f), 1.f);
  if (act == MPF_LOGISTIC) return rcpa(1.f + ex2a(-1.4426950408889634f * v));
  return v;
}
// mbarrier wait adding its duration to prof[slot] (lane 0) when profiling (MPF_FIRST_PROF=1)
__device__ __forceinline__ void fwait(uint32_t bar, uint32_t parity, unsigned long long* prof, int slot) {
  if (!prof) {
    ptx::mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  ptx::mbar_wait(bar, parity);
  if ((threadIdx.x & 31) == 0) atomicAdd(prof + slot, (unsigned long long)(clock64() - t0));
}
__device__ __forceinline__ void named_bar_f(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ uint64_t sdesc_k_sw32(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(256u >> 4) << 32;  // 8-row groups of 32-byte rows
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)6 << 61;            // SWIZZLE_32B
  return d;
}
// byte offset of element (row r, k < 8) in a K-major SW32 tile
__device__ __forceinline__ uint32_t sw32_off(int r, int k) {
  return (uint32_t)(r * 32 + ((((k >> 2) ^ (r >> 2)) & 1) << 4) + (k & 3) * 4);
}

// smem: [ring][hi|lo] slabs | W [k][hi|lo][32 co][32 B] | raw [kFRaw][8][rows] | output
// staging [2][128][C_out] | bias | barriers
struct FtLayout {
  uint32_t slab, w, raw, stage, bias, bar;
};
__host__ __device__ inline FtLayout ft_layout(int k) {
  FtLayout L;
  L.slab = 0;
  L.w = L.slab + kFRing * 2 * kFSlabBytes;
  L.raw = L.w + k * 2 * 32 * 32;
  L.stage = L.raw + kFRaw * 8 * kFSlabRows * 4;
  L.stage = (L.stage + 1023) & ~1023u;  // SW128 staging
  L.bias = L.stage + kFStage * kFT * 128;
  L.bar = L.bias + 32 * 4;
  return L;
}

__global__ void __launch_bounds__(kFThreads, 1)
    conv_first_tc_kernel(const __grid_constant__ CUtensorMap tmO, FirstConvArgs a, int n_xt, unsigned long long* prof) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (sbase - ptx::smem_u32(smem_raw));
  const int K = a.k;
  const FtLayout L = ft_layout(K);
  const uint32_t bSFull = sbase + L.bar, bSEmpty = bSFull + 8 * kFRing, bTFull = bSEmpty + 8 * kFRing,
                 bTEmpty = bTFull + 16, bOFull = bTEmpty + 16, bOEmpty = bOFull + 8 * kFStage,
                 sTmemSlot = bOEmpty + 8 * kFStage;
  float* s_bias = reinterpret_cast<float*>(gbase + L.bias);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  const long long total = (long long)a.n * a.out_gr * n_xt;
  const int n_my = blockIdx.x < total ? (int)((total - 1 - blockIdx.x) / gridDim.x) + 1 : 0;

  // weights W[co][ky][kx] -> per tap kx a K-major B tile [co][ky] (hi / lo TF32 split)
  for (int e = tid; e < K * 32 * 8; e += kFThreads) {
    const int kx = e / 256, co = (e / 8) % 32, ky = e % 8;
    const float w = (co < a.cout && ky < K) ? a.w[(co * K + ky) * K + kx] : 0.f;
    const float hi = tf32_rna_f(w);
    uint8_t* base = gbase + L.w + kx * 2048;
    *reinterpret_cast<float*>(base + sw32_off(co, ky)) = hi;
    *reinterpret_cast<float*>(base + 1024 + sw32_off(co, ky)) = w - hi;
  }
  if (tid < 32) s_bias[tid] = tid < a.cout ? a.bias[tid] : 0.f;
  if (tid == 0) {
    for (int i = 0; i < kFRing; ++i) {
      ptx::mbar_init(bSFull + 8 * i, kFBld);
      ptx::mbar_init(bSEmpty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(bTFull + 8 * i, 1);
      ptx::mbar_init(bTEmpty + 8 * i, kFEpi);

    }
    for (int i = 0; i < kFStage; ++i) {
      ptx::mbar_init(bOFull + 8 * i, kFEpi);  // staging box written by every epilogue warp
      ptx::mbar_init(bOEmpty + 8 * i, kFSt);  // ... and copied out by every store warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == kFW0) ptx::tmem_alloc(sTmemSlot, 64);
  ptx::fence_proxy_async();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(gbase + (sTmemSlot - sbase));
  auto tile_coords = [&](int i, int& img, int& y, int& x0) {
    const long long t = (long long)blockIdx.x + (long long)i * gridDim.x;
    x0 = (int)(t % n_xt) * kFT;
    const long long t2 = t / n_xt;
    y = (int)(t2 % a.out_gr);
    img = (int)(t2 / a.out_gr);
  };

  if (warp < kFBld) {
    // ------------------------------------------------------------------ slab builders
    // Element e = ky * kFSlabRows + r of a slab belongs to builder thread e % (32 kFBld):
    // the thread stages it with cp.async kFPre tiles ahead (raw ring, zero-filled outside
    // the image) and later converts that same value into the swizzled hi / lo slab, so no
    // thread waits on a load issued for the tile it is converting, and no barrier is needed.
    constexpr int kNB = 32 * kFBld;
    float* raw = reinterpret_cast<float*>(gbase + L.raw);  // [kFRaw][8][kFSlabRows]
    auto prefetch = [&](int i) {
      if (i < n_my) {
        int img, y, x0;
        tile_coords(i, img, y, x0);
        float* rb = raw + (i % kFRaw) * 8 * kFSlabRows;
        for (int e = tid; e < 8 * kFSlabRows; e += kNB) {
          const int ky = e / kFSlabRows, r = e - ky * kFSlabRows;
          const int x = x0 + r, yy = y + ky;
          const bool in = ky < K && x < a.W && yy < a.H;
          const float* src = a.img + (in ? ((long long)img * a.H + yy) * a.W + x : 0);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(rb + e)),
                       "l"(src), "r"(in ? 4 : 0)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int i = 0; i < kFPre; ++i) prefetch(i);
    for (int i = 0; i < n_my; ++i) {
      prefetch(i + kFPre);
      asm volatile("cp.async.wait_group %0;" ::"n"(kFPre) : "memory");  // tile i's group landed
      const int s = i % kFRing;
      fwait(bSEmpty + 8 * s, ((i / kFRing) & 1) ^ 1, prof, 0);
      const float* rb = raw + (i % kFRaw) * 8 * kFSlabRows;
      uint8_t* hi = gbase + L.slab + s * 2 * kFSlabBytes;
      uint8_t* lo = hi + kFSlabBytes;
      for (int e = tid; e < 8 * kFSlabRows; e += kNB) {
        const int ky = e / kFSlabRows, r = e - ky * kFSlabRows;
        const float v = rb[e];
        const float h = tf32_rna_f(v);
        const uint32_t o = sw32_off(r, ky);
        *reinterpret_cast<float*>(hi + o) = h;
        *reinterpret_cast<float*>(lo + o) = v - h;
      }
      ptx::fence_proxy_async();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bSFull + 8 * s);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else if (warp == kFW0) {
    // ------------------------------------------------------------------ MMA issuer
    const uint32_t idesc = ptx::idesc_tf32(128, 32);
    const long long t_start = clock64();
    for (int i = 0; i < n_my; ++i) {
      const int s = i % kFRing, b = i & 1;
      fwait(bTEmpty + 8 * b, ((i >> 1) & 1) ^ 1, prof, 2);
      fwait(bSFull + 8 * s, (i / kFRing) & 1, prof, 1);
      ptx::tc_fence_after();
      const uint32_t hi = sbase + L.slab + s * 2 * kFSlabBytes, lo = hi + kFSlabBytes;
      const uint32_t d = tmem + b * 32;
      for (int kx = 0; kx < K; ++kx) {
        const uint32_t w = sbase + L.w + kx * 2048;
        const uint64_t a_hi = sdesc_k_sw32(hi + kx * 32), a_lo = sdesc_k_sw32(lo + kx * 32);
        const uint64_t b_hi = sdesc_k_sw32(w), b_lo = sdesc_k_sw32(w + 1024);
        ptx::mma_tf32_elect(d, a_hi, b_hi, idesc, kx != 0);
        ptx::mma_tf32_elect(d, a_hi, b_lo, idesc, 1u);
        ptx::mma_tf32_elect(d, a_lo, b_hi, idesc, 1u);
      }
      ptx::mma_commit_elect(bSEmpty + 8 * s);
      ptx::mma_commit_elect(bTFull + 8 * b);
    }
    if (prof && lane == 0) atomicAdd(prof + 7, (unsigned long long)(clock64() - t_start));
  } else if (warp >= kFS0) {
    // ------------------------------------------------------------------ store warp
    // copies each staging box to HBM with coalesced 16-byte stores (one 512-byte run per
    // instruction: the tile's outputs are contiguous)
    const int nv = a.cout / 4;
    for (int i = 0; i < n_my; ++i) {
      const int sb = i % kFStage;
      int img, y, x0;
      tile_coords(i, img, y, x0);
      fwait(bOFull + 8 * sb, (i / kFStage) & 1, prof, 6);
      const int np = min(kFT, a.out_gc - x0);
      float* dst = a.out + (((long long)img * a.out_gr + y) * a.out_gc + x0) * a.cout;
      const uint8_t* box = gbase + L.stage + sb * kFT * 128;
      const int total4 = np * nv;  // float4s in the tile
      for (int e = (warp - kFS0) * 32 + lane; e < total4; e += 32 * kFSt) {
        const int row = e / nv, j = e - row * nv;
        const float4 v = *reinterpret_cast<const float4*>(box + row * 128 + ((j ^ (row & 7)) << 4));
        reinterpret_cast<float4*>(dst)[e] = v;
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bOEmpty + 8 * sb);
    }
  } else {
    // ------------------------------------------------------------------ epilogue
    // thread = (output position, group of 8 maps); the tile's [128][C_out] outputs go
    // through a double-buffered SW128 staging box and one TMA store per tile
    const int q = warp & 3, grp = (warp - kFE0) >> 2;
    const int r = q * 32 + lane;
    const int nv = a.cout / 4;  // float4 per position (C_out % 4 == 0)
    for (int i = 0; i < n_my; ++i) {
      const int b = i & 1;
      int img, y, x0;
      tile_coords(i, img, y, x0);
      fwait(bTFull + 8 * b, (i >> 1) & 1, prof, 4);
      ptx::tc_fence_after();
      float f[16];
      ptx::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + b * 32 + grp * 16, f);
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(bTEmpty + 8 * b);
      // staging box sb was handed to the TMA store of tile i - kFStage: wait until it was read
      const int sb = i % kFStage;
      fwait(bOEmpty + 8 * sb, ((i / kFStage) & 1) ^ 1, prof, 5);
      const int x = x0 + r;
      const bool valid = y < a.out_vr && x < a.out_vc;
      float v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        float t = 0.f;
        if (valid) {
          t = act_f(a.act, f[c] + s_bias[grp * 16 + c]);
          if (a.round_tf32) t = tf32_rna_f(t);
        }
        v[c] = t;
      }
      // SW128 staging (row r = 128 B, 16-byte chunk j at j ^ (r & 7)): conflict-free
      uint8_t* st = gbase + L.stage + sb * kFT * 128 + r * 128;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = grp * 4 + jj;
        if (j < nv)
          *reinterpret_cast<float4*>(st + ((j ^ (r & 7)) << 4)) =
              make_float4(v[4 * jj], v[4 * jj + 1], v[4 * jj + 2], v[4 * jj + 3]);
      }
      __syncwarp();  // generic stores, read back by the store warps (mbarrier release/acquire)
      if (lane == 0) ptx::mbar_arrive(bOFull + 8 * sb);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kFW0) ptx::tmem_dealloc(tmem, 64);
}

size_t ft_smem(int k) {
  const FtLayout L = ft_layout(k);
  return 1024 + L.bar + 8 * (2 * kFRing + 4 + 2 * kFStage) + 16;
}

}  // namespace

// Tensor-core first layer: one input map, k <= 8, C_out <= 32 and % 4 (N = 32, 16-byte
// output rows), TF32 precision mode.  Opt-in (MPF_FIRST_TC=1): correct (GPU parity suite)
// but not faster than the register-blocked CUDA-core kernel (conv_first.cu) on the
// BASELINE configs — 1.2 vs 1.17 ms (cfg4, k = 7), 0.62 vs 0.28 ms (cfg5, k = 4); the
// per-tile pipeline (slab build -> 21 small MMAs -> activation -> store) is latency-bound
// (role timers: MPF_FIRST_PROF=1).
bool first_conv_tc_ok(int cin, int cout, int k) {
  const char* e = getenv("MPF_FIRST_TC");
  if (!e || atoi(e) == 0) return false;
  return cin == 1 && cout >= 4 && cout <= 32 && cout % 4 == 0 && k >= 2 && k <= 8;
}

cudaError_t launch_first_conv_tc(const FirstConvArgs& a, cudaStream_t s) {
  const int n_xt = (a.out_gc + kFT - 1) / kFT;
  const long long total = (long long)a.n * a.out_gr * n_xt;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  const int grid = (int)(total < sms ? (total < 1 ? 1 : total) : sms);
  const size_t smem = ft_smem(a.k);
  cudaError_t e = cudaFuncSetAttribute(conv_first_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  CUtensorMap tmO;
  const uint64_t dims[3] = {(uint64_t)a.cout, (uint64_t)a.out_gc, (uint64_t)a.n * a.out_gr};
  const uint64_t strides[2] = {(uint64_t)a.cout * 4, (uint64_t)a.out_gc * a.cout * 4};
  const uint32_t box[3] = {32, (uint32_t)kFT, 1};
  e = make_tmap_f32(&tmO, a.out, 3, dims, strides, box, true);
  if (e != cudaSuccess) return e;
  static unsigned long long* prof = nullptr;
  const bool do_prof = getenv("MPF_FIRST_PROF") != nullptr;
  if (do_prof && !prof) cudaMalloc(&prof, 8 * sizeof(unsigned long long));
  if (do_prof) cudaMemsetAsync(prof, 0, 8 * sizeof(unsigned long long), s);
  conv_first_tc_kernel<<<grid, kFThreads, smem, s>>>(tmO, a, n_xt, do_prof ? prof : nullptr);
  if (do_prof) {
    unsigned long long h[8];
    cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const double c = grid;
    fprintf(stderr,
            "[first-prof] per CTA Mcyc: mma-warp total %.3f | builders(per warp) wait slab-empty %.3f "
            "| mma wait tmem-empty %.3f slab-full %.3f | epilogue(per warp) wait tmem-full %.3f staging %.3f | "
            "store warp wait full %.3f wait store-read %.3f\n",
            h[7] / c / 1e6, h[0] / c / kFBld / 1e6, h[2] / c / 1e6, h[1] / c / 1e6, h[4] / c / kFEpi / 1e6,
            h[5] / c / kFEpi / 1e6,
            h[6] / c / 1e6, h[3] / c / 1e6);
  }
  return cudaGetLastError();
}

}  // namespace mpf
