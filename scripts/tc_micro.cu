// tc_micro.cu — microbenchmark of tcgen05.mma kind::tf32 issue/execute rate on one SM
// per CTA (all SMs busy), to find the tensor-core ceiling of the conv kernels' MMA
// pattern: cycles per MMA vs N, vs the A start-row offset (the slab trick shifts A by
// kx rows inside a SWIZZLE_128B atom), and vs cta_group::2.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1302_1690_b200/csrc \
//        scripts/tc_micro.cu -o /tmp/tc_micro -lcuda && /tmp/tc_micro
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "tc_ptx.cuh"

using namespace mpf;

__global__ void __launch_bounds__(128, 1) micro(int n_mma, int npad, int a_row_off, int vary_k8, int two_acc,
                                                int commit_every, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t sbase = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = sbase, sB = sbase + 64 * 1024;
  const uint32_t bar = sbase + 160 * 1024, slot = bar + 8, bar2 = bar + 16;
  uint8_t* gen = smem_raw - ptx::smem_u32(smem_raw);
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(gen + sbase)[i] = 0.f;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    ptx::mbar_init(bar, 1);
    ptx::mbar_init(bar2, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(slot, 512);
  ptx::fence_proxy_async();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<uint32_t*>(gen + slot);
  if (threadIdx.x == 0) {
    const uint32_t idesc = ptx::idesc_tf32(128, npad);
    long long t0 = clock64();
    const int G = commit_every ? commit_every : 16;
    for (int g = 0; g < n_mma / G; ++g) {
      for (int j = 0; j < G; ++j) {
        const int i = g * G + j;
        const int k8 = vary_k8 ? (j & 3) : 0;
        const uint32_t aaddr = sA + a_row_off * 128 + k8 * 32;
        const uint32_t baddr = sB + k8 * 32;
        const uint32_t d = tmem + (two_acc ? (j & 1) * npad : 0);
        ptx::mma_tf32(d, ptx::sdesc_k_sw128(aaddr, 0), ptx::sdesc_k_sw128(baddr, 0), idesc, i > 1);
      }
      if (commit_every) ptx::mma_commit(bar2);  // never waited
    }
    ptx::mma_commit(bar);
    ptx::mbar_wait(bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  const int smem = 170 * 1024;
  cudaFuncSetAttribute(micro, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int n_mma = 20000;
  printf("tf32 M=128 cta_group::1, %d MMAs per SM, all 148 SMs; math = 128*N*8/2048 cycles\n", n_mma);
  printf("%5s %6s %6s %6s %10s %10s %8s\n", "N", "a_off", "commit", "2acc", "cyc/mma", "math", "eff");
  // A start-row offset (the slab trick's kx shift) x N, commit every 16 MMAs, two accumulators
  int Ns[] = {32, 64, 128, 208, 256};
  int Offs[] = {0, 1, 2, 3, 4, 8};
  for (int ni = 0; ni < 5; ++ni) {
    for (int oi = 0; oi < 6; ++oi) {
      const int two = 1, kv = 16;
      micro<<<148, 128, smem>>>(n_mma, Ns[ni], Offs[oi], 1, two, kv, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148.0 * n_mma;
      const double math = 128.0 * Ns[ni] * 8 / 2048.0;
      printf("%5d %6d %6d %6d %10.1f %10.1f %7.0f%%\n", Ns[ni], Offs[oi], kv, two, avg, math, 100 * math / avg);
    }
  }
  return 0;
}
