// exchange.cu — data-parallel gradient exchange over peer memory (include/mpf.h
// "mpf_exchange_*").
//
// Alg. 2 sums the weight gradient over every fragment and position; with the
// images of a global batch sharded over ranks that sum runs over the ranks too.  Instead of a
// separate all-reduce, every rank pushes each gradient bucket, as soon as the backward has
// finished it, into its own slot of every rank's exchange buffer (P2P stores over NVLink) and
// raises a flag there; the SGD step waits for all flags, sums the slots in rank order and
// updates the parameters — the reduction is fused into the optimizer kernel, the transfer
// overlaps the backward.
//
// Exchange buffer of one rank (bytes; ExLayout):
//   [0, 4)      epoch: completed SGD steps (written by the own SGD kernel only)
//   [8, 12)     SGD arrival counter          [12, 16) timeout flag (rank + 1 that never came)
//   [256, 512)  push arrival counters, one per bucket
//   [512, 1024) peer table: 64-bit address of every rank's buffer as seen from this process
//   [1024, ..)  flags [world][n_layers] u32: epoch of the last bucket b pushed by rank r
//   [slots, ..) slots [2 parities][world][n_params] fp32
#include <cuda_runtime.h>
#include <stdint.h>

#include "mpf_internal.h"

namespace mpf {

namespace {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(256) exchange_push_kernel(const float* __restrict__ g, long long off, long long count,
                                                            char* own, ExLayout L, int rank, int b) {
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(own) + 1;  // this step's epoch
  const int par = (int)(e & 1u);
  const uint64_t* peers = reinterpret_cast<const uint64_t*>(own + ExLayout::kPeers);
  const long long slot0 = ((long long)par * L.world + rank) * L.n_params + off;  // floats
  const long long stride = (long long)gridDim.x * blockDim.x;
  if (((off | count | L.n_params) & 3) == 0) {  // 16-byte vectors
    const long long n4 = count / 4;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(g + off) + i);
      for (int r = 0; r < L.world; ++r)
        reinterpret_cast<float4*>(reinterpret_cast<float*>(peers[r] + L.slots) + slot0)[i] = v;
    }
  } else {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += stride) {
      const float v = __ldg(g + off + i);
      for (int r = 0; r < L.world; ++r) reinterpret_cast<float*>(peers[r] + L.slots)[slot0 + i] = v;
    }
  }
  // the last block to finish raises this rank's flag for bucket b in every buffer, after every
  // block's stores are visible system-wide
  __threadfence_system();
  __syncthreads();
  __shared__ bool last;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(own + ExLayout::kPushCnt) + b;
  if (threadIdx.x == 0) last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  if (threadIdx.x < L.world) {
    __threadfence_system();
    st_release_sys(reinterpret_cast<uint32_t*>(peers[threadIdx.x] + ExLayout::kFlags) + rank * L.nbmax + b, e);
  }
  if (threadIdx.x == 0) *cnt = 0u;  // ready for the next step's push of this bucket
}

__global__ void __launch_bounds__(256) exchange_sgd_kernel(float* __restrict__ p, float* __restrict__ g, float step,
                                                           char* own, ExLayout L, int nb) {
  const uint32_t e = *reinterpret_cast<volatile uint32_t*>(own) + 1;
  const int par = (int)(e & 1u);
  __shared__ int ok;
  if (threadIdx.x == 0) {  // wait (acquire) until every rank's every bucket carries epoch e
    const uint32_t* flags = reinterpret_cast<const uint32_t*>(own + ExLayout::kFlags);
    const long long t0 = clock64();
    int bad = 0;
    for (int r = 0; r < L.world && !bad; ++r)
      for (int q = 0; q < nb && !bad; ++q)
        while ((int)(ld_acquire_sys(flags + r * L.nbmax + q) - e) < 0)
          if (clock64() - t0 > (1LL << 34)) {  // ~10 s: a rank never pushed
            bad = r + 1;
            break;
          }
    ok = !bad;
    if (bad) atomicExch(reinterpret_cast<uint32_t*>(own + ExLayout::kTimeout), (uint32_t)bad);
  }
  __syncthreads();
  if (!ok) return;
  const float* slots = reinterpret_cast<const float*>(own + L.slots) + (long long)par * L.world * L.n_params;
  const long long n = L.n_params;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    // L2 loads (peers wrote these lines over NVLink; no stale L1 copy can be used)
    float s = __ldcg(slots + i);
    for (int r = 1; r < L.world; ++r) s += __ldcg(slots + (long long)r * n + i);  // rank order, same on every rank
    p[i] -= step * s;
    g[i] = 0.f;
  }
  __syncthreads();
  __shared__ bool last;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(own + ExLayout::kSgdCnt);
  if (threadIdx.x == 0) last = atomicAdd(cnt, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    *cnt = 0u;
    *reinterpret_cast<volatile uint32_t*>(own) = e;  // step complete: the next push / SGD use e + 1
  }
}

}  // namespace

ExLayout exchange_layout(int world, int nbmax, long long n_params) {
  ExLayout L;
  L.world = world;
  L.nbmax = nbmax;
  L.n_params = n_params;
  size_t s = ExLayout::kFlags + sizeof(uint32_t) * (size_t)world * nbmax;
  s = (s + 255) & ~(size_t)255;
  L.slots = s;
  L.bytes = s + sizeof(float) * 2 * (size_t)world * (size_t)n_params;
  return L;
}

cudaError_t launch_exchange_push(const float* grads, long long off, long long count, char* own, const ExLayout& L,
                                 int rank, int bucket, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  long long blocks = (count / 4 + 255) / 256;
  if (blocks > 296) blocks = 296;
  if (blocks < 1) blocks = 1;
  exchange_push_kernel<<<(unsigned)blocks, 256, 0, s>>>(grads, off, count, own, L, rank, bucket);
  return cudaGetLastError();
}

cudaError_t launch_exchange_sgd(float* params, float* grads, float lr, float scale, char* own, const ExLayout& L,
                                int nb, cudaStream_t s) {
  long long blocks = (L.n_params + 255) / 256;
  if (blocks > 592) blocks = 592;
  if (blocks < 1) blocks = 1;
  exchange_sgd_kernel<<<(unsigned)blocks, 256, 0, s>>>(params, grads, lr * scale, own, L, nb);
  return cudaGetLastError();
}

}  // namespace mpf
