// mma_sync_micro.cu — throughput of the warp-level (legacy) tensor-core path on sm_100a:
// mma.sync.m16n8k8 TF32 (fp32 accumulate), 8 independent accumulator chains per warp, all
// SMs.  Decides whether a warp-synchronous MMA head (no TMEM round trips) can take the
// head's ~3000 FMAs per position off the FMA pipes (DESIGN.md §5 "Head").
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_micro scripts/mma_sync_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tf32(float* out, int iters) {
  float d[8][4];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) d[i][j] = 0.f;
  unsigned a0 = threadIdx.x, a1 = threadIdx.x * 3, a2 = threadIdx.x * 5, a3 = threadIdx.x * 7, b0 = 11, b1 = 13;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 4; ++j) s += d[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  for (int warps = 4; warps <= 16; warps *= 2) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_tf32<<<sms, 32 * warps>>>(out, 16);
    cudaEventRecord(e0);
    k_tf32<<<sms, 32 * warps>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * 16 * 8 * 8 * 8.0 * iters * warps * sms;
    printf("mma.sync m16n8k8 tf32: %d warps/SM: %.1f TFLOP/s (%.3f ms)\n", warps, flop / ms / 1e9, ms);
  }
  return cudaGetLastError() != cudaSuccess;
}
