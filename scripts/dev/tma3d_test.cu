// Standalone check of 3-D TMA tile loads (fp32 and uint8 maps) with mbarrier completion.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include "../../paper_1302_1690_b200/csrc/tc_ptx.cuh"
using namespace mpf;

__global__ void k(const __grid_constant__ CUtensorMap tm, int c0, int c1, int c2, uint32_t bytes, int* out) {
  extern __shared__ __align__(1024) uint8_t sm0[];
  uint8_t* sm = sm0 + ((128u - (ptx::smem_u32(sm0) & 127u)) & 127u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 8192);
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(bar), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(ptx::smem_u32(bar), bytes);
    ptx::tma_load_3d(ptx::smem_u32(sm), &tm, ptx::smem_u32(bar), c0, c1, c2);
  }
  const long long t0 = clock64();
  bool ok = true;
  while (!ptx::mbar_try_wait(ptx::smem_u32(bar), 0))
    if (clock64() - t0 > (1LL << 31)) { ok = false; break; }
  if (threadIdx.x == 0) { out[0] = ok; out[1] = ((int*)sm)[0]; out[2] = sm[1]; }
}

int main() {
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  void* buf; cudaMalloc(&buf, 64 << 20); cudaMemset(buf, 1, 64 << 20);
  int* out; cudaMalloc(&out, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  struct Case { const char* name; CUtensorMapDataType dt; int es; cuuint64_t d[3]; cuuint64_t st[2]; cuuint32_t box[3]; int c[3]; };
  Case cs[] = {
    {"f32 C64 box32x11", CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, {64, 27, 1000}, {256, 27 * 256}, {32, 11, 1}, {32, 10, 5}},
    {"f32 C24 box24x20", CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, {24, 260, 1000}, {96, 260 * 96}, {24, 20, 1}, {0, 250, 5}},
    {"u8 C64 box32x11", CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, {64, 27, 1000}, {64, 27 * 64}, {32, 11, 1}, {32, 10, 5}},
    {"u8 C48 box32x19", CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, {48, 85, 1000}, {48, 85 * 48}, {32, 19, 1}, {24, 70, 5}},
    {"u8 chunks 16x31", CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, {16, 390, 1000}, {16, 6240}, {16, 31, 1}, {0, 380, 5}},
  };
  for (auto& c : cs) {
    CUtensorMap tm;
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm, c.dt, 3, buf, c.d, c.st, c.box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    uint32_t bytes = c.box[0] * c.box[1] * c.es;
    k<<<1, 64, 16384>>>(tm, c.c[0], c.c[1], c.c[2], bytes, out);
    cudaError_t e = cudaDeviceSynchronize();
    int h[3] = {-1, -1, -1};
    if (e == cudaSuccess) cudaMemcpy(h, out, 12, cudaMemcpyDeviceToHost);
    printf("%-20s encode %d launch %s ok %d v %x %x\n", c.name, (int)r, cudaGetErrorString(e), h[0], h[1], h[2]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
