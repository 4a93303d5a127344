// Where does a cta_group::1 M = 64 accumulator land in TMEM, and can its
// D address carry a lane offset (64)?  A = B = ones (K = 16) -> D = 16.
//   nvcc -std=c++20 -gencode arch=compute_100a,code=sm_100a -I paper_2102_03161_b200/csrc/kernels \
//        -Iinclude tools/m64_layout.cu -o tools/m64_layout.bin
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace eps_k;

__global__ void __launch_bounds__(128, 1) m64(uint32_t lane_base, int m, float* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ones everywhere (swizzle irrelevant)
  for (int i = threadIdx.x; i < 16384; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x3F803F80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&slot, 128);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  {
    uint32_t z[32];
    for (int j = 0; j < 32; ++j) z[j] = 0u;
    for (int c = 0; c < 128; c += 32) tmem_st_32x32_x32(tmem + (uint32_t(warp * 32) << 16) + c, z);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    const uint64_t a = umma_sdesc(smem_addr(smem), 16, 1024);
    const uint64_t b = umma_sdesc(smem_addr(smem + 32768), 16, 1024);
    tc_mma_ss_ws(tmem + (lane_base << 16), a, b, umma_idesc_bf16(m, 64, false, false), 0u);
    tc_commit_ws(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld_32x32(tmem + (uint32_t(warp * 32) << 16), r);
  tmem_ld_wait();
  for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * 64 + j] = __uint_as_float(r[j]);
  tmem_ld_32x32(tmem + (uint32_t(warp * 32) << 16) + 32, r);
  tmem_ld_wait();
  for (int j = 0; j < 32; ++j) out[(warp * 32 + lane) * 64 + 32 + j] = __uint_as_float(r[j]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 64 * 4);
  cudaFuncSetAttribute(m64, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  static float h[128 * 64];
  for (int m : {64, 128})
    for (uint32_t lb : {0u, 16u, 48u}) {
      if (m == 128 && lb) continue;
      cudaMemset(d, 0, 128 * 64 * 4);
      m64<<<1, 128, 80 * 1024>>>(lb, m, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("M=%d D lane base %u (%s): lanes with D = 16 in cols 0..63:\n  ", m, lb,
             cudaGetErrorString(e));
      for (int l = 0; l < 128; ++l) {
        int n = 0;
        for (int c = 0; c < 64; ++c) n += h[l * 64 + c] == 16.f;
        printf("%c", n == 64 ? '#' : n == 0 ? '.' : '+');
      }
      printf("\n");
    }
  return 0;
}
