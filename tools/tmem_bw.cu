// Microbenchmark: tcgen05.ld / tcgen05.st throughput per SM as a function of
// the number of warps issuing.  nvcc -gencode arch=compute_100a,code=sm_100a
//   -I paper_2102_03161_b200/csrc/kernels -Iinclude tools/tmem_bw.cu -o /tmp/tmem_bw
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace eps_k;

__global__ void tmem_ld_bench(int iters, long long* out, int mode) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 32 % 512);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) {
      uint32_t r[32];
      tmem_ld_32x32(base, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += r[j];
    } else {
      uint32_t r[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) r[j] = i + j;
      tmem_st_32x32_x16(base, r);
      tmem_st_wait();
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345678) out[1000] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int nw : {1, 2, 4, 8, 16}) {
      const int iters = 2000;
      tmem_ld_bench<<<1, nw * 32>>>(iters, d, mode);
      cudaDeviceSynchronize();
      long long cyc;
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      const double bytes = double(iters) * nw * 32 * (mode == 0 ? 32 : 16) * 4;
      printf("%s warps=%2d cycles=%lld  bytes/cycle/SM=%.1f\n", mode == 0 ? "ld.x32" : "st.x16", nw,
             cyc, bytes / double(cyc));
    }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
