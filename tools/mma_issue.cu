// Microbenchmark: tcgen05.mma issue rate from one warp, two issue styles.
//   mode 0: one lane (if lane == 0), descriptors rebuilt per MMA (old style)
//   mode 1: whole warp converged, elect.sync per MMA, descriptors precomputed
//   mode 2: one lane, descriptors precomputed
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a
//   -I paper_2102_03161_b200/csrc/kernels -Iinclude tools/mma_issue.cu -o tools/mma_issue.bin
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace eps_k;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(pred));
  return pred != 0;
}

template <int N>
__global__ void mma_bench(int iters, long long* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* a = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* b = a + 128 * 128;
  for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(a)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t idesc = umma_idesc_bf16(128, N, false, false);
  long long t0 = clock64();
  if (warp == 0) {
    if (mode == 0) {
      if (lane == 0) {
        for (int i = 0; i < iters; ++i)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_bf16(tmem, umma_sdesc(smem_addr(a) + kk * 32, 16, 1024),
                        umma_sdesc(smem_addr(b) + kk * 32, 16, 1024), idesc, (i | kk) ? 1u : 0u);
        tc_commit(&bar);
      }
    } else if (mode == 2) {
      // one lane, descriptors precomputed (uniform arithmetic only)
      const uint64_t da = umma_sdesc(smem_addr(a), 16, 1024), db = umma_sdesc(smem_addr(b), 16, 1024);
      if (lane == 0) {
        for (int i = 0; i < iters; ++i)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            tc_mma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, (i | kk) ? 1u : 0u);
        tc_commit(&bar);
      }
    } else {
      const uint64_t da = umma_sdesc(smem_addr(a), 16, 1024), db = umma_sdesc(smem_addr(b), 16, 1024);
      for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          if (elect_one())
            tc_mma_bf16(tmem, da + 2 * kk, db + 2 * kk, idesc, (i | kk) ? 1u : 0u);
      if (elect_one()) tc_commit(&bar);
    }
    __syncwarp();
    long long t1 = clock64();
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (lane == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N>
void run(long long* d) {
  const int smem = (128 + N) * 128 + 2048;
  cudaFuncSetAttribute(mma_bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 0; mode < 3; ++mode) {
    const int iters = 1000;
    mma_bench<N><<<1, 128, smem>>>(iters, d, mode);
    cudaDeviceSynchronize();
    long long c[2];
    cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
    printf("N=%3d mode=%d  issue %.1f cyc/mma, complete %.1f cyc/mma (floor %d)\n", N, mode,
           double(c[0]) / (4 * iters), double(c[1]) / (4 * iters), 128 * N / 256);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<64>(d);
  run<128>(d);
  run<256>(d);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
