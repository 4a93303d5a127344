// Microbenchmark: tcgen05.mma completion rate for the attention-forward MMA
// shapes (M = 128, K = 16), SS vs TS (A = P from TMEM), with and without
// concurrent tcgen05.ld traffic from 8 "softmax" warps.
//   nvcc -std=c++20 -gencode arch=compute_100a,code=sm_100a -I paper_2102_03161_b200/csrc/kernels \
//        -Iinclude tools/mma_rate.cu -o /tmp/mma_rate -lcuda
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"

using namespace eps_k;

__global__ void __launch_bounds__(384, 1) mma_rate(int iters, int n, int ts, int loaders,
                                                  int nd, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    const uint64_t a = umma_sdesc(smem_addr(smem), 16, 1024);
    const uint64_t b = umma_sdesc(smem_addr(smem + 32768), 16, 1024);
    const uint64_t bmn = umma_sdesc(smem_addr(smem + 32768), 64 * 128, 1024);
    const uint32_t idesc = umma_idesc_bf16(128, n, false, ts != 0);
    long long t0 = clock64();
    if (nd <= 0) {  // unrolled by 8, constant descriptor offsets (GEMM-mainloop style);
                    // nd = -k: k distinct accumulators in rotation
      const int k = nd == 0 ? 1 : -nd;
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t dcol = k == 1 ? 0u : k == 2 ? uint32_t((u & 1) * 64) : uint32_t((u & 3) * 64);
          if (ts)
            tc_mma_ts_ws(tmem + 256 + (n <= 64 ? dcol : 0u), tmem + uint32_t(u * 8), bmn, idesc, 1u);
          else
            tc_mma_ss_ws(tmem + 256 + (n <= 64 ? dcol : 0u), a + uint64_t(2 * (u & 3)), b + uint64_t(2 * (u & 3)), idesc, 1u);
        }
      }
    } else {
      for (int i = 0; i < iters; ++i) {
        if (ts)
          tc_mma_ts_ws(tmem + 256 + uint32_t((i % nd) * 64), tmem + uint32_t((i & 7) * 8), bmn, idesc, 1u);
        else
          tc_mma_ss_ws(tmem + 256 + uint32_t((i % nd) * (n <= 64 ? 64 : 0)), a + uint64_t(2 * (i & 3)), b + uint64_t(2 * (i & 3)), idesc, 1u);
      }
    }
    long long t1 = clock64();
    tc_commit_ws(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (lane == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
      done = 1;
    }
  } else if (warp >= 4 && warp - 4 < loaders) {
    const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(64 + 32 * ((warp >> 2) & 1));
    uint32_t acc = 0;
    while (!done) {
      uint32_t r[32];
      tmem_ld_32x32(base, r);
      tmem_ld_wait_regs(r);
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += r[j];
    }
    if (acc == 12345) out[2] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// cta_group::2 (cluster of 2): M = 256 (128 rows per CTA), N, K = 16; and
// cta_group::1 M = 64 for comparison.
__device__ __forceinline__ void tc_mma_pair_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// mode: 0 SS K-major, 1 TS (A from TMEM, B MN-major SW128), 2 SS A MN-major + B MN-major
template <int mode>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_rate_pair(int iters, int n, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc_pair(&slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1 && rank == 0) {
    const uint64_t a = umma_sdesc(smem_addr(smem), 16, 1024);
    const uint64_t b = umma_sdesc(smem_addr(smem + 32768), 16, 1024);
    const uint64_t amn = umma_sdesc(smem_addr(smem), 64 * 128, 1024);
    const uint64_t bmn = umma_sdesc(smem_addr(smem + 32768), 64 * 128, 1024);
    const uint32_t idesc = umma_idesc_bf16(256, n, mode == 2, mode >= 1);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (lane == 0) {
          if constexpr (mode == 0)
            tc_mma_pair(tmem + 256, a + uint64_t(2 * (u & 3)), b + uint64_t(2 * (u & 3)), idesc, 1u);
          else if constexpr (mode == 1)
            tc_mma_pair_ts(tmem + 256, tmem + uint32_t(u * 8), bmn + uint64_t(128 * (u & 3)), idesc, 1u);
          else
            tc_mma_pair(tmem + 256, amn + uint64_t(128 * (u & 3)), bmn + uint64_t(128 * (u & 3)), idesc, 1u);
        }
        __syncwarp();
      }
    }
    long long t1 = clock64();
    if (lane == 0) tc_commit_pair(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (lane == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  } else if (warp == 1) {
    mbar_wait(&bar, 0);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
  }
}

__global__ void __launch_bounds__(128, 1) mma_rate_m64(int iters, int n, long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    const uint64_t a = umma_sdesc(smem_addr(smem), 16, 1024);
    const uint64_t b = umma_sdesc(smem_addr(smem + 32768), 16, 1024);
    const uint32_t idesc = umma_idesc_bf16(64, n, false, false);
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u)
        tc_mma_ss_ws(tmem + 256, a + uint64_t(2 * (u & 3)), b + uint64_t(2 * (u & 3)), idesc, 1u);
    }
    long long t1 = clock64();
    tc_commit_ws(&bar);
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

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  for (int ts = 0; ts < 2; ++ts)
    for (int n : {16, 64, 128, 208, 256}) {
      if (ts && n != 64) continue;
      for (int nd : {0, -2, -4})
      for (int loaders : {0, 8}) {
        if (nd != 0 && n > 64) continue;
        if (loaders && nd != 0) continue;
        mma_rate<<<1, 384, 100 * 1024>>>(iters, n, ts, loaders, nd, d);
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%s N=%3d accumulators=%d loaders=%d: issue %.1f, complete %.1f cycles/MMA\n",
               ts ? "TS" : "SS", n, nd, loaders, double(h[0]) / iters, double(h[1]) / iters);
      }
    }
  cudaFuncSetAttribute(mma_rate_pair<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(mma_rate_pair<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(mma_rate_pair<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaFuncSetAttribute(mma_rate_m64, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {32, 64, 128, 256}) {
      if (mode == 0) mma_rate_pair<0><<<2, 128, 100 * 1024>>>(iters, n, d);
      if (mode == 1) mma_rate_pair<1><<<2, 128, 100 * 1024>>>(iters, n, d);
      if (mode == 2) mma_rate_pair<2><<<2, 128, 100 * 1024>>>(iters, n, d);
      long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("PAIR %s M=256 N=%3d: issue %.1f, complete %.1f cycles/MMA (%s)\n",
             mode == 0 ? "SS" : mode == 1 ? "TS" : "SS-MN", n, double(h[0]) / iters,
             double(h[1]) / iters, cudaGetErrorString(cudaGetLastError()));
    }
  for (int n : {32, 64, 128, 256}) {
    mma_rate_m64<<<1, 128, 100 * 1024>>>(iters, n, d);
    long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("M=64 N=%3d: issue %.1f, complete %.1f cycles/MMA (%s)\n", n, double(h[0]) / iters,
           double(h[1]) / iters, cudaGetErrorString(cudaGetLastError()));
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
