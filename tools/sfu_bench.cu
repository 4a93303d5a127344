// Microbenchmark: per-SM throughput of the softmax instruction mix on B200.
//   ex2.approx.f32, ex2.approx.f16x2, tanh.approx.f32, FFMA (3-reg), FFMA2
// Each thread runs 8 independent dependency chains; one block of `threads`
// per SM; result = lane-operations per SM clock (clock64 inside the block).
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/sfu_bench.cu -o tools/sfu_bench.bin
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int OP>
__global__ void bench(int iters, float seed, float* sink, long long* cyc) {
  float v[8];
  float2 w[8];
  uint32_t h[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    v[j] = seed * (threadIdx.x + j) * 1e-6f - 0.5f;
    w[j] = make_float2(v[j], v[j] + 0.25f);
    const __half2 hh = __floats2half2_rn(v[j], v[j] * 0.5f);
    h[j] = *reinterpret_cast<const uint32_t*>(&hh);
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if constexpr (OP == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[j]));
      } else if constexpr (OP == 1) {
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[j]));
      } else if constexpr (OP == 2) {
        asm volatile("tanh.approx.f32 %0, %0;" : "+f"(v[j]));
      } else if constexpr (OP == 3) {
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(v[j]) : "f"(w[j].x), "f"(w[j].y));
      } else if constexpr (OP == 4) {
        w[j] = __ffma2_rn(w[j], w[(j + 1) & 7], w[(j + 2) & 7]);
      } else if constexpr (OP == 5) {
        // the fwd softmax inner step: FFMA2 -> 2x ex2 -> FADD2 -> F2FP
        const float2 a = __ffma2_rn(w[j], make_float2(0.18f, 0.18f), make_float2(-1.f, -1.f));
        float e0, e1;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(a.x));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(a.y));
        w[(j + 3) & 7] = __fadd2_rn(w[(j + 3) & 7], make_float2(e0, e1));
        uint32_t pk;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(pk) : "f"(e1), "f"(e0));
        h[j] ^= pk;
      }
    }
  }
  const long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) acc += v[j] + w[j].x + w[j].y + __uint_as_float(h[j]);
  if (acc == 12345.f) sink[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads, int lanes_per_op) {
  float* sink;
  long long* cyc;
  cudaMalloc(&sink, 4096 * sizeof(float));
  cudaMalloc(&cyc, 148 * sizeof(long long));
  const int iters = 4096;
  bench<OP><<<148, threads>>>(iters, 1.f, sink, cyc);
  bench<OP><<<148, threads>>>(iters, 1.f, sink, cyc);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += double(c[i]) / 148;
  const double ops = double(iters) * 8 * threads * lanes_per_op;
  printf("{\"op\": \"%s\", \"threads\": %d, \"lane_ops_per_sm_clk\": %.2f}\n", name, threads,
         ops / avg);
  cudaFree(sink);
  cudaFree(cyc);
}

int main() {
  for (int t : {128, 256, 512, 1024}) {
    run<0>("ex2.f32", t, 1);
    run<1>("ex2.f16x2 (results)", t, 2);
    run<2>("tanh.f32", t, 1);
    run<3>("ffma", t, 1);
    run<4>("ffma2 (flops/2)", t, 2);
    run<5>("softmax step (exp results)", t, 2);
  }
  return 0;
}
