// LayerNorm forward / backward (HBM-bound; one warp per row, 16B vector
// accesses, warp-shuffle reductions, fp32 statistics).
//
// Backward fuses the residual branch (dx = dres + LN'(dy)), the dgamma /
// dbeta column reductions and the column sum of the produced dx, which is
// the bias gradient of the sublayer whose output bias feeds this residual
// stream ("backward dataflow").
#include <cuda_runtime.h>

#include "eps_capi.h"
#include "ptx.cuh"

namespace eps_k {

constexpr int kLnWarps = 8;

// Elements per lane EPL = d / 32; a lane owns EPL/VEC vectors of VEC bf16,
// vector v of lane l covering columns (v * 32 + l) * VEC ... + VEC - 1.
template <int EPL>
struct LnShape {
  static constexpr int VEC = (EPL % 8 == 0) ? 8 : 4;
  static constexpr int NV = EPL / VEC;
};

template <int VEC>
__device__ __forceinline__ void load_vec(const uint16_t* p, float* out) {
  if constexpr (VEC == 8) {
    const uint4 w = *reinterpret_cast<const uint4*>(p);
    out[0] = bf16_lo(w.x); out[1] = bf16_hi(w.x); out[2] = bf16_lo(w.y); out[3] = bf16_hi(w.y);
    out[4] = bf16_lo(w.z); out[5] = bf16_hi(w.z); out[6] = bf16_lo(w.w); out[7] = bf16_hi(w.w);
  } else {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
    out[0] = bf16_lo(w.x); out[1] = bf16_hi(w.x); out[2] = bf16_lo(w.y); out[3] = bf16_hi(w.y);
  }
}

template <int VEC>
__device__ __forceinline__ void store_vec(uint16_t* p, const float* v) {
  if constexpr (VEC == 8) {
    *reinterpret_cast<uint4*>(p) = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                                              pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
  } else {
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]));
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int EPL>
__global__ void __launch_bounds__(kLnWarps * 32)
    ln_fwd_kernel(const uint16_t* __restrict__ x, const float* __restrict__ gamma,
                  const float* __restrict__ beta, uint16_t* __restrict__ y,
                  float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows,
                  float eps) {
  using S = LnShape<EPL>;
  constexpr int D = EPL * 32;
  const int lane = threadIdx.x & 31;
  const int64_t row = int64_t(blockIdx.x) * kLnWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint16_t* xr = x + row * D;
  float v[EPL];
#pragma unroll
  for (int i = 0; i < S::NV; ++i) load_vec<S::VEC>(xr + (i * 32 + lane) * S::VEC, v + i * S::VEC);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) s += v[i];
  const float mu = warp_sum(s) * (1.0f / D);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < EPL; ++i) {
    const float d = v[i] - mu;
    q += d * d;
  }
  const float rs = rsqrtf(warp_sum(q) * (1.0f / D) + eps);
  float o[EPL];
#pragma unroll
  for (int i = 0; i < S::NV; ++i) {
    // gamma / beta as 16B vectors (VEC consecutive columns per lane)
    const float4* g4 = reinterpret_cast<const float4*>(gamma + (i * 32 + lane) * S::VEC);
    const float4* b4 = reinterpret_cast<const float4*>(beta + (i * 32 + lane) * S::VEC);
#pragma unroll
    for (int j4 = 0; j4 < S::VEC / 4; ++j4) {
      const float4 gg = __ldg(g4 + j4), bb = __ldg(b4 + j4);
      float* vo = o + i * S::VEC + 4 * j4;
      const float* vi = v + i * S::VEC + 4 * j4;
      vo[0] = (vi[0] - mu) * rs * gg.x + bb.x;
      vo[1] = (vi[1] - mu) * rs * gg.y + bb.y;
      vo[2] = (vi[2] - mu) * rs * gg.z + bb.z;
      vo[3] = (vi[3] - mu) * rs * gg.w + bb.w;
    }
  }
  uint16_t* yr = y + row * D;
#pragma unroll
  for (int i = 0; i < S::NV; ++i) store_vec<S::VEC>(yr + (i * 32 + lane) * S::VEC, o + i * S::VEC);
  if (lane == 0) {
    mean_out[row] = mu;
    rstd_out[row] = rs;
  }
}

// Grid-stride over rows; per-lane column partials of dgamma, dbeta and
// colsum(dx) are reduced across the block in smem, then one atomic per
// column per block.
template <int EPL>
__global__ void __launch_bounds__(kLnWarps * 32)
    ln_bwd_kernel(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ x,
                  const float* __restrict__ gamma, const float* __restrict__ mean,
                  const float* __restrict__ rstd, const uint16_t* __restrict__ dres,
                  uint16_t* __restrict__ dx, float* __restrict__ dgamma,
                  float* __restrict__ dbeta, float* __restrict__ colsum, int64_t rows) {
  using S = LnShape<EPL>;
  constexpr int D = EPL * 32;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  float acc_g[EPL], acc_b[EPL], acc_c[EPL], gam[EPL];
#pragma unroll
  for (int i = 0; i < S::NV; ++i)
#pragma unroll
    for (int j = 0; j < S::VEC; ++j) {
      acc_g[i * S::VEC + j] = acc_b[i * S::VEC + j] = acc_c[i * S::VEC + j] = 0.f;
      gam[i * S::VEC + j] = __ldg(gamma + (i * 32 + lane) * S::VEC + j);
    }
  for (int64_t row = int64_t(blockIdx.x) * kLnWarps + warp; row < rows;
       row += int64_t(gridDim.x) * kLnWarps) {
    float g[EPL], xv[EPL], r[EPL];
#pragma unroll
    for (int i = 0; i < S::NV; ++i) {
      load_vec<S::VEC>(dy + row * D + (i * 32 + lane) * S::VEC, g + i * S::VEC);
      load_vec<S::VEC>(x + row * D + (i * 32 + lane) * S::VEC, xv + i * S::VEC);
    }
    // all of the row's loads in flight at once (one HBM round trip per row)
    if (dres != nullptr) {
#pragma unroll
      for (int i = 0; i < S::NV; ++i)
        load_vec<S::VEC>(dres + row * D + (i * 32 + lane) * S::VEC, r + i * S::VEC);
    } else {
#pragma unroll
      for (int i = 0; i < EPL; ++i) r[i] = 0.f;
    }
    const float mu = __ldg(mean + row), rs = __ldg(rstd + row);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      const float xh = (xv[i] - mu) * rs;
      xv[i] = xh;
      acc_g[i] += g[i] * xh;
      acc_b[i] += g[i];
      const float gg = g[i] * gam[i];
      g[i] = gg;
      s1 += gg;
      s2 += gg * xh;
    }
    s1 = warp_sum(s1) * (1.0f / D);
    s2 = warp_sum(s2) * (1.0f / D);
#pragma unroll
    for (int i = 0; i < EPL; ++i) {
      r[i] += rs * (g[i] - s1 - xv[i] * s2);
      // column sums from the fp32 value (bias grads are sums over many rows
      // that cancel; summing bf16-rounded rows would add ~2^-9 sqrt(rows) noise)
      acc_c[i] += r[i];
    }
    if (dx != nullptr) {
#pragma unroll
      for (int i = 0; i < S::NV; ++i)
        store_vec<S::VEC>(dx + row * D + (i * 32 + lane) * S::VEC, r + i * S::VEC);
    }
  }
  // block reduction of the three column accumulators
  extern __shared__ float red[];  // [kLnWarps][3][D]
#pragma unroll
  for (int i = 0; i < S::NV; ++i)
#pragma unroll
    for (int j = 0; j < S::VEC; ++j) {
      const int col = (i * 32 + lane) * S::VEC + j;
      red[(warp * 3 + 0) * D + col] = acc_g[i * S::VEC + j];
      red[(warp * 3 + 1) * D + col] = acc_b[i * S::VEC + j];
      red[(warp * 3 + 2) * D + col] = acc_c[i * S::VEC + j];
    }
  __syncthreads();
  for (int c = threadIdx.x; c < 3 * D; c += blockDim.x) {
    const int which = c / D, col = c % D;
    float s = 0.f;
    for (int w = 0; w < kLnWarps; ++w) s += red[(w * 3 + which) * D + col];
    float* dst = which == 0 ? dgamma : which == 1 ? dbeta : colsum;
    if (dst != nullptr) atomicAdd(dst + col, s);
  }
}

int ln_grid_bwd(int64_t rows) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (rows + kLnWarps - 1) / kLnWarps;
  return int(need < 2 * sms ? need : 2 * sms);
}

template <int EPL>
int ln_launch(const void* x, const float* gamma, const float* beta, void* y, float* mean,
              float* rstd, int64_t rows, float eps, cudaStream_t st) {
  const int64_t blocks = (rows + kLnWarps - 1) / kLnWarps;
  count_launch(); ln_fwd_kernel<EPL><<<unsigned(blocks), kLnWarps * 32, 0, st>>>(
      static_cast<const uint16_t*>(x), gamma, beta, static_cast<uint16_t*>(y), mean, rstd, rows,
      eps);
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

template <int EPL>
int ln_bwd_launch(const void* dy, const void* x, const float* gamma, const float* mean,
                  const float* rstd, const void* dres, void* dx, float* dgamma, float* dbeta,
                  float* colsum, int64_t rows, cudaStream_t st) {
  constexpr int D = EPL * 32;
  const size_t smem = size_t(kLnWarps) * 3 * D * sizeof(float);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(ln_bwd_kernel<EPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    configured = true;
  }
  count_launch(); ln_bwd_kernel<EPL><<<ln_grid_bwd(rows), kLnWarps * 32, smem, st>>>(
      static_cast<const uint16_t*>(dy), static_cast<const uint16_t*>(x), gamma, mean, rstd,
      static_cast<const uint16_t*>(dres), static_cast<uint16_t*>(dx), dgamma, dbeta, colsum,
      rows);
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

}  // namespace eps_k

extern "C" int eps_layernorm_fwd(const void* x, const float* gamma, const float* beta, void* y,
                                 float* mean, float* rstd, int64_t rows, int64_t d, float eps,
                                 void* stream) {
  using namespace eps_k;
  if (rows <= 0) return EPS_OK;
  auto st = static_cast<cudaStream_t>(stream);
  switch (d) {
    case 128: return ln_launch<4>(x, gamma, beta, y, mean, rstd, rows, eps, st);
    case 256: return ln_launch<8>(x, gamma, beta, y, mean, rstd, rows, eps, st);
    case 768: return ln_launch<24>(x, gamma, beta, y, mean, rstd, rows, eps, st);
    case 1024: return ln_launch<32>(x, gamma, beta, y, mean, rstd, rows, eps, st);
    default: return EPS_EINVAL;
  }
}

extern "C" int eps_layernorm_bwd(const void* dy, const void* x, const float* gamma,
                                 const float* mean, const float* rstd, const void* dres,
                                 void* dx, float* dgamma, float* dbeta, float* colsum_dx,
                                 int64_t rows, int64_t d, float* workspace, void* stream) {
  using namespace eps_k;
  (void)workspace;
  if (rows <= 0) return EPS_OK;
  auto st = static_cast<cudaStream_t>(stream);
  switch (d) {
    case 128:
      return ln_bwd_launch<4>(dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta, colsum_dx, rows, st);
    case 256:
      return ln_bwd_launch<8>(dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta, colsum_dx, rows, st);
    case 768:
      return ln_bwd_launch<24>(dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta, colsum_dx, rows, st);
    case 1024:
      return ln_bwd_launch<32>(dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta, colsum_dx, rows, st);
    default:
      return EPS_EINVAL;
  }
}
