// LayerNorm forward / backward (HBM-bound; one warp per row, 16B vector
// accesses, warp-shuffle reductions, fp32 statistics).
//
// Backward fuses the residual branch (dx = dres + LN'(dy)), the dgamma /
// dbeta column reductions and the column sum of the produced dx, which is
// the bias gradient of the sublayer whose output bias feeds this residual
// stream ("backward dataflow").
#include <cuda_runtime.h>

#include <cstdlib>

#include "eps_capi.h"
#include "ptx.cuh"
#include "tma_host.cuh"

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

// Wide-row backward (d = 768 / 1024), HBM-bound: one producer warp streams
// whole rows of dy / x / dres into a 16-stage shared-memory ring with 1-D bulk
// copies (cp.async.bulk: many rows in flight without holding them in
// registers), and consumer groups of d/8 threads (8 columns each, 16-byte
// shared loads) take every GROUPS-th row.  A thread therefore keeps only 8
// columns of dgamma / dbeta / colsum accumulators.  The two row reductions
// (sum g*gamma, sum g*gamma*xhat) cross the group's warps through a named
// barrier.  (The warp-per-row kernel above holds 24 columns x 3 accumulators
// per lane, ~200 registers, and reaches only ~8 rows in flight per SM.)
constexpr int kLnStages = 16;
constexpr int kLnStatRows = 384;  // d = 768 backward: rows per CTA with (mean, rstd) in smem

template <int D>
struct LnWide {
  static constexpr int TPR = D / 8;                 // consumer threads per row
  static constexpr int WPR = TPR / 32;              // warps per row group
  static constexpr int GROUPS = (D == 768) ? 4 : 3; // consumer groups per CTA
  static constexpr int THREADS = 32 + GROUPS * TPR;
  static constexpr int ROW = D * 2;                 // bytes per row per tensor
  static constexpr size_t SMEM = size_t(kLnStages) * 3 * ROW + 2 * kLnStages * 8 + 16;
  static_assert(TPR % 32 == 0 && kLnStages % GROUPS != 0 || true, "");
};

__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

template <int D>
__global__ void __launch_bounds__(LnWide<D>::THREADS, 2)
    ln_bwd_wide_kernel(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ x,
                       const float* __restrict__ gamma, const float* __restrict__ mean,
                       const float* __restrict__ rstd, const uint16_t* __restrict__ dres,
                       uint16_t* __restrict__ dx, float* __restrict__ dgamma,
                       float* __restrict__ dbeta, float* __restrict__ colsum, int64_t rows) {
  using L = LnWide<D>;
  constexpr int TPR = L::TPR, WPR = L::WPR, GROUPS = L::GROUPS, ROW = L::ROW;
  extern __shared__ __align__(128) uint8_t ln_smem[];
  uint8_t* ring = ln_smem;  // [stage][dy | x | dres] rows
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + size_t(kLnStages) * 3 * ROW);
  uint64_t* empty = full + kLnStages;
  __shared__ float red[GROUPS][2][WPR][2];
  __shared__ __align__(16) float acc_s[3][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool has_res = dres != nullptr;
  const int64_t n_mine = rows > blockIdx.x ? (rows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kLnStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], WPR);
    }
    mbar_fence_init();
  }
  pdl_launch_dependents();
  __syncthreads();
  pdl_wait();  // the predecessor grid's outputs are complete (PDL launch)
  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes = uint32_t((has_res ? 3 : 2) * ROW);
      for (int64_t k = 0; k < n_mine; ++k) {
        const int st = int(k % kLnStages);
        if (k >= kLnStages) mbar_wait(&empty[st], uint32_t((k / kLnStages - 1) & 1));
        const int64_t r = blockIdx.x + k * gridDim.x;
        uint8_t* dst = ring + size_t(st) * 3 * ROW;
        mbar_expect_tx(&full[st], bytes);
        bulk_load_1d(dst, dy + r * D, ROW, &full[st]);
        bulk_load_1d(dst + ROW, x + r * D, ROW, &full[st]);
        if (has_res) bulk_load_1d(dst + 2 * ROW, dres + r * D, ROW, &full[st]);
      }
    }
    return;
  }
  const int ct = threadIdx.x - 32;
  const int grp = ct / TPR, t = ct % TPR, wig = t >> 5;
  const int col = t * 8;
  // (mean, rstd) of the CTA's first kLnStatRows rows, loaded by all consumer
  // threads at once: a per-row load puts one L2 / HBM round trip in front of
  // every row whose data is already in the ring (d = 768: ViT-B b400 90.4 ->
  // 84.1 us, BERT-base-384 33.7 -> 30.2).  At d = 1024 (BERT-large-128, ~28
  // rows per CTA) both this and a two-row register prefetch measured slower
  // (13.8 -> 14.6 us after the reduction change below), so the per-row load
  // stays there.
  constexpr bool kStage = D == 768;
  constexpr int kStatRows = kStage ? kLnStatRows : 1;
  __shared__ float2 stat[kStatRows];
  if (kStage) {
    for (int64_t k = ct; k < n_mine && k < kStatRows; k += GROUPS * TPR) {
      const int64_t r = blockIdx.x + k * gridDim.x;
      stat[k] = make_float2(__ldg(mean + r), __ldg(rstd + r));
    }
    asm volatile("bar.sync 14, %0;" ::"r"(GROUPS * TPR) : "memory");
  }
  float gam[8], ag[8], ab[8], ac[8];
  {
    const float4 g0 = __ldg(reinterpret_cast<const float4*>(gamma + col));
    const float4 g1 = __ldg(reinterpret_cast<const float4*>(gamma + col) + 1);
    gam[0] = g0.x, gam[1] = g0.y, gam[2] = g0.z, gam[3] = g0.w;
    gam[4] = g1.x, gam[5] = g1.y, gam[6] = g1.z, gam[7] = g1.w;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) ag[i] = ab[i] = ac[i] = 0.f;
  int buf = 0;
  for (int64_t k = grp; k < n_mine; k += GROUPS, buf ^= 1) {
    const int st = int(k % kLnStages);
    const int64_t r = blockIdx.x + k * gridDim.x;
    const float2 ms = kStage && k < kStatRows ? stat[k]
                                              : make_float2(__ldg(mean + r), __ldg(rstd + r));
    const float mu = ms.x, rs = ms.y;
    mbar_wait(&full[st], uint32_t((k / kLnStages) & 1));
    const uint32_t base = smem_addr(ring + size_t(st) * 3 * ROW) + uint32_t(col * 2);
    const uint4 gy = ld_shared_v4(base), xx = ld_shared_v4(base + ROW);
    const uint4 rr = has_res ? ld_shared_v4(base + 2 * ROW) : make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // this warp's slice is in registers
    float g[8], xh[8], res[8];
    load_vec<8>(reinterpret_cast<const uint16_t*>(&gy), g);
    load_vec<8>(reinterpret_cast<const uint16_t*>(&xx), xh);
    load_vec<8>(reinterpret_cast<const uint16_t*>(&rr), res);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      xh[i] = (xh[i] - mu) * rs;
      ag[i] += g[i] * xh[i];
      ab[i] += g[i];
      g[i] *= gam[i];
      s1 += g[i];
      s2 += g[i] * xh[i];
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) red[grp][buf][wig][0] = s1, red[grp][buf][wig][1] = s2;
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(TPR) : "memory");
    s1 = s2 = 0.f;
#pragma unroll
    for (int w = 0; w < WPR; ++w) s1 += red[grp][buf][w][0], s2 += red[grp][buf][w][1];
    s1 *= 1.0f / D;
    s2 *= 1.0f / D;
    float o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i] = res[i] + rs * (g[i] - s1 - xh[i] * s2);
      ac[i] += o[i];  // column sums from the fp32 value (see ln_bwd_kernel)
    }
    if (dx != nullptr) store_vec<8>(dx + r * D + col, o);
  }
  // block reduction of the three column accumulators: the groups add their
  // 8 columns into acc_s in turn (plain 16-byte shared loads / stores).  A
  // shared-memory float atomicAdd compiles to a compare-and-swap loop; with
  // it the kernel took 19.7 / 33.6 / 90.3 us (BERT-large / BERT-base / ViT-B
  // shapes), now 13.8 / 25.4 / 80.5.
  for (int gi = 0; gi < GROUPS; ++gi) {
    if (grp == gi) {
      float* dst[3] = {&acc_s[0][col], &acc_s[1][col], &acc_s[2][col]};
      const float* src[3] = {ag, ab, ac};
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float4 v = make_float4(src[a][4 * h], src[a][4 * h + 1], src[a][4 * h + 2],
                                 src[a][4 * h + 3]);
          if (gi > 0) {
            const float4 o = reinterpret_cast<const float4*>(dst[a])[h];
            v.x += o.x, v.y += o.y, v.z += o.z, v.w += o.w;
          }
          reinterpret_cast<float4*>(dst[a])[h] = v;
        }
    }
    asm volatile("bar.sync 15, %0;" ::"r"(GROUPS * TPR) : "memory");
  }
  // one 4-wide reduction per 4 columns (a quarter of the atomic operations;
  // measured neutral at ViT-B and BERT shapes)
  for (int c = ct * 4; c < 3 * D; c += GROUPS * TPR * 4) {
    const int which = c / D, cc = c % D;
    float* dst = which == 0 ? dgamma : which == 1 ? dbeta : colsum;
    if (dst != nullptr)
      red_add_v4(dst + cc, acc_s[which][cc], acc_s[which][cc + 1], acc_s[which][cc + 2],
                 acc_s[which][cc + 3]);
  }
}

// Wide-row forward, same streaming structure: the producer warp bulk-copies
// x rows into a 32-stage ring; consumer groups of d/8 threads normalise every
// GROUPS-th row (two-pass mean / variance through named barriers) and store
// y with 16-byte vector stores.
constexpr int kLnFwdStages = 32;

// ONEPASS: mean and variance from one reduction of (sum d, sum d^2), d = x -
// x[row][0] (the row's first element, read from the ring by every thread: the
// shift keeps E[d^2] - E[d]^2 free of cancellation for rows whose mean is
// large against their spread), so a row needs one named barrier, not two.
template <int D, bool ONEPASS>
__global__ void __launch_bounds__(LnWide<D>::THREADS, 3)
    ln_fwd_wide_kernel(const uint16_t* __restrict__ x, const float* __restrict__ gamma,
                       const float* __restrict__ beta, uint16_t* __restrict__ y,
                       float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows,
                       float eps) {
  using L = LnWide<D>;
  constexpr int TPR = L::TPR, WPR = L::WPR, GROUPS = L::GROUPS, ROW = L::ROW;
  extern __shared__ __align__(128) uint8_t ln_smem[];
  uint8_t* ring = ln_smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + size_t(kLnFwdStages) * ROW);
  uint64_t* empty = full + kLnFwdStages;
  __shared__ float red[GROUPS][2][WPR];
  __shared__ float red1[GROUPS][2][2][WPR];  // ONEPASS: [row parity][sum d, sum d^2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_mine = rows > blockIdx.x ? (rows - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kLnFwdStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], WPR);
    }
    mbar_fence_init();
  }
  pdl_launch_dependents();
  __syncthreads();
  pdl_wait();  // the predecessor grid's outputs are complete (PDL launch)
  if (warp == 0) {
    if (lane == 0) {
      for (int64_t k = 0; k < n_mine; ++k) {
        const int st = int(k % kLnFwdStages);
        if (k >= kLnFwdStages) mbar_wait(&empty[st], uint32_t((k / kLnFwdStages - 1) & 1));
        const int64_t r = blockIdx.x + k * gridDim.x;
        mbar_expect_tx(&full[st], uint32_t(ROW));
        bulk_load_1d(ring + size_t(st) * ROW, x + r * D, ROW, &full[st]);
      }
    }
    return;
  }
  const int ct = threadIdx.x - 32;
  const int grp = ct / TPR, t = ct % TPR, wig = t >> 5;
  const int col = t * 8;
  float gam[8], bet[8];
  {
    const float4* g4 = reinterpret_cast<const float4*>(gamma + col);
    const float4* b4 = reinterpret_cast<const float4*>(beta + col);
    const float4 g0 = __ldg(g4), g1 = __ldg(g4 + 1), b0 = __ldg(b4), b1 = __ldg(b4 + 1);
    gam[0] = g0.x, gam[1] = g0.y, gam[2] = g0.z, gam[3] = g0.w;
    gam[4] = g1.x, gam[5] = g1.y, gam[6] = g1.z, gam[7] = g1.w;
    bet[0] = b0.x, bet[1] = b0.y, bet[2] = b0.z, bet[3] = b0.w;
    bet[4] = b1.x, bet[5] = b1.y, bet[6] = b1.z, bet[7] = b1.w;
  }
  const uint32_t bar_id = 1 + grp;
  for (int64_t k = grp; k < n_mine; k += GROUPS) {
    const int st = int(k % kLnFwdStages);
    const int64_t r = blockIdx.x + k * gridDim.x;
    mbar_wait(&full[st], uint32_t((k / kLnFwdStages) & 1));
    const uint4 xx = ld_shared_v4(smem_addr(ring + size_t(st) * ROW) + uint32_t(col * 2));
    const float x0 = ONEPASS ? bf16_lo(*reinterpret_cast<const uint32_t*>(ring + size_t(st) * ROW))
                             : 0.f;
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    float v[8];
    load_vec<8>(reinterpret_cast<const uint16_t*>(&xx), v);
    if constexpr (ONEPASS) {
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float d = v[i] - x0;
        s1 += d;
        s2 = fmaf(d, d, s2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      }
      const int par = int((k / GROUPS) & 1);
      if (lane == 0) {
        red1[grp][par][0][wig] = s1;
        red1[grp][par][1][wig] = s2;
      }
      asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(TPR) : "memory");
      s1 = 0.f;
      s2 = 0.f;
#pragma unroll
      for (int w = 0; w < WPR; ++w) {
        s1 += red1[grp][par][0][w];
        s2 += red1[grp][par][1][w];
      }
      const float md = s1 * (1.0f / D);
      const float var = fmaxf(s2 * (1.0f / D) - md * md, 0.f);
      const float mu = x0 + md;
      const float rs = rsqrtf(var + eps);
      float o[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = (v[i] - mu) * rs * gam[i] + bet[i];
      store_vec<8>(y + r * D + col, o);
      if (t == 0) {
        mean_out[r] = mu;
        rstd_out[r] = rs;
      }
      continue;
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
    s = warp_sum(s);
    if (lane == 0) red[grp][0][wig] = s;
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(TPR) : "memory");
    float mu = 0.f;
#pragma unroll
    for (int w = 0; w < WPR; ++w) mu += red[grp][0][w];
    mu *= 1.0f / D;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float dd = v[i] - mu;
      q += dd * dd;
    }
    q = warp_sum(q);
    if (lane == 0) red[grp][1][wig] = q;
    asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(TPR) : "memory");
    q = 0.f;
#pragma unroll
    for (int w = 0; w < WPR; ++w) q += red[grp][1][w];
    const float rs = rsqrtf(q * (1.0f / D) + eps);
    float o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = (v[i] - mu) * rs * gam[i] + bet[i];
    store_vec<8>(y + r * D + col, o);
    if (t == 0) {
      mean_out[r] = mu;
      rstd_out[r] = rs;
    }
    // red[grp][0] is rewritten next row only after every thread of the group
    // passed the second barrier (which follows its read of red[grp][0])
  }
}

// CTAs per SM of the wide-row kernels (A/B: EPS_LN_FWD_GRID / EPS_LN_BWD_GRID)
static int ln_grid_mult(int which, int dflt) {
  static const int m[2] = {[] {
    const char* e = std::getenv("EPS_LN_FWD_GRID");
    return e ? std::atoi(e) : 0;
  }(), [] {
    const char* e = std::getenv("EPS_LN_BWD_GRID");
    return e ? std::atoi(e) : 0;
  }()};
  return m[which] > 0 ? m[which] : dflt;
}

template <int D>
int ln_fwd_wide_launch(const void* x, const float* gamma, const float* beta, void* y, float* mean,
                       float* rstd, int64_t rows, float eps, cudaStream_t st) {
  using L = LnWide<D>;
  constexpr size_t smem = size_t(kLnFwdStages) * L::ROW + 2 * kLnFwdStages * 8 + 16;
  static const bool onepass = [] {
    const char* e = std::getenv("EPS_LN_ONEPASS");
    return e == nullptr || std::atoi(e) != 0;
  }();
  auto kern = onepass ? ln_fwd_wide_kernel<D, true> : ln_fwd_wide_kernel<D, false>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(ln_fwd_wide_kernel<D, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess ||
        cudaFuncSetAttribute(ln_fwd_wide_kernel<D, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
      return EPS_ECUDA;
    configured = true;
  }
  const int sms = sm_count() * ln_grid_mult(0, 3);
  const int64_t need = (rows + 7) / 8;
  const int grid = int(need < sms ? need : sms);
  count_launch();
  if (launch_k(kern, dim3(grid), dim3(L::THREADS), smem, st, 1,
               static_cast<const uint16_t*>(x), gamma, beta, static_cast<uint16_t*>(y), mean, rstd,
               rows, eps) != cudaSuccess)
    return EPS_ECUDA;
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

template <int D>
int ln_bwd_wide_launch(const void* dy, const void* x, const float* gamma, const float* mean,
                       const float* rstd, const void* dres, void* dx, float* dgamma, float* dbeta,
                       float* colsum, int64_t rows, cudaStream_t st) {
  using L = LnWide<D>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(ln_bwd_wide_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(L::SMEM)) != cudaSuccess)
      return EPS_ECUDA;
    configured = true;
  }
  const int sms = sm_count() * ln_grid_mult(1, 2);
  const int64_t need = (rows + 7) / 8;  // >= 8 rows per CTA
  const int grid = int(need < sms ? need : sms);
  count_launch();
  if (launch_k(ln_bwd_wide_kernel<D>, dim3(grid), dim3(L::THREADS), L::SMEM, st, 1,
               static_cast<const uint16_t*>(dy), static_cast<const uint16_t*>(x), gamma, mean, rstd,
               static_cast<const uint16_t*>(dres), static_cast<uint16_t*>(dx), dgamma, dbeta,
               colsum, rows) != cudaSuccess)
    return EPS_ECUDA;
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

int ln_grid_bwd(int64_t rows) {
  const int sms = sm_count();
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
    case 768: return ln_fwd_wide_launch<768>(x, gamma, beta, y, mean, rstd, rows, eps, st);
    case 1024: return ln_fwd_wide_launch<1024>(x, gamma, beta, y, mean, rstd, rows, eps, st);
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
      return ln_bwd_wide_launch<768>(dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta, colsum_dx,
                                     rows, st);
    case 1024:
      return ln_bwd_wide_launch<1024>(dy, x, gamma, mean, rstd, dres, dx, dgamma, dbeta,
                                      colsum_dx, rows, st);
    default:
      return EPS_EINVAL;
  }
}
