// Multi-head attention on the 5th-generation tensor cores (tcgen05 + TMEM +
// TMA) for head_dim 64 and sequence lengths up to 384 -- the ViT-B/16 (T=197),
// BERT-base-384 and BERT-large-128 shapes.  Every (batch, head) slice of keys
// fits on chip, so the softmax is exact in one pass (no online rescaling).
//
// Layout (same contract as attention.cu): qkv [B*T, 3*H*64] with Q | K | V
// column blocks, head h at h*64; out / dout [B*T, H*64]; lse [B, H, T].
// Operands are loaded by 3D TMA boxes of 64 rows x 64 columns with 128B
// swizzle; the [B][T][cols] view zero-fills rows >= T of each sample.
//
// Forward, one CTA per (128-query tile, b, h):
//   warp 0  TMA: Q tile, all K and V rows of the head (one mbarrier)
//   warp 1  TMEM alloc + MMA issue: S = Q K^T into TMEM (N <= 256 per MMA),
//           then O = P V with P read from TMEM (A operand, .kind::f16 TS form)
//   warps 2-5  one query row per thread: row max, exp2, row sum; P written
//           back as bf16 into the S columns in place (tcgen05.st); lse; final
//           O / rowsum -> bf16 -> global.
// Backward = dQ kernel (query tile per CTA, loops 64-key chunks; also emits
// D = rowsum(dO * O)) then dK/dV kernel (key tile per CTA, loops 64-query
// chunks).  P and dS live in TMEM as the A operands of the dQ / dK / dV
// MMAs; all accumulators are TMEM.  Column sums of dQ / dK / dV (= the QKV
// bias gradient) are accumulated in the epilogues.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cfloat>

#include "eps_capi.h"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace eps_k {
namespace attn_tc {

constexpr int kD = 64;
constexpr int kRowBytes = kD * 2;  // one 128B swizzle row
constexpr int kThreads = 192;
constexpr int kTile = 128;         // query rows (fwd, dQ) or key rows (dK/dV) per CTA
constexpr int kChunk = 64;         // TMA box rows; inner-loop chunk of keys / queries
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.69314718055994531f;

__host__ __device__ constexpr int pad64(int t) { return (t + 63) / 64 * 64; }
__host__ __device__ constexpr uint32_t tmem_cols_for(int n) {
  return n <= 32 ? 32u : n <= 64 ? 64u : n <= 128 ? 128u : n <= 256 ? 256u : 512u;
}

// K-major SW128 operand (rows of 64 bf16), 16-element K slice kk.
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int kk) {
  return umma_sdesc(base + uint32_t(kk) * 32u, 16, 1024);
}
// MN-major SW128 operand whose K rows start at `base` (N = 64 = one chunk).
__device__ __forceinline__ uint64_t mndesc(uint32_t base) { return umma_sdesc(base, 64 * 128, 1024); }

__device__ __forceinline__ void load_rows(uint8_t* dst, const CUtensorMap* map, uint64_t* bar,
                                          int col, int row0, int rows, int b) {
  for (int r = 0; r < rows; r += kChunk) tma_load_3d(dst + r * kRowBytes, map, bar, col, row0 + r, b);
}

__device__ __forceinline__ void store_row64(uint16_t* dst, const float (&v)[64]) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int i = 0; i < 8; ++i)
    d4[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                       pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
}

// Column sums over the 128 rows of a CTA tile: per warp a 32-lane transpose
// sum for each 32-column half, then one atomic per column per warp.
__device__ __forceinline__ void colsum64(float (&v)[64], float* dbias) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    float t[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) t[j] = v[half * 32 + j];
    const float s = warp_transpose_sum32(t);
    atomicAdd(dbias + half * 32 + lane, s);
  }
}

__device__ __forceinline__ void load_tmem_row64(uint32_t taddr, float (&v)[64]) {
  uint32_t a[32], c[32];
  tmem_ld_32x32(taddr, a);
  tmem_ld_32x32(taddr + 32, c);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    v[j] = __uint_as_float(a[j]);
    v[32 + j] = __uint_as_float(c[j]);
  }
}

struct Params {
  int T, H, Tp, n_split;
  float scale, scale_log2;
  const uint16_t* out;  // forward output (bwd: for D = rowsum(dO * O))
  uint16_t* out_w;      // forward: written
  float* lse;
  float* dsum;
  uint16_t* dqkv;
  float* dbias;
};

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 2)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap map_qkv, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int Tp = p.Tp;
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + kTile * kRowBytes;
  uint8_t* sV = sK + Tp * kRowBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + Tp * kRowBytes);  // load, s, p, o
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 4);
  const int bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int q0 = blockIdx.x * kTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ncols = tmem_cols_for(max(Tp, Tp / 2 + kD));

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 4);
    mbar_init(&bar[3], 1);
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tmem_o = tmem + uint32_t(Tp / 2);

  if (warp == 0) {
    if (lane == 0) {
      const int HD = p.H * kD;
      mbar_expect_tx(&bar[0], uint32_t(kTile + 2 * Tp) * kRowBytes);
      load_rows(sQ, &map_qkv, &bar[0], h * kD, q0, kTile, b);
      load_rows(sK, &map_qkv, &bar[0], HD + h * kD, 0, Tp, b);
      load_rows(sV, &map_qkv, &bar[0], 2 * HD + h * kD, 0, Tp, b);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(&bar[0], 0);
      tc_fence_after();
      const uint32_t q_s = smem_addr(sQ), k_s = smem_addr(sK), v_s = smem_addr(sV);
      const int nc = Tp / p.n_split;
      const uint32_t idesc_s = umma_idesc_bf16(128, nc, false, false);
      for (int c = 0; c < p.n_split; ++c)
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          tc_mma_bf16(tmem + uint32_t(c * nc), kdesc(q_s, kk),
                      kdesc(k_s + uint32_t(c * nc) * kRowBytes, kk), idesc_s, kk > 0 ? 1u : 0u);
      tc_commit(&bar[1]);
      mbar_wait(&bar[2], 0);
      tc_fence_after();
      const uint32_t idesc_o = umma_idesc_bf16(128, kD, false, true);
      for (int kk = 0; kk < Tp / 16; ++kk)
        tc_mma_bf16_ts(tmem_o, tmem + uint32_t(kk * 8), mndesc(v_s + uint32_t(kk * 16) * kRowBytes),
                       idesc_o, kk > 0 ? 1u : 0u);
      tc_commit(&bar[3]);
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int q = q0 + row;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    mbar_wait(&bar[1], 0);
    tc_fence_after();
    float m = -FLT_MAX;
    for (int c = 0; c < Tp / 32; ++c) {
      uint32_t r[32];
      tmem_ld_32x32(tmem + lane_off + uint32_t(c * 32), r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (c * 32 + j < p.T) m = fmaxf(m, __uint_as_float(r[j]));
    }
    const float ms = m * p.scale_log2;
    float sum = 0.f;
    for (int c = 0; c < Tp / 32; ++c) {
      uint32_t r[32];
      tmem_ld_32x32(tmem + lane_off + uint32_t(c * 32), r);
      tmem_ld_wait();
      uint32_t pk[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int k = c * 32 + 2 * j;
        const float e0 = k < p.T ? fast_exp2(fmaf(__uint_as_float(r[2 * j]), p.scale_log2, -ms)) : 0.f;
        const float e1 =
            k + 1 < p.T ? fast_exp2(fmaf(__uint_as_float(r[2 * j + 1]), p.scale_log2, -ms)) : 0.f;
        sum += e0 + e1;
        pk[j] = pack_bf16(e0, e1);
      }
      // P overwrites S columns [16c, 16c+16) -- already consumed (16c+16 <= 32c+32)
      tmem_st_32x32_x16(tmem + lane_off + uint32_t(c * 16), pk);
    }
    tmem_st_wait();
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bar[2]);
    if (q < p.T) p.lse[int64_t(bh) * p.T + q] = (ms + __log2f(sum)) * kLn2;
    mbar_wait(&bar[3], 0);
    tc_fence_after();
    float o[64];
    load_tmem_row64(tmem_o + lane_off, o);
    if (q < p.T) {
      const float inv = 1.f / sum;
#pragma unroll
      for (int j = 0; j < 64; ++j) o[j] *= inv;
      store_row64(p.out_w + (int64_t(b) * p.T + q) * (p.H * kD) + h * kD, o);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, ncols);
  }
}

// ---------------------------------------------------------------------------
// dQ (and D = rowsum(dO * O)): one CTA per (128-query tile, b, h).
__global__ void __launch_bounds__(kThreads, 2)
    attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap map_qkv,
                          const __grid_constant__ CUtensorMap map_do, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int Tp = p.Tp;
  uint8_t* sQ = smem;
  uint8_t* sO = sQ + kTile * kRowBytes;  // dO tile
  uint8_t* sK = sO + kTile * kRowBytes;
  uint8_t* sV = sK + Tp * kRowBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sV + Tp * kRowBytes);  // load, s, p, acc, done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 5);
  const int bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int q0 = blockIdx.x * kTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HD = p.H * kD;
  const int n_chunks = Tp / kChunk;

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    tma_prefetch(&map_do);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 4);
    mbar_init(&bar[3], 1);
    mbar_init(&bar[4], 1);
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tdP = tmem + 64, tdQ = tmem + 128;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(&bar[0], uint32_t(2 * kTile + 2 * Tp) * kRowBytes);
      load_rows(sQ, &map_qkv, &bar[0], h * kD, q0, kTile, b);
      load_rows(sO, &map_do, &bar[0], h * kD, q0, kTile, b);
      load_rows(sK, &map_qkv, &bar[0], HD + h * kD, 0, Tp, b);
      load_rows(sV, &map_qkv, &bar[0], 2 * HD + h * kD, 0, Tp, b);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(&bar[0], 0);
      tc_fence_after();
      const uint32_t q_s = smem_addr(sQ), o_s = smem_addr(sO), k_s = smem_addr(sK),
                     v_s = smem_addr(sV);
      const uint32_t idesc_kk = umma_idesc_bf16(128, kChunk, false, false);
      const uint32_t idesc_km = umma_idesc_bf16(128, kD, false, true);
      for (int c = 0; c < n_chunks; ++c) {
        if (c > 0) {
          mbar_wait(&bar[3], (c - 1) & 1);
          tc_fence_after();
        }
        const uint32_t kc = k_s + uint32_t(c * kChunk) * kRowBytes;
        const uint32_t vc = v_s + uint32_t(c * kChunk) * kRowBytes;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          tc_mma_bf16(tS, kdesc(q_s, kk), kdesc(kc, kk), idesc_kk, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          tc_mma_bf16(tdP, kdesc(o_s, kk), kdesc(vc, kk), idesc_kk, kk > 0 ? 1u : 0u);
        tc_commit(&bar[1]);
        mbar_wait(&bar[2], c & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kChunk / 16; ++kk)
          tc_mma_bf16_ts(tdQ, tdP + uint32_t(kk * 8), mndesc(kc + uint32_t(kk * 16) * kRowBytes),
                         idesc_km, (c > 0 || kk > 0) ? 1u : 0u);
        tc_commit(&bar[3]);
      }
      tc_commit(&bar[4]);
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int q = q0 + row;
    const bool valid_q = q < p.T;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    float Dq = 0.f, lse2 = 0.f;
    mbar_wait(&bar[0], 0);  // dO tile resident
    if (valid_q) {
      const uint4* o4 =
          reinterpret_cast<const uint4*>(p.out + (int64_t(b) * p.T + q) * HD + h * kD);
      const uint32_t o_s = smem_addr(sO);
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const uint4 a = __ldg(o4 + v);
        const uint4 d = ld_shared_v4(o_s + swz128(row, v));
        Dq += bf16_lo(a.x) * bf16_lo(d.x) + bf16_hi(a.x) * bf16_hi(d.x) +
              bf16_lo(a.y) * bf16_lo(d.y) + bf16_hi(a.y) * bf16_hi(d.y) +
              bf16_lo(a.z) * bf16_lo(d.z) + bf16_hi(a.z) * bf16_hi(d.z) +
              bf16_lo(a.w) * bf16_lo(d.w) + bf16_hi(a.w) * bf16_hi(d.w);
      }
      p.dsum[int64_t(bh) * p.T + q] = Dq;
      lse2 = p.lse[int64_t(bh) * p.T + q] * kLog2e;
    }
    for (int c = 0; c < n_chunks; ++c) {
      mbar_wait(&bar[1], c & 1);
      tc_fence_after();
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t s[32], dp[32];
        tmem_ld_32x32(tS + lane_off + uint32_t(half * 32), s);
        tmem_ld_32x32(tdP + lane_off + uint32_t(half * 32), dp);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int k = c * kChunk + half * 32 + 2 * j;
          const float p0 = (valid_q && k < p.T)
                               ? fast_exp2(fmaf(__uint_as_float(s[2 * j]), p.scale_log2, -lse2))
                               : 0.f;
          const float p1 =
              (valid_q && k + 1 < p.T)
                  ? fast_exp2(fmaf(__uint_as_float(s[2 * j + 1]), p.scale_log2, -lse2))
                  : 0.f;
          pk[j] = pack_bf16(p0 * (__uint_as_float(dp[2 * j]) - Dq),
                            p1 * (__uint_as_float(dp[2 * j + 1]) - Dq));
        }
        tmem_st_32x32_x16(tdP + lane_off + uint32_t(half * 16), pk);  // dS in place
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[2]);
    }
    mbar_wait(&bar[4], 0);
    tc_fence_after();
    float v[64];
    load_tmem_row64(tdQ + lane_off, v);
#pragma unroll
    for (int j = 0; j < 64; ++j)
      v[j] = valid_q ? __bfloat162float(__float2bfloat16_rn(v[j] * p.scale)) : 0.f;
    if (valid_q) store_row64(p.dqkv + (int64_t(b) * p.T + q) * (3 * HD) + h * kD, v);
    if (p.dbias != nullptr) colsum64(v, p.dbias + h * kD);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

// ---------------------------------------------------------------------------
// dK / dV: one CTA per (128-key tile, b, h); loops over 64-query chunks.
//   S^T = K Q^T, P^T = exp(S^T*scale - lse[q]), dP^T = V dO^T,
//   dS^T = P^T (dP^T - D[q]), dV += P^T dO, dK += dS^T Q (* scale at the end).
__global__ void __launch_bounds__(kThreads, 2)
    attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap map_qkv,
                            const __grid_constant__ CUtensorMap map_do, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int Tp = p.Tp;
  uint8_t* sK = smem;
  uint8_t* sV = sK + kTile * kRowBytes;
  uint8_t* sQ = sV + kTile * kRowBytes;
  uint8_t* sO = sQ + Tp * kRowBytes;  // dO, all queries
  float* sL = reinterpret_cast<float*>(sO + Tp * kRowBytes);
  float* sD = sL + Tp;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sD + Tp);  // load, s, p, acc, done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 5);
  const int bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int k0 = blockIdx.x * kTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HD = p.H * kD;
  const int n_chunks = Tp / kChunk;

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    tma_prefetch(&map_do);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 4);
    mbar_init(&bar[3], 1);
    mbar_init(&bar[4], 1);
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tdP = tmem + 64, tdV = tmem + 128, tdK = tmem + 192;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(&bar[0], uint32_t(2 * kTile + 2 * Tp) * kRowBytes);
      load_rows(sK, &map_qkv, &bar[0], HD + h * kD, k0, kTile, b);
      load_rows(sV, &map_qkv, &bar[0], 2 * HD + h * kD, k0, kTile, b);
      load_rows(sQ, &map_qkv, &bar[0], h * kD, 0, Tp, b);
      load_rows(sO, &map_do, &bar[0], h * kD, 0, Tp, b);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(&bar[0], 0);
      tc_fence_after();
      const uint32_t k_s = smem_addr(sK), v_s = smem_addr(sV), q_s = smem_addr(sQ),
                     o_s = smem_addr(sO);
      const uint32_t idesc_kk = umma_idesc_bf16(128, kChunk, false, false);
      const uint32_t idesc_km = umma_idesc_bf16(128, kD, false, true);
      for (int c = 0; c < n_chunks; ++c) {
        if (c > 0) {
          mbar_wait(&bar[3], (c - 1) & 1);
          tc_fence_after();
        }
        const uint32_t qc = q_s + uint32_t(c * kChunk) * kRowBytes;
        const uint32_t oc = o_s + uint32_t(c * kChunk) * kRowBytes;
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          tc_mma_bf16(tS, kdesc(k_s, kk), kdesc(qc, kk), idesc_kk, kk > 0 ? 1u : 0u);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          tc_mma_bf16(tdP, kdesc(v_s, kk), kdesc(oc, kk), idesc_kk, kk > 0 ? 1u : 0u);
        tc_commit(&bar[1]);
        mbar_wait(&bar[2], c & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kChunk / 16; ++kk) {
          const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
          tc_mma_bf16_ts(tdV, tS + uint32_t(kk * 8), mndesc(oc + uint32_t(kk * 16) * kRowBytes),
                         idesc_km, acc);
          tc_mma_bf16_ts(tdK, tdP + uint32_t(kk * 8), mndesc(qc + uint32_t(kk * 16) * kRowBytes),
                         idesc_km, acc);
        }
        tc_commit(&bar[3]);
      }
      tc_commit(&bar[4]);
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int key = k0 + row;
    const bool valid_k = key < p.T;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    // per-query log2-domain lse and D into smem (the 128 softmax threads)
    for (int i = threadIdx.x - 64; i < Tp; i += 128) {
      const bool ok = i < p.T;
      sL[i] = ok ? p.lse[int64_t(bh) * p.T + i] * kLog2e : 0.f;
      sD[i] = ok ? p.dsum[int64_t(bh) * p.T + i] : 0.f;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    for (int c = 0; c < n_chunks; ++c) {
      mbar_wait(&bar[1], c & 1);
      tc_fence_after();
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t s[32], dp[32];
        tmem_ld_32x32(tS + lane_off + uint32_t(half * 32), s);
        tmem_ld_32x32(tdP + lane_off + uint32_t(half * 32), dp);
        tmem_ld_wait();
        uint32_t pp[16], pd[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int qa = c * kChunk + half * 32 + 2 * j;
          const bool ok0 = valid_k && qa < p.T, ok1 = valid_k && qa + 1 < p.T;
          const float p0 = ok0 ? fast_exp2(fmaf(__uint_as_float(s[2 * j]), p.scale_log2, -sL[qa])) : 0.f;
          const float p1 =
              ok1 ? fast_exp2(fmaf(__uint_as_float(s[2 * j + 1]), p.scale_log2, -sL[qa + 1])) : 0.f;
          pp[j] = pack_bf16(p0, p1);
          pd[j] = pack_bf16(p0 * (__uint_as_float(dp[2 * j]) - sD[qa]),
                            p1 * (__uint_as_float(dp[2 * j + 1]) - sD[qa + 1]));
        }
        tmem_st_32x32_x16(tS + lane_off + uint32_t(half * 16), pp);
        tmem_st_32x32_x16(tdP + lane_off + uint32_t(half * 16), pd);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[2]);
    }
    mbar_wait(&bar[4], 0);
    tc_fence_after();
    float v[64];
    load_tmem_row64(tdV + lane_off, v);
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = valid_k ? __bfloat162float(__float2bfloat16_rn(v[j])) : 0.f;
    if (valid_k) store_row64(p.dqkv + (int64_t(b) * p.T + key) * (3 * HD) + 2 * HD + h * kD, v);
    if (p.dbias != nullptr) colsum64(v, p.dbias + 2 * HD + h * kD);
    load_tmem_row64(tdK + lane_off, v);
#pragma unroll
    for (int j = 0; j < 64; ++j)
      v[j] = valid_k ? __bfloat162float(__float2bfloat16_rn(v[j] * p.scale)) : 0.f;
    if (valid_k) store_row64(p.dqkv + (int64_t(b) * p.T + key) * (3 * HD) + HD + h * kD, v);
    if (p.dbias != nullptr) colsum64(v, p.dbias + HD + h * kD);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

size_t fwd_smem(int Tp) { return size_t(kTile + 2 * Tp) * kRowBytes + 1024 + 64; }
size_t bwd_dq_smem(int Tp) { return size_t(2 * kTile + 2 * Tp) * kRowBytes + 1024 + 64; }
size_t bwd_dkdv_smem(int Tp) {
  return size_t(2 * kTile + 2 * Tp) * kRowBytes + size_t(2 * Tp) * 4 + 1024 + 64;
}

template <typename K>
bool ensure_smem(K kern, size_t bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) ==
         cudaSuccess;
}

}  // namespace attn_tc

// Entry points used by attention.cu's C ABI for head_dim 64, T <= 384.
bool attn_tc_supported(int T, int head_dim) { return head_dim == 64 && T >= 1 && T <= 384; }

int attn_fwd_tc(const void* qkv, void* out, float* lse, int B, int T, int H, float scale,
                cudaStream_t st) {
  using namespace attn_tc;
  const int Tp = pad64(T);
  const int64_t W = int64_t(3) * H * kD;
  CUtensorMap m;
  if (!make_map_3d(&m, qkv, W, T, B, W, int64_t(T) * W, kD, kChunk, CU_TENSOR_MAP_SWIZZLE_128B))
    return EPS_ECUDA;
  Params p{};
  p.T = T;
  p.H = H;
  p.Tp = Tp;
  p.n_split = Tp > 256 ? 2 : 1;
  p.scale = scale;
  p.scale_log2 = scale * kLog2e;
  p.out_w = static_cast<uint16_t*>(out);
  p.lse = lse;
  const size_t smem = fwd_smem(Tp);
  if (!ensure_smem(attn_fwd_tc_kernel, smem)) return EPS_ECUDA;
  dim3 grid((T + kTile - 1) / kTile, B * H);
  count_launch();
  attn_fwd_tc_kernel<<<grid, kThreads, smem, st>>>(m, p);
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

int attn_bwd_tc(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv,
                float* dbias, float* dsum, int B, int T, int H, float scale, cudaStream_t st) {
  using namespace attn_tc;
  const int Tp = pad64(T);
  const int64_t W = int64_t(3) * H * kD, WO = int64_t(H) * kD;
  CUtensorMap mq, mo;
  if (!make_map_3d(&mq, qkv, W, T, B, W, int64_t(T) * W, kD, kChunk, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_map_3d(&mo, dout, WO, T, B, WO, int64_t(T) * WO, kD, kChunk,
                   CU_TENSOR_MAP_SWIZZLE_128B))
    return EPS_ECUDA;
  Params p{};
  p.T = T;
  p.H = H;
  p.Tp = Tp;
  p.scale = scale;
  p.scale_log2 = scale * kLog2e;
  p.out = static_cast<const uint16_t*>(out);
  p.lse = const_cast<float*>(lse);
  p.dsum = dsum;
  p.dqkv = static_cast<uint16_t*>(dqkv);
  p.dbias = dbias;
  const size_t s1 = bwd_dq_smem(Tp), s2 = bwd_dkdv_smem(Tp);
  if (!ensure_smem(attn_bwd_dq_tc_kernel, s1) || !ensure_smem(attn_bwd_dkdv_tc_kernel, s2))
    return EPS_ECUDA;
  dim3 grid((T + kTile - 1) / kTile, B * H);
  count_launch();
  attn_bwd_dq_tc_kernel<<<grid, kThreads, s1, st>>>(mq, mo, p);
  count_launch();
  attn_bwd_dkdv_tc_kernel<<<grid, kThreads, s2, st>>>(mq, mo, p);
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

}  // namespace eps_k
