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
#include <cstdlib>
#include <string>
#include <unordered_map>

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
  int trace;  // record phase stamps of CTA 0 (eps_attn_trace_*)
  int dbg;    // EPS_ATTN_DBG bit 0: every head loads head (0, 0) (L2-resident; experiments)
  int T, H, Tp, n_split;
  float scale, scale_log2;
  const uint16_t* out;  // forward output (bwd: for D = rowsum(dO * O))
  const float* drow;  // bwd (fused): D = rowsum(dO * O), fp32 [B*T, H]
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
// Forward for 256 < T <= 384 (BERT-base-384): one CTA per (128-query tile,
// b, h), keys in blocks of 192 (three 64-key chunks) so a CTA needs only 256
// TMEM columns (S block [0, 192), O [192, 256)) and K / V stream through a
// kFwdRing-deep ring of 64-key chunks (80 KB of smem): two CTAs share an SM
// and overlap each other's loads, exps and MMAs.
//   MMA warp: per block, S = Q K_c^T for its chunks (N = 64 each) -> SF;
//             after the softmax, O += P V_c (TS form, P packed in TMEM) -> OB,
//             and the block's ring slots are released; the next block's S
//             waits for OB (it overwrites the P columns).
//   softmax warps: one row per thread, one pass per 32 keys; exponent
//             reference = max of the first 32 keys; a later 32-key group that
//             leads it by > 2^32 rescales this block's P chunks, the row sum,
//             and (from the second block on) O -- complete, since the block's
//             S was issued after the previous PV finished (rare path).
constexpr int kFwdRing = 4;
constexpr int kFwdBlock = 3;  // 64-key chunks per key block
__global__ void __launch_bounds__(kThreads, 2)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap map_qkv, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int Tp = p.Tp;
  const int n_chunks = Tp / kChunk;
  const int n_blocks = (n_chunks + kFwdBlock - 1) / kFwdBlock;
  constexpr int kStage = 2 * kChunk * kRowBytes;  // K chunk | V chunk
  uint8_t* sQ = smem;
  uint8_t* sR = sQ + kTile * kRowBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sR + kFwdRing * kStage);
  enum { BQ = 0, SF, PF, OB, DONE, FULL0 };
  uint64_t* full = bar + FULL0;
  uint64_t* empty = full + kFwdRing;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty + kFwdRing);
  const int bh = blockIdx.y, b = bh / p.H, h = bh % p.H;
  const int q0 = blockIdx.x * kTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr uint32_t kO = uint32_t(kFwdBlock * kChunk);  // 192

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    for (int i = 0; i < FULL0; ++i) mbar_init(&bar[i], i == PF ? 4 : 1);
    for (int i = 0; i < kFwdRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const int HD = p.H * kD;
      mbar_expect_tx(&bar[BQ], uint32_t(kTile * kRowBytes));
      load_rows(sQ, &map_qkv, &bar[BQ], h * kD, q0, kTile, b);
      for (int c = 0; c < n_chunks; ++c) {
        const int st = c % kFwdRing;
        mbar_wait(&empty[st], ((c / kFwdRing) & 1) ^ 1);
        uint8_t* slot = sR + st * kStage;
        mbar_expect_tx(&full[st], uint32_t(kStage));
        tma_load_3d(slot, &map_qkv, &full[st], HD + h * kD, c * kChunk, b);
        tma_load_3d(slot + kChunk * kRowBytes, &map_qkv, &full[st], 2 * HD + h * kD, c * kChunk, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(&bar[BQ], 0);
      tc_fence_after();
      const uint32_t q_s = smem_addr(sQ);
      const uint32_t idesc_s = umma_idesc_bf16(128, kChunk, false, false);
      const uint32_t idesc_o = umma_idesc_bf16(128, kD, false, true);
      for (int kb = 0; kb < n_blocks; ++kb) {
        const int c0 = kb * kFwdBlock, c1 = min(c0 + kFwdBlock, n_chunks);
        if (kb > 0) {  // the previous PV has read the P columns S overwrites
          mbar_wait(&bar[OB], (kb - 1) & 1);
          tc_fence_after();
        }
        for (int c = c0; c < c1; ++c) {
          const int st = c % kFwdRing;
          mbar_wait(&full[st], (c / kFwdRing) & 1);
          tc_fence_after();
          const uint32_t kc = smem_addr(sR + st * kStage);
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk)
            tc_mma_bf16(tmem + uint32_t((c - c0) * kChunk), kdesc(q_s, kk), kdesc(kc, kk), idesc_s,
                        kk > 0 ? 1u : 0u);
        }
        tc_commit(&bar[SF]);
        mbar_wait(&bar[PF], kb & 1);
        tc_fence_after();
        for (int c = c0; c < c1; ++c) {
          const uint32_t vc = smem_addr(sR + (c % kFwdRing) * kStage) + uint32_t(kChunk * kRowBytes);
#pragma unroll
          for (int kk = 0; kk < kChunk / 16; ++kk)
            tc_mma_bf16_ts(tmem + kO, tmem + uint32_t((c - c0) * 32 + kk * 8),
                           mndesc(vc + uint32_t(kk * 16) * kRowBytes), idesc_o,
                           (kb > 0 || c > c0 || kk > 0) ? 1u : 0u);
          tc_commit(&empty[c % kFwdRing]);
        }
        tc_commit(&bar[OB]);
      }
      tc_commit(&bar[DONE]);
    }
  } else {
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const int q = q0 + row;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const uint32_t tS = tmem + lane_off;
    const float sl2 = p.scale_log2;
    float ms = 0.f, sum = 0.f;
    for (int kb = 0; kb < n_blocks; ++kb) {
      const int k0 = kb * kFwdBlock * kChunk;
      const int ncol = min(kFwdBlock, n_chunks - kb * kFwdBlock) * kChunk;
      mbar_wait(&bar[SF], kb & 1);
      tc_fence_after();
      for (int g = 0; g < ncol / 32; ++g) {
        uint32_t r[32];
        tmem_ld_32x32(tS + uint32_t(g * 32), r);
        tmem_ld_wait();
        const int kbase = k0 + g * 32;  // keys >= T are masked (zero-filled K rows)
        float cm = -FLT_MAX;
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (kbase + j < p.T) cm = fmaxf(cm, __uint_as_float(r[j]));
        cm *= sl2;
        if (kb == 0 && g == 0) {
          ms = cm;
        } else if (__any_sync(0xffffffffu, cm > ms + 32.f)) {
          const float ms_new = cm > ms + 32.f ? cm : ms;
          const float f = fast_exp2(ms - ms_new);  // 1 on lanes without overflow
          sum *= f;
          tmem_st_wait();
          for (int pc = 0; pc < g; ++pc) {  // this block's P
            uint32_t q16[16];
            tmem_ld_32x32_x16(tS + uint32_t(pc * 16), q16);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) q16[j] = pack_bf16(bf16_lo(q16[j]) * f, bf16_hi(q16[j]) * f);
            tmem_st_32x32_x16(tS + uint32_t(pc * 16), q16);
          }
          if (kb > 0) {  // O of the earlier blocks (their PV finished before this S)
            uint32_t o32[32];
#pragma unroll
            for (int hlf = 0; hlf < 2; ++hlf) {
              tmem_ld_32x32(tS + kO + uint32_t(hlf * 32), o32);
              tmem_ld_wait();
#pragma unroll
              for (int j = 0; j < 32; ++j) o32[j] = __float_as_uint(__uint_as_float(o32[j]) * f);
              tmem_st_32x32_x32(tS + kO + uint32_t(hlf * 32), o32);
            }
          }
          ms = ms_new;
        }
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int k = kbase + 2 * j;
          const float e0 = k < p.T ? fast_exp2(fmaf(__uint_as_float(r[2 * j]), sl2, -ms)) : 0.f;
          const float e1 = k + 1 < p.T ? fast_exp2(fmaf(__uint_as_float(r[2 * j + 1]), sl2, -ms)) : 0.f;
          sum += e0 + e1;
          pk[j] = pack_bf16(e0, e1);
        }
        // P overwrites S columns [16g, 16g+16) -- already consumed (16g+16 <= 32g+32)
        tmem_st_32x32_x16(tS + uint32_t(g * 16), pk);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[PF]);
    }
    if (q < p.T) p.lse[int64_t(bh) * p.T + q] = (ms + __log2f(sum)) * kLn2;
    mbar_wait(&bar[DONE], 0);
    tc_fence_after();
    float o[64];
    load_tmem_row64(tS + kO, o);
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
    tmem_dealloc(tmem, 256);
  }
}

// ---------------------------------------------------------------------------
// dQ (and D = rowsum(dO * O)): one CTA per (128-query tile, b, h).  K and V
// stream through a kBwdRing-deep ring of 64-key chunks (a slot is refilled
// once the dQ MMA that last reads its K chunk completes), so a CTA holds
// 32 KB + kBwdRing x 16 KB of smem and two CTAs share an SM: one's loads and
// exp work overlap the other's MMAs (T = 384, BERT-base).
constexpr int kBwdRing = 3;
__global__ void __launch_bounds__(kThreads, 2)
    attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap map_qkv,
                          const __grid_constant__ CUtensorMap map_do, const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int Tp = p.Tp;
  uint8_t* sQ = smem;
  uint8_t* sO = sQ + kTile * kRowBytes;      // dO tile
  uint8_t* sR = sO + kTile * kRowBytes;      // ring: stage s = K chunk | V chunk
  constexpr int kStage = 2 * kChunk * kRowBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sR + kBwdRing * kStage);
  // 0 tile loaded, 1 S/dP ready, 2 dS written, 3 dQ MMA done, 4 all done,
  // 5.. full[kBwdRing], empty[kBwdRing]
  uint64_t* full = bar + 5;
  uint64_t* empty = full + kBwdRing;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty + kBwdRing);
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
    for (int i = 0; i < kBwdRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
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
      mbar_expect_tx(&bar[0], uint32_t(2 * kTile) * kRowBytes);
      load_rows(sQ, &map_qkv, &bar[0], h * kD, q0, kTile, b);
      load_rows(sO, &map_do, &bar[0], h * kD, q0, kTile, b);
      for (int c = 0; c < n_chunks; ++c) {
        const int st = c % kBwdRing;
        mbar_wait(&empty[st], ((c / kBwdRing) & 1) ^ 1);
        uint8_t* slot = sR + st * kStage;
        mbar_expect_tx(&full[st], uint32_t(kStage));
        tma_load_3d(slot, &map_qkv, &full[st], HD + h * kD, c * kChunk, b);
        tma_load_3d(slot + kChunk * kRowBytes, &map_qkv, &full[st], 2 * HD + h * kD, c * kChunk, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(&bar[0], 0);
      tc_fence_after();
      const uint32_t q_s = smem_addr(sQ), o_s = smem_addr(sO);
      const uint32_t idesc_kk = umma_idesc_bf16(128, kChunk, false, false);
      const uint32_t idesc_km = umma_idesc_bf16(128, kD, false, true);
      for (int c = 0; c < n_chunks; ++c) {
        const int st = c % kBwdRing;
        if (c > 0) {
          mbar_wait(&bar[3], (c - 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&full[st], (c / kBwdRing) & 1);
        tc_fence_after();
        const uint32_t kc = smem_addr(sR + st * kStage);
        const uint32_t vc = kc + uint32_t(kChunk * kRowBytes);
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
        tc_commit(&empty[st]);  // K_c / V_c read by every MMA of this chunk
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
  uint8_t* sR = sV + kTile * kRowBytes;  // ring: stage s = Q chunk | dO chunk
  constexpr int kStage = 2 * kChunk * kRowBytes;
  float* sL = reinterpret_cast<float*>(sR + kBwdRing * kStage);
  float* sD = sL + Tp;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sD + Tp);  // load, s, p, acc, done
  uint64_t* full = bar + 5;
  uint64_t* empty = full + kBwdRing;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(empty + kBwdRing);
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
    for (int i = 0; i < kBwdRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
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
      mbar_expect_tx(&bar[0], uint32_t(2 * kTile) * kRowBytes);
      load_rows(sK, &map_qkv, &bar[0], HD + h * kD, k0, kTile, b);
      load_rows(sV, &map_qkv, &bar[0], 2 * HD + h * kD, k0, kTile, b);
      for (int c = 0; c < n_chunks; ++c) {
        const int st = c % kBwdRing;
        mbar_wait(&empty[st], ((c / kBwdRing) & 1) ^ 1);
        uint8_t* slot = sR + st * kStage;
        mbar_expect_tx(&full[st], uint32_t(kStage));
        tma_load_3d(slot, &map_qkv, &full[st], h * kD, c * kChunk, b);
        tma_load_3d(slot + kChunk * kRowBytes, &map_do, &full[st], h * kD, c * kChunk, b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      mbar_wait(&bar[0], 0);
      tc_fence_after();
      const uint32_t k_s = smem_addr(sK), v_s = smem_addr(sV);
      const uint32_t idesc_kk = umma_idesc_bf16(128, kChunk, false, false);
      const uint32_t idesc_km = umma_idesc_bf16(128, kD, false, true);
      for (int c = 0; c < n_chunks; ++c) {
        const int st = c % kBwdRing;
        if (c > 0) {
          mbar_wait(&bar[3], (c - 1) & 1);
          tc_fence_after();
        }
        mbar_wait(&full[st], (c / kBwdRing) & 1);
        tc_fence_after();
        const uint32_t qc = smem_addr(sR + st * kStage);
        const uint32_t oc = qc + uint32_t(kChunk * kRowBytes);
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
        tc_commit(&empty[st]);  // Q_c / dO_c read by every MMA of this chunk
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

// ---------------------------------------------------------------------------
// Profiling aid: clock64 phase stamps of CTA 0 of the fused backward (off
// unless eps_attn_trace_enable(1)).  Layout: [it*8 + e] for the first 64
// iterations (e: 0 S issued, 1 PF seen by MMA, 2 post issued, 3 SF seen by
// exp warp 2, 4 PF arrive by exp warp 2), [512 + kt*2 + e] per key tile
// (KVF seen, KVE arrive), [640 + hi*4 + e] per head (DQF seen, DQE arrive,
// FULL seen by MMA, table ready seen by exp).
__device__ long long g_attn_trace[1024];
#define EPS_TRACE(cond, idx) \
  do {                        \
    if (p.trace && blockIdx.x == 0 && (cond)) g_attn_trace[(idx)] = clock64(); \
  } while (0)

// Fused, persistent backward for T <= 256.  One CTA per SM walks the (b, h)
// heads; per head Q, dO, K, V (<= 256 rows each) sit in smem and the
// (128-key tile j, 64-query chunk c) pairs are visited once, so every exp is
// evaluated once:
//   S^T = K_j Q_c^T, dP^T = V_j dO_c^T                 (SS MMAs -> TMEM)
//   P^T = exp2(S^T*scale*log2e - lse2[q]), dS^T = P^T (dP^T - D[q])
//        (8 exp warps: key row per lane, 32 queries per warp; P^T / dS^T
//         back into TMEM as bf16, dS^T also into a smem staging tile)
//   dV_j += P^T dO_c, dK_j += dS^T Q_c                 (TS MMAs, A in TMEM)
//   dQ_t += dS_t K_j once both 64-query halves of 128-query tile t are staged
//                                                     (SS MMA, A MN-major)
// Roles (448 threads):
//   warp 0       TMA: the head's Q, dO, K, V; L2 prefetch two heads ahead
//   warp 1       TMEM alloc + single-thread MMA issue, one chunk ahead of exp
//   warps 2-9    exp / dS only: they never wait on an epilogue
//   warps 10-13  epilogue: the NEXT head's per-query (-lse*log2e, D) into a
//                double-buffered smem table (D = rowsum(dO * O) arrives
//                precomputed, fused into the GEMM that produced dO); dV / dK
//                per key tile and dQ per head: TMEM -> bf16 -> global, plus
//                the QKV bias column sums
// S^T / dP^T are double-buffered in TMEM, dS staging is double-buffered in
// smem.  TMEM (512 cols): [S^T 64 | dP^T 64] x 2 | dV 64 | dK 64 | dQ_t 64 x NT.
// NT (= ceil(T / 128)) is a template parameter so the iteration bookkeeping
// is shifts and masks.
constexpr int kDsChunk = kTile * kRowBytes;  // [128 keys][64 queries] bf16 = 16 KB
constexpr int kBwdExpWarps = 8, kBwdEpiWarps = 4;
// dK MMAs read dS^T from the smem staging tile (SS) instead of TMEM (TS)
constexpr bool kBwdDkSS = false;
// T <= 128: operand regions double-buffered across heads (attn_bwd_fused_tc_kernel DB;
// measured neutral at BERT-large-128, 0.0444 -> 0.0448 ms, off)
#ifndef EPS_BWD_DB
#define EPS_BWD_DB 0
#endif
constexpr bool kBwdDoubleBuffer = EPS_BWD_DB != 0;
// 256 < T <= 384 (UNIT): L2 prefetch of the next unit's operands
#ifndef EPS_BWD_UNIT_PF
#define EPS_BWD_UNIT_PF 1
#endif
constexpr bool kBwdUnitPrefetch = EPS_BWD_UNIT_PF != 0;
// epilogue staging tiles (16 KB each) by key-tile count: T <= 128 has room for
// three (dV / dK / dQ of a head leave without waiting on each other: BERT-large-128
// 0.0446 -> 0.0423 ms), unless its operands are double-buffered
__host__ __device__ constexpr int bwd_stage_tiles(int nt) {
  return nt == 1 && !kBwdDoubleBuffer ? 3 : 1;
}
// T <= 128: the epilogue fills the next head's (-lse2, D) table before it
// waits for this head's dV / dK
#ifndef EPS_BWD_EARLY_TABLE
#define EPS_BWD_EARLY_TABLE 1
#endif
constexpr bool kBwdEarlyTable = EPS_BWD_EARLY_TABLE != 0;
// Issue the S^T / dP^T MMAs of iteration it + 2 ahead of dQ(it) (see the post issuer)
constexpr bool kBwdSFirst = false;  // measured 0.2937 -> 0.297 ms (ViT-B), off  // measured neutral-to-slower (0.295 -> 0.297 ms, ViT-B)
// queries of a 64-query chunk per exp warp (4 warps per TMEM lane quarter)
constexpr int kBwdQPW = kChunk / (kBwdExpWarps / 4);
constexpr int kBwdPasses = kBwdQPW / 16;  // 16-query passes per warp
// TMEM column (within an S^T / dP^T buffer) of the packed bf16 P^T / dS^T of
// 16-query slice g: inside the columns of the warp that owns the slice
__host__ __device__ constexpr int pk_col(int g) {
  return (g / kBwdPasses) * kBwdQPW + (g % kBwdPasses) * 8;
}
constexpr int kBwdPostWarp = 2 + kBwdExpWarps + kBwdEpiWarps;  // second MMA issuer
constexpr int kBwdThreads = 32 * (kBwdPostWarp + 1);

__device__ __forceinline__ void tma_prefetch_3d(const void* tmap, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// One row of 64 fp32 TMEM columns -> scaled, bf16-rounded pairs (the stored
// values; bias column sums are taken from the same rounded values).
__device__ __forceinline__ void load_tmem_packed64(uint32_t taddr, float sc, uint32_t (&pk)[32]) {
  uint32_t a[32];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    tmem_ld_32x32(taddr + uint32_t(h * 32), a);
    tmem_ld_wait();
#pragma unroll
    for (int d = 0; d < 16; ++d)
      pk[h * 16 + d] = pack_bf16(__uint_as_float(a[2 * d]) * sc, __uint_as_float(a[2 * d + 1]) * sc);
  }
}

__device__ __forceinline__ void zero32(uint32_t (&pk)[32]) {
#pragma unroll
  for (int d = 0; d < 32; ++d) pk[d] = 0u;
}


// UNIT (256 < T <= 384, NT = 3): a work unit is one (head, key tile): the
// unit's K / V tile plus the head's whole Q / dO sit in smem (a head's four
// 384-row operands do not fit), dV / dK of the tile accumulate as above, and
// each 128-query tile's dQ partial (dS_t K_j over this key tile) is read out
// as soon as its two chunks are done -- two TMEM dQ buffers in turn -- and
// stored in bf16 into slice j of a partial buffer (map_dqp, [NT*B][T][HD]);
// attn_dq_reduce_kernel sums the slices into dQ and its bias column sums.
// PH (T <= 128, NT = 2): a work unit is a PAIR of heads laid out as one
// 256-row problem: key tile j and query tile t are heads 2u + j / 2u + t, and
// only the diagonal (j = t) iterations run -- four per unit instead of two per
// head, so the per-unit fill / drain is paid half as often.
template <int NT, bool UNIT = false, bool PH = false>
__global__ void __launch_bounds__(kBwdThreads, 1)
    attn_bwd_fused_tc_kernel(const __grid_constant__ CUtensorMap map_qkv,
                             const __grid_constant__ CUtensorMap map_do,
                             const __grid_constant__ CUtensorMap map_dq,
                             const __grid_constant__ CUtensorMap map_dqp, const Params p,
                             int n_heads) {
  constexpr int Tr = NT * kTile;   // Q / dO rows loaded (zero-filled past T)
  constexpr int NK = UNIT ? 1 : NT;  // key tiles per work unit
  constexpr int KR = NK * kTile;   // K / V rows loaded
  constexpr int NC = Tr / kChunk;  // 64-query chunks per key tile (2, 4 or 6)
  constexpr int NIT = PH ? NC : NK * NC;  // iterations per unit (2, 8, 6; PH: 4)
  constexpr int NU = UNIT ? NT : 1;  // units per head
  constexpr int NR = NK + NT;      // operand regions
  static_assert(NR <= 4 && NIT % 2 == 0, "regions / iterations");
  const int n_units = PH ? n_heads / 2 : n_heads * NU;
  static_assert(!PH || (NT == 2 && !UNIT), "paired heads: NT = 2 layout");
  // DB (T <= 128): the operand regions are double-buffered across heads --
  // head hi uses slot hi & 1 (KV region slot, QO region 2 + slot, the smem
  // rows of tile `slot` of an NT = 2 layout), so the next head's Q / dO / K /
  // V load while this head computes.
  constexpr bool DB = NT == 1 && !UNIT && !PH && kBwdDoubleBuffer;
  constexpr int TrA = DB ? 2 * kTile : Tr, KRA = DB ? 2 * kTile : KR;  // rows allocated
  auto slot_of = [](int hi) { return DB ? (hi & 1) : 0; };
  auto par_of = [](int hi) { return uint32_t(DB ? (hi >> 1) & 1 : hi & 1); };
  // iteration k of a unit -> (key tile j, query chunk c); PH: diagonal only
  auto jc = [](int k, int& j, int& c) {
    if (PH) {
      j = k >> 1;
      c = 2 * j + (k & 1);
    } else {
      j = k / NC;
      c = k % NC;
    }
  };
  // PH: global (b, h) of tile x of unit u (head 2u + x); else of the unit's head
  auto head_of = [&](int u, int x) { return PH ? 2 * u + x : u / NU; };
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sO = sQ + TrA * kRowBytes;  // dO
  uint8_t* sK = sO + TrA * kRowBytes;
  uint8_t* sV = sK + KRA * kRowBytes;
  uint8_t* sS = sV + KRA * kRowBytes;  // dS staging: 2 buffers x 2 chunks x 16 KB
  // epilogue: NSTG 128x64 bf16 output tiles in turn (T <= 128: three, so a
  // head's dV / dK / dQ stores never wait for each other; the larger layouts
  // have room for one)
  constexpr int NSTG = bwd_stage_tiles(NT);
  uint8_t* sStage = sS + 4 * kDsChunk;
  float2* sLD = reinterpret_cast<float2*>(sStage + NSTG * kDsChunk);  // [2][Tr] (-lse2, D)
  float* sRed = reinterpret_cast<float*>(sLD + 2 * Tr);  // [4][64] per-warp bias column sums
  uint64_t* bar = reinterpret_cast<uint64_t*>(sRed + 4 * 64);
  // Operand regions, each with its own full / empty barrier pair so a unit's
  // tiles are reloaded as soon as their last reader is done: KV_j = rows of
  // key tile j of K and V; QO_t = rows of query tile t of Q and dO.
  //   whole head: 0 = KV0, 1 = KV1, 2 = QO0, 3 = QO1;  UNIT: 0 = KV, 1 + t = QO_t
  // SI0 / SI1: S^T / dP^T of an iteration issued (plain arrive by the S issuer);
  // UNIT: DQF / DQE (buffer 0) and DQF1 / DQE1 (buffer 1) per dQ tile
  enum { FR = 0, ER = 4, SF0 = 8, SF1, PF0, PF1, AC0, AC1, KVF, KVE, DQF, DQE, LF0, LF1, LE0, LE1,
         SI0, SI1, DQF1, DQE1,
         NBAR };
  // (DB: key tile j / query tile t are 0; `sl` is the head's slot)
  auto kv_region = [](int j, int sl = 0) { return j + sl; };
  auto qo_region = [](int t, int sl = 0) { return UNIT ? 1 + t : 2 + t + sl; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + NBAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HD = p.H * kD;
  // last iteration of a unit that reads region r: KV_j is read by S (key
  // tile j) and by the dQ MMAs of its odd chunks; QO_t by the S and post MMAs
  // of chunks 2t, 2t+1 of the last key tile; -1: region unused
  auto last_use = [](int r) {
    if (DB) return NC - 1;  // both slots' KV and QO: the head's last iteration
    if (PH) return r < 2 ? 2 * r + 1 : 2 * (r - 2) + 1;
    if (UNIT) return r == 0 ? NC - 1 : r <= NT ? 2 * (r - 1) + 1 : -1;
    if (r < 2) return r < NT ? r * NC + NC - 1 : -1;
    return r - 2 < NT ? (NT - 1) * NC + 2 * (r - 2) + 1 : -1;
  };

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    tma_prefetch(&map_do);
    tma_prefetch(&map_dq);
    if (UNIT) tma_prefetch(&map_dqp);
    for (int i = 0; i < NBAR; ++i) {
      uint32_t cnt = 1;
      if (i == PF0 || i == PF1) cnt = kBwdExpWarps;
      if (i == KVE || i == DQE || i == DQE1) cnt = kBwdEpiWarps;
      if (i == LF0 || i == LF1) cnt = 32 * kBwdEpiWarps;
      if (i == LE0 || i == LE1) cnt = 32 * kBwdExpWarps;
      for (int t = 0; t < NT; ++t)
        for (int sl = 0; sl < (DB ? 2 : 1); ++sl)
          if (i == ER + qo_region(t, sl)) cnt = 2;  // post issuer's commit + the TMA warp's dO sums
      mbar_init(&bar[i], cnt);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the predecessor grid's outputs are complete (PDL launch)
  const uint32_t tdV = tmem + 256, tdK = tmem + 320, tdQ = tmem + 384;

  if (warp == 0) {
    int hi = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++hi) {
      const int bh = head_of(u, 0), jb = u % NU;  // head, key-tile block of the unit
      const int b = bh / p.H, h = bh % p.H;
      // regions in the order the previous unit releases them (whole head:
      // KV0, QO0, KV1, QO1; UNIT: QO0, QO1, KV, QO2)
      const int sl = slot_of(hi);
      int order[4] = {0, 0, 0, 0}, n_ord = 0;
      if (DB) {  // this head's slot: KV, then QO
        order[0] = kv_region(0, sl);
        order[1] = qo_region(0, sl);
        n_ord = 2;
      } else {
        for (int lu = 0; lu < NIT; ++lu)
          for (int r = 0; r < 4; ++r)
            if (last_use(r) == lu) order[n_ord++] = r;
      }
      for (int oi = 0; oi < n_ord; ++oi) {
        const int r = order[oi];
        const bool kv = UNIT ? r == 0 : r < 2;
        // smem tile (DB: the slot) and the tile's global rows (DB: tile 0)
        const int t = kv ? r : r - qo_region(0);  // key tile (KV) or query tile (QO)
        const int tg = DB ? 0 : t;
        mbar_wait(&bar[ER + r], par_of(hi) ^ 1);
        if (lane == 0) {
          mbar_expect_tx(&bar[FR + r], uint32_t(2 * kTile * kRowBytes));
          // PH: tile t is head 2u + t, rows 0..127 of that head
          const int bt = PH ? head_of(u, t) / p.H : b, ht = PH ? head_of(u, t) % p.H : h;
          if (kv) {
            const int kr = PH ? 0 : (jb * NK + tg) * kTile;  // global key row
            load_rows(sK + t * kTile * kRowBytes, &map_qkv, &bar[FR + r], HD + ht * kD, kr,
                      kTile, bt);
            load_rows(sV + t * kTile * kRowBytes, &map_qkv, &bar[FR + r], 2 * HD + ht * kD, kr,
                      kTile, bt);
          } else {
            load_rows(sQ + t * kTile * kRowBytes, &map_qkv, &bar[FR + r], ht * kD,
                      PH ? 0 : tg * kTile, kTile, bt);
            load_rows(sO + t * kTile * kRowBytes, &map_do, &bar[FR + r], ht * kD,
                      PH ? 0 : tg * kTile, kTile, bt);
          }
        }
      }
      if (lane == 0 && !UNIT && !PH) {
        // warm L2 with the next head's tiles
        const int nb = bh + gridDim.x;
        if (nb < n_heads) {
          const int b2 = nb / p.H, h2 = nb % p.H;
#pragma unroll
          for (int r = 0; r < Tr; r += kChunk) {
            tma_prefetch_3d(&map_qkv, h2 * kD, r, b2);
            tma_prefetch_3d(&map_do, h2 * kD, r, b2);
            tma_prefetch_3d(&map_qkv, HD + h2 * kD, r, b2);
            tma_prefetch_3d(&map_qkv, 2 * HD + h2 * kD, r, b2);
          }
        }
      }
      if (lane == 0 && UNIT && kBwdUnitPrefetch) {
        // warm L2 with the next unit's Q / dO and K / V tile: its K / V (and
        // last Q / dO tile) load only once this unit's last iteration is done
        const int nu = u + int(gridDim.x);
        if (nu < n_units) {
          const int bh2 = head_of(nu, 0), jb2 = nu % NU;
          const int b2 = bh2 / p.H, h2 = bh2 % p.H;
#pragma unroll
          for (int r = 0; r < Tr; r += kChunk) {
            tma_prefetch_3d(&map_qkv, h2 * kD, r, b2);
            tma_prefetch_3d(&map_do, h2 * kD, r, b2);
          }
#pragma unroll
          for (int r = 0; r < kTile; r += kChunk) {
            tma_prefetch_3d(&map_qkv, HD + h2 * kD, jb2 * kTile + r, b2);
            tma_prefetch_3d(&map_qkv, 2 * HD + h2 * kD, jb2 * kTile + r, b2);
          }
        }
      }
      __syncwarp();
      // V bias gradient = sum_q dO[q, :] of the head (rows of P sum to one),
      // from the dO tiles in smem by this warp's 32 lanes; the QO regions are
      // released by two arrivals (the post issuer's commit and this one).
      // The K bias gradient is exactly zero (softmax is shift-invariant per
      // query), so no K column sums are formed.
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      const int g = lane & 7, rs = lane >> 3;  // 16-byte column group, row set
      // (UNIT: the head's first key-tile unit forms the sums)
      const bool vsum = p.dbias != nullptr && (!UNIT || jb == 0);
      for (int t = 0; t < NT; ++t) {
        mbar_wait(&bar[FR + qo_region(t, sl)], par_of(hi));
        if (vsum) {
          const uint32_t o_s = smem_addr(sO);
          const int r0 = (t + sl) * kTile + rs * 32;  // (DB: the slot's rows)
#pragma unroll 4
          for (int r = r0; r < r0 + 32; ++r) {
            const uint4 w = ld_shared_v4(o_s + swz128(r, g));
            acc[0] += bf16_lo(w.x), acc[1] += bf16_hi(w.x), acc[2] += bf16_lo(w.y);
            acc[3] += bf16_hi(w.y), acc[4] += bf16_lo(w.z), acc[5] += bf16_hi(w.z);
            acc[6] += bf16_lo(w.w), acc[7] += bf16_hi(w.w);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar[ER + qo_region(t, sl)]);
        if (PH && vsum) {  // each query tile is its own head
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 8);
            acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 16);
          }
          if (lane < 8) {
            float* dst = p.dbias + 2 * HD + (head_of(u, t) % p.H) * kD + g * 8;
#pragma unroll
            for (int i = 0; i < 8; ++i) atomicAdd(dst + i, acc[i]);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = 0.f;
        }
      }
      if (vsum && !PH) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 8);
          acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 16);
        }
        if (lane < 8) {
          float* dst = p.dbias + 2 * HD + h * kD + g * 8;
#pragma unroll
          for (int i = 0; i < 8; ++i) atomicAdd(dst + i, acc[i]);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1 || warp == kBwdPostWarp) {
    // Two MMA issuers: warp 1 issues S^T / dP^T of each iteration, warp
    // kBwdPostWarp the dV / dK / dQ work that follows the exp warps, so the
    // next iteration's S^T / dP^T never queues behind a post.  Each issuer
    // runs converged (warp-uniform descriptors in uniform registers) and one
    // elected lane issues each MMA / commit; a commit tracks its own
    // thread's MMAs, so AC / KVF / DQF / EMPTY come from the post issuer.
    // Descriptor arithmetic: +2 per 16-element K slice of a K-major operand
    // (32 B), +128 per 16 K-rows of an MN-major one (2 KB), +8 per row (128 B).
    constexpr uint32_t idesc_kk = umma_idesc_bf16(128, kChunk, false, false);
    constexpr uint32_t idesc_km = umma_idesc_bf16(128, kD, false, true);
    constexpr uint32_t idesc_mm = umma_idesc_bf16(128, kD, true, true);
    if (warp == 1) {
      const uint64_t dQ0 = umma_sdesc(smem_addr(sQ), 16, 1024);
      const uint64_t dO0 = umma_sdesc(smem_addr(sO), 16, 1024);
      const uint64_t dK0 = umma_sdesc(smem_addr(sK), 16, 1024);
      const uint64_t dV0 = umma_sdesc(smem_addr(sV), 16, 1024);
      int hi = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++hi) {
        const int it0 = hi * NIT, sl = slot_of(hi);
        for (int k = 0; k < NIT; ++k) {
          const int it = it0 + k, bsel = k & 1;
          int j, c;
          jc(k, j, c);
          mbar_wait(&bar[FR + kv_region(j, sl)], par_of(hi));       // K_j, V_j of this unit
          mbar_wait(&bar[FR + qo_region(c >> 1, sl)], par_of(hi));  // Q, dO rows of chunk c
          if (k == 0) EPS_TRACE(hi < 16 && lane == 0, 640 + hi * 4 + 2);
          if (it >= 2) {  // post(it - 2) finished reading this S^T / dP^T buffer
            mbar_wait(&bar[AC0 + bsel], ((it >> 1) - 1) & 1);
          }
          tc_fence_after();
          const uint32_t tS = tmem + uint32_t(bsel * 128), tdP = tS + 64;
          const int jr = (j + sl) * kTile, qr = sl * kTile + c * kChunk;  // smem rows (DB slot)
          const uint64_t kj = dK0 + uint64_t(jr * 8), vj = dV0 + uint64_t(jr * 8);
          const uint64_t qc = dQ0 + uint64_t(qr * 8), oc = dO0 + uint64_t(qr * 8);
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk)
            tc_mma_ss_ws(tS, kj + uint64_t(2 * kk), qc + uint64_t(2 * kk), idesc_kk, kk > 0 ? 1u : 0u);
#pragma unroll
          for (int kk = 0; kk < kD / 16; ++kk)
            tc_mma_ss_ws(tdP, vj + uint64_t(2 * kk), oc + uint64_t(2 * kk), idesc_kk, kk > 0 ? 1u : 0u);
          tc_commit_ws(&bar[SF0 + bsel]);
          if (kBwdSFirst) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar[SI0 + bsel]);
          }
          EPS_TRACE(it < 64 && lane == 0, it * 8 + 0);
        }
      }
    } else {
      const uint64_t mQ0 = umma_sdesc(smem_addr(sQ), 64 * 128, 1024);
      const uint64_t mO0 = umma_sdesc(smem_addr(sO), 64 * 128, 1024);
      const uint64_t mK0 = umma_sdesc(smem_addr(sK), 64 * 128, 1024);
      const uint64_t mS0 = umma_sdesc(smem_addr(sS), kDsChunk, 1024);
      int kt = 0, hi = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++hi) {
        const int sl = slot_of(hi);
        for (int k = 0; k < NIT; ++k) {
          const int it = hi * NIT + k, bsel = k & 1;
          int j, c;
          jc(k, j, c);
          mbar_wait(&bar[PF0 + bsel], (it >> 1) & 1);
          tc_fence_after();
          EPS_TRACE(it < 64 && lane == 0, it * 8 + 1);
          if ((PH ? (c & 1) == 0 : c == 0) && kt > 0) {  // dK / dV of the previous key tile read out
            mbar_wait(&bar[KVE], (kt - 1) & 1);
            tc_fence_after();
          }
          const uint32_t tS = tmem + uint32_t(bsel * 128), tdP = tS + 64;
          const int qr = sl * kTile + c * kChunk;  // smem rows of chunk c (DB: the slot's)
          const uint64_t qc = mQ0 + uint64_t(qr * 8), oc = mO0 + uint64_t(qr * 8);
          // dK_j += dS^T Q_c with dS^T read from its smem staging tile (K-major,
          // [128 keys][64 queries]): an SS MMA is ~15 % cheaper than the TS form
          // (tools/mma_rate.cu: M = 128, N = 64, K = 16 in 89 vs 105 cycles)
          const uint64_t dsk = umma_sdesc(smem_addr(sS) + uint32_t(((it >> 1) & 1) * 2 + (c & 1)) *
                                              uint32_t(kDsChunk),
                                          16, 1024);
#pragma unroll
          for (int kk = 0; kk < kChunk / 16; ++kk) {
            // dV / dK of key tile j start at its first chunk (PH: chunk 2j)
            const uint32_t acc = ((PH ? (c & 1) : c) > 0 || kk > 0) ? 1u : 0u;
            const uint32_t pcol = uint32_t(pk_col(kk));  // see the exp loop
            tc_mma_ts_ws(tdV, tS + pcol, oc + uint64_t(kk * 128), idesc_km, acc);
            if (kBwdDkSS)
              tc_mma_ss_ws(tdK, dsk + uint64_t(2 * kk), qc + uint64_t(kk * 128), idesc_km, acc);
            else
              tc_mma_ts_ws(tdK, tdP + pcol, qc + uint64_t(kk * 128), idesc_km, acc);
          }
          // P^T / dS^T in this TMEM buffer are consumed: release it to the S
          // issuer before the dQ MMAs (they read dS from the smem staging)
          tc_commit_ws(&bar[AC0 + bsel]);
          const bool tile_end = PH ? (c & 1) == 1 : c == NC - 1;  // last chunk of key tile j
          if (tile_end) tc_commit_ws(&bar[KVF]);
          if (c & 1) {  // both halves of 128-query tile c/2 staged: dQ_t += dS_t K_j
            const int t = c >> 1;
            // S^T / dP^T of iteration it + 2 (the next user of the TMEM buffer
            // just released) go into the tensor pipe before these dQ MMAs,
            // so the exp warps find them complete (same head only: the next
            // head's first S may wait for K regions these dQ MMAs release)
            if (kBwdSFirst && k + 2 < NIT) mbar_wait(&bar[SI0 + bsel], ((it + 2) >> 1) & 1);
            const int g = hi * NT + t;  // UNIT: dQ tile counter -> buffer g & 1
            if (UNIT) {
              if (g >= 2) {  // the epilogue read out buffer g & 1's previous tile
                mbar_wait(&bar[(g & 1) ? DQE1 : DQE], ((g >> 1) - 1) & 1);
                tc_fence_after();
              }
            } else if (j == 0 && t == 0 && hi > 0) {
              mbar_wait(&bar[DQE], (hi - 1) & 1);
              tc_fence_after();
            }
            const uint64_t stg = mS0 + uint64_t(((it >> 1) & 1) * 2 * (kDsChunk >> 4));
            const uint64_t kj = mK0 + uint64_t((j + sl) * kTile * 8);
            const uint32_t tq = tdQ + uint32_t((UNIT ? (g & 1) : t) * kD);
#pragma unroll
            for (int kk = 0; kk < kTile / 16; ++kk)
              tc_mma_ss_ws(tq, stg + uint64_t(kk * 128), kj + uint64_t(kk * 128), idesc_mm,
                           ((!UNIT && !PH && j > 0) || kk > 0) ? 1u : 0u);
            if (UNIT) tc_commit_ws(&bar[(g & 1) ? DQF1 : DQF]);
          }
          EPS_TRACE(it < 64 && lane == 0, it * 8 + 2);
          if (tile_end) ++kt;
          // operand regions whose last reader this was (tracks the dQ MMAs too)
          if (DB) {
            if (k == NIT - 1) {
              tc_commit_ws(&bar[ER + kv_region(0, sl)]);
              tc_commit_ws(&bar[ER + qo_region(0, sl)]);
            }
          } else {
#pragma unroll
            for (int r = 0; r < 4; ++r)
              if (last_use(r) == k) tc_commit_ws(&bar[ER + r]);
          }
        }
        if (!UNIT) tc_commit_ws(&bar[DQF]);
      }
    }
  } else if (warp < 2 + kBwdExpWarps) {
    // ---- exp / dS warps --------------------------------------------------
    // 4 warps per TMEM lane quarter; warp `sub` of a quarter owns queries
    // [sub*QPW, +QPW) of each 64-query chunk and S^T / dP^T columns of the
    // same range, and writes its packed bf16 P^T / dS^T inside that range
    // (already read), so warps never wait on each other; the MMAs address
    // the pieces (pk_col).
    const int sub = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const float sl2 = p.scale_log2;
    int hi = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++hi) {
      const int jb = u % NU;
      const int lb = hi & 1;
      mbar_wait(&bar[LF0 + lb], (hi >> 1) & 1);
      EPS_TRACE(hi < 16 && warp == 2 && lane == 0, 640 + hi * 4 + 3);
      const uint32_t ld = smem_addr(sLD + lb * Tr);
#pragma unroll 1
      for (int k = 0; k < NIT; ++k) {
        const int it = hi * NIT + k, bsel = k & 1;
        int j, c;
        jc(k, j, c);
        // this warp's 32 keys (index within the key tile's head for PH)
        const int kbase = PH ? quarter * 32 : (jb * NK + j) * kTile + quarter * 32;
        const int q0 = c * kChunk + sub * kBwdQPW;
        mbar_wait(&bar[SF0 + bsel], (it >> 1) & 1);
        tc_fence_after();
        EPS_TRACE(it < 64 && warp == 2 && lane == 0, it * 8 + 3);
        const uint32_t tS = tmem + uint32_t(bsel * 128) + (uint32_t(quarter * 32) << 16);
        const uint32_t tdP = tS + 64;
        const uint32_t chunk = smem_addr(sS) +
                               uint32_t(((it >> 1) & 1) * 2 + (c & 1)) * uint32_t(kDsChunk) +
                               uint32_t(row >> 3) * 1024u;
        // Query columns past T need no mask: their Q / dO rows are zero-filled
        // and -lse2 = D = 0, so P^T = 1 and dS^T = 0, and dV += P^T dO adds
        // zero rows.  Keys past T are masked per warp (P^T = dS^T = 0, so an
        // extreme lse can never reach the dQ MMA as inf * 0).
        if (kbase >= p.T) {
          const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
          for (int hh = 0; hh < kBwdPasses; ++hh) {
            tmem_st_32x32_x8(tS + uint32_t(pk_col(sub * kBwdPasses + hh)), z);
            tmem_st_32x32_x8(tdP + uint32_t(pk_col(sub * kBwdPasses + hh)), z);
#pragma unroll
            for (int v = 0; v < 2; ++v)
              st_shared_v4(chunk + uint32_t(swz128(row & 7, (sub * kBwdQPW + hh * 16) / 8 + v)),
                           0u, 0u, 0u, 0u);
          }
        } else {
          const bool mixed = kbase + 32 > p.T;
          const bool kvalid = kbase + lane < p.T;
          uint32_t sv[kBwdPasses][16], dp[kBwdPasses][16];
#pragma unroll
          for (int hh = 0; hh < kBwdPasses; ++hh) {
            tmem_ld_32x32_x16(tS + uint32_t(sub * kBwdQPW + hh * 16), sv[hh]);
            tmem_ld_32x32_x16(tdP + uint32_t(sub * kBwdQPW + hh * 16), dp[hh]);
          }
          tmem_ld_wait();
#pragma unroll
          for (int hh = 0; hh < kBwdPasses; ++hh) {
            const uint32_t l4 = ld + uint32_t(q0 + hh * 16) * 8u;
            uint32_t pp[8], pd[8];
            if (((q0 + hh * 16) & (PH ? kTile - 1 : 0x7fffffff)) >= p.T) {
              // 16 query columns wholly past T (up to 23 % of a ViT head's
              // columns): their dO rows are zero, so P^T = dS^T = 0 is exact
              // and the exps are skipped
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) pp[jj] = pd[jj] = 0u;
            } else {
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const uint4 w = ld_shared_v4(l4 + 16u * jj);  // (-lse2, D) of queries 2jj, 2jj+1
              const float4 a = make_float4(__uint_as_float(w.x), __uint_as_float(w.y),
                                           __uint_as_float(w.z), __uint_as_float(w.w));
              float p0 = fast_exp2(fmaf(__uint_as_float(sv[hh][2 * jj]), sl2, a.x));
              float p1 = fast_exp2(fmaf(__uint_as_float(sv[hh][2 * jj + 1]), sl2, a.z));
              if (mixed) {
                p0 = kvalid ? p0 : 0.f;
                p1 = kvalid ? p1 : 0.f;
              }
              pp[jj] = pack_bf16(p0, p1);
              pd[jj] = pack_bf16(p0 * (__uint_as_float(dp[hh][2 * jj]) - a.y),
                                 p1 * (__uint_as_float(dp[hh][2 * jj + 1]) - a.w));
            }
            }
            tmem_st_32x32_x8(tS + uint32_t(pk_col(sub * kBwdPasses + hh)), pp);
            if (!kBwdDkSS) tmem_st_32x32_x8(tdP + uint32_t(pk_col(sub * kBwdPasses + hh)), pd);
#pragma unroll
            for (int v = 0; v < 2; ++v)
              st_shared_v4(chunk + uint32_t(swz128(row & 7, (sub * kBwdQPW + hh * 16) / 8 + v)),
                           pd[4 * v], pd[4 * v + 1], pd[4 * v + 2], pd[4 * v + 3]);
          }
        }
        fence_proxy_async_smem();
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar[PF0 + bsel]);
        EPS_TRACE(it < 64 && warp == 2 && lane == 0, it * 8 + 4);
      }
      mbar_arrive(&bar[LE0 + lb]);  // done reading this head's (-lse2, D) table
    }
  } else if (warp < 2 + kBwdExpWarps + kBwdEpiWarps) {
    // ---- epilogue warps ----------------------------------------------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const int te = threadIdx.x - (64 + 32 * kBwdExpWarps);  // 0..127
    // (-lse * log2e, D = rowsum(dO * O)) of every query of head `bh` into
    // table hi & 1, once the exp warps released it (head hi - 2).
    // bh: the unit's (first) head; PH: rows 128 r .. of the table are head bh + r
    auto fill_table = [&](int bh, int hi) {
      const int lb = hi & 1;
      if (hi >= 2) mbar_wait(&bar[LE0 + lb], ((hi >> 1) - 1) & 1);
      EPS_TRACE(hi < 16 && warp == 2 + kBwdExpWarps && lane == 0, 704 + hi * 2);
#pragma unroll
      for (int r = 0; r < Tr / 128; ++r) {
        const int q = te + 128 * r;
        const int bhr = PH ? bh + r : bh, ql = PH ? te : q;
        const int b = bhr / p.H, h = bhr % p.H;
        // queries past T: -lse2 = D = 0 (see the exp loop)
        float2 e = make_float2(0.f, 0.f);
        if (ql < p.T)
          e = make_float2(-__ldg(p.lse + int64_t(bhr) * p.T + ql) * kLog2e,
                          __ldg(p.drow + (int64_t(b) * p.T + ql) * p.H + h));
        sLD[lb * Tr + q] = e;
      }
      mbar_arrive(&bar[LF0 + lb]);
      EPS_TRACE(hi < 16 && warp == 2 + kBwdExpWarps && lane == 0, 704 + hi * 2 + 1);
    };
    // Tiles leave through a swizzled 16 KB staging buffer and TMA stores
    // (coalesced, asynchronous); `te == 0` owns the bulk groups.
    auto epi_sync = [] { asm volatile("bar.sync 1, 128;" ::: "memory"); };
    int stg = 0;  // staging tile of the next store
    auto store_tile_to = [&](const CUtensorMap* map, const uint32_t (&pk)[32], int col, int row0,
                             int z) {
      uint8_t* buf = sStage + stg * kDsChunk;
      const uint32_t stage_s = smem_addr(buf);
      stg = stg + 1 == NSTG ? 0 : stg + 1;
      if (te == 0) bulk_wait_read<NSTG - 1>();  // this buffer's previous tile read out
      epi_sync();
#pragma unroll
      for (int c = 0; c < 8; ++c)
        st_shared_v4(stage_s + swz128(row, c), pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
      fence_proxy_async_smem();
      epi_sync();
      if (te == 0) {
        tma_store_3d(map, buf, col, row0, z);
        tma_store_3d(map, buf + 64 * kRowBytes, col, row0 + 64, z);
        bulk_commit();
      }
    };
    auto store_tile = [&](const uint32_t (&pk)[32], int col, int row0, int b) {
      store_tile_to(&map_dq, pk, col, row0, b);
    };
    int hi = 0, kt = 0;
    if (int(blockIdx.x) < n_units) fill_table(head_of(int(blockIdx.x), 0), 0);
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++hi) {
      const int bh = head_of(u, 0), jb = u % NU;
      const int b = bh / p.H, h = bh % p.H;
      if constexpr (UNIT) {
        // dQ partials of the unit's key tile, one 128-query tile at a time
        for (int t = 0; t < NT; ++t) {
          const int g = hi * NT + t;
          mbar_wait(&bar[(g & 1) ? DQF1 : DQF], (g >> 1) & 1);
          tc_fence_after();
          uint32_t pq[32];
          load_tmem_packed64(tdQ + uint32_t((g & 1) * kD) + lane_off, p.scale, pq);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bar[(g & 1) ? DQE1 : DQE]);
          store_tile_to(&map_dqp, pq, h * kD, t * kTile, jb * (n_heads / p.H) + b);
          if (t == 0 && u + int(gridDim.x) < n_units)
            fill_table(head_of(u + int(gridDim.x), 0), hi + 1);
        }
        mbar_wait(&bar[KVF], kt & 1);
        tc_fence_after();
        uint32_t pv[32], pk[32];
        load_tmem_packed64(tdV + lane_off, 1.f, pv);
        load_tmem_packed64(tdK + lane_off, p.scale, pk);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar[KVE]);
        store_tile(pv, 2 * HD + h * kD, jb * kTile, b);
        store_tile(pk, HD + h * kD, jb * kTile, b);
        ++kt;
        continue;
      }
      // NT = 1: the next head's table first -- its exp work can start as soon
      // as this head's last S^T is consumed, before dV / dK / dQ are out
      if (kBwdEarlyTable && NT == 1 && u + int(gridDim.x) < n_units)
        fill_table(head_of(u + int(gridDim.x), 0), hi + 1);
      // TMEM is read out and released first (the MMA warp is waiting for
      // it); stores work from the packed registers.
      for (int j = 0; j < NT; ++j, ++kt) {
        mbar_wait(&bar[KVF], kt & 1);
        tc_fence_after();
        EPS_TRACE(kt < 64 && warp == 2 + kBwdExpWarps && lane == 0, 512 + kt * 2);
        uint32_t pv[32], pk[32];
        load_tmem_packed64(tdV + lane_off, 1.f, pv);
        load_tmem_packed64(tdK + lane_off, p.scale, pk);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar[KVE]);
        EPS_TRACE(kt < 64 && warp == 2 + kBwdExpWarps && lane == 0, 512 + kt * 2 + 1);
        {
          const int hbj = head_of(u, PH ? j : 0), bj = hbj / p.H, hj = hbj % p.H;
          store_tile(pv, 2 * HD + hj * kD, PH ? 0 : j * kTile, bj);
          store_tile(pk, HD + hj * kD, PH ? 0 : j * kTile, bj);
        }
        EPS_TRACE(hi < 16 && j == 0 && warp == 2 + kBwdExpWarps && lane == 0, 760 + hi * 4 + 2);
        // the next unit's table, off the key-tile hand-off path (its exp work
        // starts only after this unit's remaining iterations)
        if (j == 0 && !(kBwdEarlyTable && NT == 1) && u + int(gridDim.x) < n_units)
          fill_table(head_of(u + int(gridDim.x), 0), hi + 1);
      }
      mbar_wait(&bar[DQF], hi & 1);
      tc_fence_after();
      EPS_TRACE(hi < 16 && warp == 2 + kBwdExpWarps && lane == 0, 640 + hi * 4);
      uint32_t pq[UNIT ? 1 : NT][32];
#pragma unroll
      for (int t = 0; t < (UNIT ? 1 : NT); ++t) load_tmem_packed64(tdQ + uint32_t(t * kD) + lane_off, p.scale, pq[t]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[DQE]);
      EPS_TRACE(hi < 16 && warp == 2 + kBwdExpWarps && lane == 0, 640 + hi * 4 + 1);
#pragma unroll
      for (int t = 0; t < (UNIT ? 1 : NT); ++t) {
        const int hbt = head_of(u, PH ? t : 0);
        if ((PH ? row : t * kTile + row) >= p.T) zero32(pq[t]);
        store_tile(pq[t], (hbt % p.H) * kD, PH ? 0 : t * kTile, hbt / p.H);
      }
      if (p.dbias != nullptr) {  // Q bias gradient: column sums of dQ (PH: per head)
#pragma unroll
        for (int grp = 0; grp < (PH ? NT : 1); ++grp) {
          float uu[64];
#pragma unroll
          for (int d = 0; d < 32; ++d) {
            uu[2 * d] = 0.f;
            uu[2 * d + 1] = 0.f;
#pragma unroll
            for (int t = 0; t < (UNIT ? 1 : NT); ++t)
              if (!PH || t == grp) uu[2 * d] += bf16_lo(pq[t][d]), uu[2 * d + 1] += bf16_hi(pq[t][d]);
          }
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float t32[32];
#pragma unroll
            for (int d = 0; d < 32; ++d) t32[d] = uu[half * 32 + d];
            sRed[quarter * 64 + half * 32 + lane] = warp_transpose_sum32(t32);
          }
          epi_sync();
          if (te < 64)
            atomicAdd(p.dbias + (head_of(u, PH ? grp : 0) % p.H) * kD + te,
                      sRed[te] + sRed[64 + te] + sRed[128 + te] + sRed[192 + te]);
          epi_sync();
        }
      }
      EPS_TRACE(hi < 16 && warp == 2 + kBwdExpWarps && lane == 0, 760 + hi * 4);
    }
    if (te == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

size_t bwd_fused_smem(int T) {
  const int nt = (T + kTile - 1) / kTile;
  const int Tr = (T + kTile - 1) / kTile * kTile;
  const int KR = Tr > 2 * kTile ? kTile : Tr;  // UNIT (T > 256): one key tile per unit
  // T <= 128: two operand slots (the kernel's DB layout)
  const int ops = Tr == kTile && kBwdDoubleBuffer ? 2 : 1;
  return size_t(ops * (2 * Tr + 2 * KR)) * kRowBytes +
         size_t(4 + bwd_stage_tiles(nt > 3 ? 3 : nt)) * size_t(kDsChunk) + size_t(2 * Tr) * 8 +
         1024 /* sRed */ + 1024 + 256;
}

// ---------------------------------------------------------------------------
// Persistent forward for T <= 256, two ping-pong pipelines per CTA.  One CTA
// per SM walks the (b, h) heads; pipeline c (one MMA-issuer warp + one
// softmax warpgroup + smem buffer c + TMEM context c) takes every other head
// and runs both of its 128-query tiles in turn:
//   S = Q_t K^T -> TMEM context c (N = Tp <= 256 columns)
//   row max, exp2, row sum; P written back as bf16 into the S columns
//   O = P V, a TS-form MMA (A = P from TMEM) into columns 128..191 of c
//   O / rowsum -> bf16 -> global, lse
// The two pipelines are decoupled, so one's MMAs and latencies overlap the
// other's exp work (the SFU is the floor: T*Tp exp2 per head).  (The
// previous design ran both tiles of one head in lock step, so the two
// warpgroups waited on the same MMAs and competed for the SFU at the same
// time.)  A single TMA warp loads head i into buffer i & 1.
constexpr int kFwdThreads = 12 * 32;  // TMA, MMA0, MMA1, (alloc), WG0 (4-7), WG1 (8-11)

// POLY of the 16 exp pairs of a full 32-key chunk run as poly_exp2_x2 on the
// FMA / ALU pipes, the rest on the SFU (evenly interleaved).
template <int POLY>
__device__ __forceinline__ constexpr bool fwd_poly_pair(int j) {
  return (j * POLY) / 16 != ((j + 1) * POLY) / 16;
}

// V2 (round 2): the overflow test of chunks after the first reads their exp
// sum instead of a 32-key max (as in attn_fwd_ring_tc_kernel), the first
// chunk's max is an FMNMX3 tree, and warps whose rows are all >= T skip the
// softmax and the O read-out.
template <int POLY, bool V2>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_persistent_tc_kernel(const __grid_constant__ CUtensorMap map_qkv, const Params p,
                                  int n_heads) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int nt = (p.T + kTile - 1) / kTile;
  const int Tr = nt * kTile;
  // S columns: N = pad16(T) <= 256 (keys T..Tn-1 hit the zero-filled K rows;
  // their P is written as 0, and the PV contraction stops at Tn)
  const int Tn = (p.T + 15) / 16 * 16;
  const size_t buf_bytes = size_t(3 * Tr) * kRowBytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * buf_bytes);
  // per pipeline c: full / empty of the operand regions Q_0, Q_1, K, V (so the
  // next head's Q_0 loads once S(tile 0) is done, K and Q_1 after S(tile 1),
  // V after the last PV), SF (S ready), PF (P written), OF (O ready), TF (O
  // read out)
  enum { FQ0 = 0, FQ1, FK, FV, EQ0, EQ1, EK, EV, SF, PF, OF, TF, NB };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2 * NB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HD = p.H * kD;

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    for (int c = 0; c < 2; ++c)
      for (int i = 0; i < NB; ++i) mbar_init(&bar[c * NB + i], (i == PF || i == TF) ? 4 : 1);
    mbar_fence_init();
  }
  if (warp == 3) tmem_alloc(tmem_slot, 512);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // the predecessor grid's outputs are complete (PDL launch)

  if (warp == 0 || warp == 3) {
    // TMA producer of pipeline c (warp 0: c = 0, warp 3: c = 1), region by
    // region in the order the previous head of the pipeline releases them
    const int c = warp == 0 ? 0 : 1;
    uint64_t* pb = bar + c * NB;
    uint8_t* base = smem + c * buf_bytes;
    if (lane == 0) {
      int i = 0;
      for (int bh = blockIdx.x; bh < n_heads; bh += gridDim.x, ++i) {
        if ((i & 1) != c) continue;
        const int b = (p.dbg & 1) ? 0 : bh / p.H, h = (p.dbg & 1) ? 0 : bh % p.H;
        const uint32_t par = ((i >> 1) & 1) ^ 1;
        for (int t = 0; t < nt; ++t) {
          mbar_wait(&pb[EQ0 + t], par);
          mbar_expect_tx(&pb[FQ0 + t], uint32_t(kTile * kRowBytes));
          load_rows(base + t * kTile * kRowBytes, &map_qkv, &pb[FQ0 + t], h * kD, t * kTile,
                    kTile, b);
          if (t == 0) {
            mbar_wait(&pb[EK], par);
            mbar_expect_tx(&pb[FK], uint32_t(Tr * kRowBytes));
            load_rows(base + Tr * kRowBytes, &map_qkv, &pb[FK], HD + h * kD, 0, Tr, b);
          }
        }
        mbar_wait(&pb[EV], par);
        mbar_expect_tx(&pb[FV], uint32_t(Tr * kRowBytes));
        load_rows(base + 2 * Tr * kRowBytes, &map_qkv, &pb[FV], 2 * HD + h * kD, 0, Tr, b);
      }
    }
  } else if (warp == 1 || warp == 2) {
    // MMA issuer of pipeline c, warp-converged (one elected lane issues)
    const int c = warp - 1;
    uint64_t* pb = bar + c * NB;
    const uint32_t tS = tmem + uint32_t(256 * c);
    const uint32_t idesc_s = umma_idesc_bf16(128, Tn, false, false);
    const uint32_t idesc_o = umma_idesc_bf16(128, kD, false, true);
    int i = 0, k = 0;  // k: tiles done by this pipeline
    for (int bh = blockIdx.x; bh < n_heads; bh += gridDim.x, ++i) {
      if ((i & 1) != c) continue;
      const int n = i >> 1;  // this pipeline's head count
      const uint64_t q0 = umma_sdesc(smem_addr(smem + c * buf_bytes), 16, 1024);
      const uint64_t k0 = q0 + uint64_t((Tr * kRowBytes) >> 4);
      const uint64_t v0 = umma_sdesc(smem_addr(smem + c * buf_bytes + 2 * Tr * kRowBytes),
                                     64 * 128, 1024);
      for (int t = 0; t < nt; ++t, ++k) {
        if (k > 0)  // the warpgroup has read out the previous tile's O
          mbar_wait(&pb[TF], (k - 1) & 1);
        mbar_wait(&pb[FQ0 + t], n & 1);
        mbar_wait(&pb[FK], n & 1);
        tc_fence_after();
        const uint64_t qt = q0 + uint64_t((t * kTile * kRowBytes) >> 4);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          tc_mma_ss_ws(tS, qt + uint64_t(2 * kk), k0 + uint64_t(2 * kk), idesc_s, kk > 0 ? 1u : 0u);
        tc_commit_ws(&pb[SF]);
        tc_commit_ws(&pb[EQ0 + t]);             // Q_t read
        if (t == nt - 1) tc_commit_ws(&pb[EK]);  // K read by the last S
        EPS_TRACE(c == 0 && k < 32 && lane == 0, 832 + k * 5);
        mbar_wait(&pb[PF], k & 1);
        if (t == 0) mbar_wait(&pb[FV], n & 1);
        tc_fence_after();
        for (int kk = 0; kk < Tn / 16; ++kk)
          tc_mma_ts_ws(tS + 128, tS + uint32_t(kk * 8), v0 + uint64_t(kk * 128), idesc_o,
                       kk > 0 ? 1u : 0u);
        tc_commit_ws(&pb[OF]);
      }
      tc_commit_ws(&pb[EV]);  // V read by the last PV
    }
  } else if (warp >= 4) {
    const int c = (warp - 4) >> 2;  // pipeline of this warpgroup
    uint64_t* pb = bar + c * NB;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    const uint32_t tS = tmem + uint32_t(256 * c) + lane_off;
    const float sl2 = p.scale_log2;
    int i = 0, k = 0;
    for (int bh = blockIdx.x; bh < n_heads; bh += gridDim.x, ++i) {
      if ((i & 1) != c) continue;
      const int b = bh / p.H, h = bh % p.H;
      for (int t = 0; t < nt; ++t, ++k) {
        const int q = t * kTile + row;
        mbar_wait(&pb[SF], k & 1);
        tc_fence_after();
        EPS_TRACE(c == 0 && k < 32 && warp == 4 && lane == 0, 832 + k * 5 + 1);
        // One pass over S.  The exponent reference ms is the max of chunk 0,
        // not the row max: any reference within a few dozen binades of the row
        // max gives the same P / rowsum in fp32 and bf16 (both scale-free), so
        // the separate max pass (a second TMEM read of S, the binding
        // bandwidth here) is skipped.  A chunk whose max exceeds ms by more
        // than 2^32 rescales the P chunks already written (warp-collective,
        // rare) and raises ms.
        float ms = 0.f;
        const float2 sl2x2 = make_float2(sl2, sl2);
        float2 sum2 = make_float2(0.f, 0.f);  // two interleaved partial sums (packed FADD2)
        const int nch = (Tn + 31) / 32;
        uint32_t ra[32];
        auto issue = [&](int ch, uint32_t(&r)[32]) {
          if (p.T - ch * 32 <= 16)
            tmem_ld_32x32_x16(tS + uint32_t(ch * 32), reinterpret_cast<uint32_t(&)[16]>(r));
          else
            tmem_ld_32x32(tS + uint32_t(ch * 32), r);
        };
        auto process = [&](int ch, uint32_t(&r)[32]) {
          uint32_t pk[16];
          const int rem = p.T - ch * 32;  // valid keys in this chunk (>= 1)
          // the chunk max is needed up front only for chunk 0; later chunks
          // compute exps and max side by side and redo the exps on a rescale
          auto chunk_max = [&]() {
            float cm = -FLT_MAX;
            if (V2 && rem >= 32) {
              float m1 = -FLT_MAX, m2 = -FLT_MAX, m3 = -FLT_MAX;
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                cm = fmax3f(cm, __uint_as_float(r[j]), __uint_as_float(r[j + 1]));
                m1 = fmax3f(m1, __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                m2 = fmax3f(m2, __uint_as_float(r[j + 4]), __uint_as_float(r[j + 5]));
                m3 = fmax3f(m3, __uint_as_float(r[j + 6]), __uint_as_float(r[j + 7]));
              }
              cm = fmaxf(fmaxf(cm, m1), fmaxf(m2, m3));
            } else if (rem >= 32) {
#pragma unroll
              for (int j = 0; j < 32; ++j) cm = fmaxf(cm, __uint_as_float(r[j]));
            } else if (rem <= 16) {
#pragma unroll
              for (int j = 0; j < 16; ++j)
                if (j < rem) cm = fmaxf(cm, __uint_as_float(r[j]));
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (j < rem) cm = fmaxf(cm, __uint_as_float(r[j]));
            }
            return cm * sl2;
          };
          auto chunk_exp = [&](float msr) {
            const float2 nms2 = make_float2(-msr, -msr);
            float2 cs = make_float2(0.f, 0.f);
            if (rem >= 32) {  // full chunk: no key mask; POLY of the 16 pairs on the FMA pipe
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float2 a = __ffma2_rn(
                    make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])), sl2x2, nms2);
                const float2 e = fwd_poly_pair<POLY>(j) ? poly_exp2_x2<V2>(a)
                                                        : make_float2(fast_exp2(a.x), fast_exp2(a.y));
                cs = __fadd2_rn(cs, e);
                pk[j] = pack_bf16(e.x, e.y);
              }
            } else if (rem <= 16) {  // tail chunk with <= 16 valid keys: half the exps
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float2 a = __ffma2_rn(
                    make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])), sl2x2, nms2);
                const float2 e = make_float2(2 * j < rem ? fast_exp2(a.x) : 0.f,
                                             2 * j + 1 < rem ? fast_exp2(a.y) : 0.f);
                cs = __fadd2_rn(cs, e);
                pk[j] = pack_bf16(e.x, e.y);
              }
#pragma unroll
              for (int j = 8; j < 16; ++j) pk[j] = 0u;
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float2 a = __ffma2_rn(
                    make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])), sl2x2, nms2);
                const float2 e = make_float2(2 * j < rem ? fast_exp2(a.x) : 0.f,
                                             2 * j + 1 < rem ? fast_exp2(a.y) : 0.f);
                cs = __fadd2_rn(cs, e);
                pk[j] = pack_bf16(e.x, e.y);
              }
            }
            return cs;
          };
          if (ch == 0) ms = chunk_max();
          float2 cs = chunk_exp(ms);
          if (ch > 0) {
            // V2: an exp sum above 2^32 (or inf) means a key leads ms by > 2^27
            const float cms = V2 ? 0.f : chunk_max();
            const bool up = V2 ? cs.x + cs.y > 4294967296.0f : cms > ms + 32.f;
            if (__any_sync(0xffffffffu, up)) {
              const float ms_new = up ? (V2 ? fmaxf(ms, chunk_max()) : cms) : ms;
              const float f = fast_exp2(ms - ms_new);  // 1 on lanes without overflow
              sum2 = __fmul2_rn(sum2, make_float2(f, f));
              tmem_st_wait();
              for (int pc = 0; pc < ch; ++pc) {
                uint32_t q16[16];
                tmem_ld_32x32_x16(tS + uint32_t(pc * 16), q16);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j)
                  q16[j] = pack_bf16(bf16_lo(q16[j]) * f, bf16_hi(q16[j]) * f);
                tmem_st_32x32_x16(tS + uint32_t(pc * 16), q16);
              }
              ms = ms_new;
              cs = chunk_exp(ms);
            }
          }
          sum2 = __fadd2_rn(sum2, cs);
          tmem_st_32x32_x16(tS + uint32_t(ch * 16), pk);
        };
        // (a register double-buffered variant -- the load of chunk ch + 1 in
        // flight while chunk ch is exponentiated -- measured 10 % slower)
        const bool live = !V2 || t * kTile + quarter * 32 < p.T;  // warp-uniform
        if (live) {
          for (int ch = 0; ch < nch; ++ch) {
            issue(ch, ra);
            tmem_ld_wait_regs(ra);
            process(ch, ra);
          }
        }
        const float sum = sum2.x + sum2.y;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pb[PF]);
        EPS_TRACE(c == 0 && k < 32 && warp == 4 && lane == 0, 832 + k * 5 + 2);
        if (q < p.T) p.lse[int64_t(bh) * p.T + q] = (ms + __log2f(sum)) * kLn2;
        mbar_wait(&pb[OF], k & 1);
        tc_fence_after();
        EPS_TRACE(c == 0 && k < 32 && warp == 4 && lane == 0, 832 + k * 5 + 3);
        float o[64];
        if (live) load_tmem_row64(tS + 128, o);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pb[TF]);
        EPS_TRACE(c == 0 && k < 32 && warp == 4 && lane == 0, 832 + k * 5 + 4);
        if (q < p.T) {
          const float inv = 1.f / sum;
#pragma unroll
          for (int j = 0; j < 64; ++j) o[j] *= inv;
          store_row64(p.out_w + (int64_t(b) * p.T + q) * HD + h * kD, o);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 3) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

size_t fwd_persistent_smem(int T) {
  const int Tr = (T + kTile - 1) / kTile * kTile;
  return 2 * size_t(3 * Tr) * kRowBytes + 1024 + 256;
}

// ---------------------------------------------------------------------------
// Ring forward for T <= 256 (the default since round 2).  Same roles and
// Q / K / V smem buffers as attn_fwd_persistent_tc_kernel (one TMA warp, one
// MMA warp and one softmax warpgroup per pipeline c, heads alternating
// between the two pipelines), but the softmax warpgroups never wait for a
// tile's O: the persistent kernel's per-tile chain
//   S (all keys) -> softmax -> PV -> O read-out -> next S
// kept a warpgroup busy ~5.0 k of ~7.9 k cycles per tile (CTA-0 clock trace,
// ViT-B/16).  Here keys go in blocks of 64 through a ring of three 64-column
// S slots per pipeline; O owns the pipeline's first 64 TMEM columns:
//   pipeline c: O [256c, 256c + 64), slot s [256c + 64 + 64s, +64)
//   MMA warp:  S(g) = Q_t K_j^T into slot g % 3 up to two blocks ahead of
//              the block it feeds to PV (in-order tensor pipe: S(g + 3) is
//              issued after PV(g), which read slot g % 3 as P);
//              PV(g): O (+)= P_g V_j (TS form, P packed bf16 in the slot)
//   softmax:   block by block, one row per thread; P written back packed
//              into the slot's first 32 columns; after block 0 of tile k it
//              reads O(k-1) (complete: OF) and only then releases P(k, 0),
//              so PV(k, 0) (accumulate = 0) cannot overwrite an unread O.
//              O(k-1) / rowsum goes out through a per-warp 32-row smem stage
//              and a TMA store (rows >= T clipped by the tensor map).
// Softmax per row: the exponent reference is the max of the first 32 keys
// (FMNMX3 tree); later chunks test their exp sum instead of a max: a sum
// above 2^32 (or inf) means some key leads the reference by > 2^27, and the
// chunk is redone after rescaling the row sum, the block's earlier P chunk
// and -- when earlier blocks already went to PV -- O (rare, warp-collective).
// Warps whose 32 rows are all >= T (the last query tile's padding) skip the
// softmax and only arrive.
constexpr int kRingSlots = 3;
constexpr int kStageBytes = 32 * kRowBytes;  // one warp's 32 O rows
template <int POLY, bool PIPE>
__global__ void __launch_bounds__(kFwdThreads, 1)
    attn_fwd_ring_tc_kernel(const __grid_constant__ CUtensorMap map_qkv,
                            const __grid_constant__ CUtensorMap map_out, const Params p,
                            int n_heads) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1024(smem_raw);
  const int nt = (p.T + kTile - 1) / kTile;
  const int Tr = nt * kTile;
  const int Tn = (p.T + 15) / 16 * 16;
  const int nb = (Tn + 63) / 64;  // 64-key blocks per query tile
  const size_t buf_bytes = size_t(3 * Tr) * kRowBytes;
  uint8_t* stage_base = smem + 2 * buf_bytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(stage_base + 8 * kStageBytes);
  // per pipeline: operand regions full / empty; per slot SF (S ready), PF (P
  // written), PD (PV done); OF (a tile's O complete)
  // Q tiles, K / V 64-row blocks: full / empty each, so the next head's
  // block j loads as soon as this head's last S / PV of block j is done
  enum { FQ = 0, EQ = 2, FK = 4, EK = 8, FV = 12, EV = 16, SF = 20, PF = SF + kRingSlots,
         PD = PF + kRingSlots, OF = PD + kRingSlots, NB };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2 * NB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int HD = p.H * kD;

  if (threadIdx.x == 0) {
    tma_prefetch(&map_qkv);
    tma_prefetch(&map_out);
    for (int c = 0; c < 2; ++c)
      for (int i = 0; i < NB; ++i) mbar_init(&bar[c * NB + i], (i >= PF && i < PD) ? 4 : 1);
    mbar_fence_init();
  }
  if (warp == 3) tmem_alloc(tmem_slot, 512);
  pdl_launch_dependents();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();

  if (warp == 0 || warp == 3) {
    const int c = warp == 0 ? 0 : 1;
    uint64_t* pb = bar + c * NB;
    uint8_t* base = smem + c * buf_bytes;
    if (lane == 0) {
      int i = 0;
      for (int bh = blockIdx.x; bh < n_heads; bh += gridDim.x, ++i) {
        if ((i & 1) != c) continue;
        const int b = (p.dbg & 1) ? 0 : bh / p.H, h = (p.dbg & 1) ? 0 : bh % p.H;
        const uint32_t par = ((i >> 1) & 1) ^ 1;
        // in release order: Q_0, K blocks, Q_1, V blocks
        for (int t = 0; t < nt; ++t) {
          mbar_wait(&pb[EQ + t], par);
          mbar_expect_tx(&pb[FQ + t], uint32_t(kTile * kRowBytes));
          load_rows(base + t * kTile * kRowBytes, &map_qkv, &pb[FQ + t], h * kD, t * kTile,
                    kTile, b);
          if (t == 0) {
            for (int j = 0; j < nb; ++j) {
              mbar_wait(&pb[EK + j], par);
              mbar_expect_tx(&pb[FK + j], uint32_t(kChunk * kRowBytes));
              tma_load_3d(base + (Tr + j * kChunk) * kRowBytes, &map_qkv, &pb[FK + j],
                          HD + h * kD, j * kChunk, b);
            }
          }
        }
        for (int j = 0; j < nb; ++j) {
          mbar_wait(&pb[EV + j], par);
          mbar_expect_tx(&pb[FV + j], uint32_t(kChunk * kRowBytes));
          tma_load_3d(base + (2 * Tr + j * kChunk) * kRowBytes, &map_qkv, &pb[FV + j],
                      2 * HD + h * kD, j * kChunk, b);
        }
      }
    }
  } else if (warp == 1 || warp == 2) {
    const int c = warp - 1;
    uint64_t* pb = bar + c * NB;
    const uint32_t tO = tmem + uint32_t(256 * c);
    const uint32_t idesc_o = umma_idesc_bf16(128, kD, false, true);
    // this pipeline's heads: bh = blockIdx.x + (2m + c) gridDim.x
    const int first = int(blockIdx.x) + c * int(gridDim.x);
    const int n_my = first < n_heads ? (n_heads - first + 2 * int(gridDim.x) - 1) /
                                           (2 * int(gridDim.x))
                                     : 0;
    const int per_head = nt * nb;
    const int G = n_my * per_head;
    const uint64_t q0 = umma_sdesc(smem_addr(smem + c * buf_bytes), 16, 1024);
    const uint64_t k0 = q0 + uint64_t((Tr * kRowBytes) >> 4);
    const uint64_t v0 = umma_sdesc(smem_addr(smem + c * buf_bytes + 2 * Tr * kRowBytes),
                                   64 * 128, 1024);
    int gs = 0;  // next block whose S is issued
    for (int g = 0; g < G; ++g) {
      const int m = g / per_head;
      // S ahead: at most two blocks past g, and not into head m + 2 (its Q /
      // K load waits for V(m + 1), i.e. for PV(m))
      while (gs < G && gs <= g + kRingSlots - 1 && gs / per_head <= m + 1) {
        const int ms_ = gs / per_head, ts = (gs / nb) % nt, js = gs % nb;
        const int w = min(64, Tn - 64 * js);
        if (js == 0) mbar_wait(&pb[FQ + ts], ms_ & 1);
        if (ts == 0) mbar_wait(&pb[FK + js], ms_ & 1);
        if (!PIPE && gs >= kRingSlots)
          mbar_wait(&pb[PD + gs % kRingSlots], ((gs - kRingSlots) / kRingSlots) & 1);
        tc_fence_after();
        const uint64_t qt = q0 + uint64_t((ts * kTile * kRowBytes) >> 4);
        const uint64_t kj = k0 + uint64_t((js * 64 * kRowBytes) >> 4);
        const uint32_t idesc_s = umma_idesc_bf16(128, w, false, false);
        const uint32_t tS = tO + 64u + uint32_t(64 * (gs % kRingSlots));
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk)
          tc_mma_ss_ws(tS, qt + uint64_t(2 * kk), kj + uint64_t(2 * kk), idesc_s, kk > 0 ? 1u : 0u);
        tc_commit_ws(&pb[SF + gs % kRingSlots]);
        EPS_TRACE(c == 0 && gs < 60 && lane == 0, 832 + gs * 3 + 2);
        if (js == nb - 1) tc_commit_ws(&pb[EQ + ts]);   // Q_t read
        if (ts == nt - 1) tc_commit_ws(&pb[EK + js]);  // K block js read
        ++gs;
      }
      const int t = (g / nb) % nt, j = g % nb;
      const int w = min(64, Tn - 64 * j);
      mbar_wait(&pb[PF + g % kRingSlots], (g / kRingSlots) & 1);
      if (t == 0) mbar_wait(&pb[FV + j], m & 1);
      tc_fence_after();
      const uint32_t tP = tO + 64u + uint32_t(64 * (g % kRingSlots));
      for (int kk = 0; kk < w / 16; ++kk)
        tc_mma_ts_ws(tO, tP + uint32_t(kk * 8), v0 + uint64_t((4 * j + kk) * 128), idesc_o,
                     (j > 0 || kk > 0) ? 1u : 0u);
      tc_commit_ws(&pb[PD + g % kRingSlots]);
      if (t == nt - 1) tc_commit_ws(&pb[EV + j]);  // V block j read by the head's last PV
      if (j == nb - 1) tc_commit_ws(&pb[OF]);
    }
  } else if (warp >= 4) {
    const int c = (warp - 4) >> 2;
    uint64_t* pb = bar + c * NB;
    const int quarter = warp & 3;
    const uint32_t tO = tmem + uint32_t(256 * c) + (uint32_t(quarter * 32) << 16);
    uint8_t* stage = stage_base + (c * 4 + quarter) * kStageBytes;
    const uint32_t stage_s = smem_addr(stage);
    const float sl2 = p.scale_log2;
    const float2 sl2x2 = make_float2(sl2, sl2);
    // previous tile of this pipeline: live warp, 1 / rowsum, TMA coordinates
    bool prev_live = false;
    float prev_inv = 0.f;
    int prev_row = 0, prev_b = 0, prev_col = 0;
    auto emit_o = [&]() {  // O(prev) from TMEM -> smem stage -> TMA store
      uint32_t oa[32], ob[32];
      tmem_ld_32x32(tO, oa);
      tmem_ld_32x32(tO + 32, ob);
      tmem_ld_wait_regs(oa);
      tmem_ld_wait_regs(ob);
      if (lane == 0) bulk_wait_read<0>();  // the stage's previous store has read it
      __syncwarp();
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const uint32_t* s = v < 4 ? &oa[8 * v] : &ob[8 * (v - 4)];
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(s[e]) * prev_inv;
        st_shared_v4(stage_s + uint32_t(lane * kRowBytes + ((v ^ (lane & 7)) << 4)),
                     pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]),
                     pack_bf16(f[6], f[7]));
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(&map_out, stage, prev_col, prev_row, prev_b);
        bulk_commit();
      }
    };
    int g = 0, k = 0;
    for (int bh = blockIdx.x, i = 0; bh < n_heads; bh += gridDim.x, ++i) {
      if ((i & 1) != c) continue;
      const int b = bh / p.H, h = bh % p.H;
      for (int t = 0; t < nt; ++t, ++k) {
        const int row0 = t * kTile + quarter * 32;
        const int q = row0 + lane;
        const bool live = row0 < p.T;  // warp-uniform
        float ms = 0.f;
        float2 sum2 = make_float2(0.f, 0.f);
        for (int j = 0; j < nb; ++j, ++g) {
          const int w = min(64, Tn - 64 * j);
          const uint32_t tS = tO + 64u + uint32_t(64 * (g % kRingSlots));
          mbar_wait(&pb[SF + g % kRingSlots], (g / kRingSlots) & 1);
          tc_fence_after();
          EPS_TRACE(c == 0 && g < 60 && warp == 4 && lane == 0, 832 + g * 3);
          if (live) {
            for (int ch = 0; ch < (w + 31) / 32; ++ch) {
              const int rem = p.T - 64 * j - 32 * ch;  // valid keys in the chunk (>= 1)
              uint32_t ra[32];
              if (rem <= 16)
                tmem_ld_32x32_x16(tS + uint32_t(32 * ch), reinterpret_cast<uint32_t(&)[16]>(ra));
              else
                tmem_ld_32x32(tS + uint32_t(32 * ch), ra);
              tmem_ld_wait_regs(ra);
              uint32_t pk[16];
              auto chunk_exp = [&](float msr) {
                const float2 nms2 = make_float2(-msr, -msr);
                float2 cs = make_float2(0.f, 0.f);
                if (rem >= 32) {
#pragma unroll
                  for (int e = 0; e < 16; ++e) {
                    const float2 a = __ffma2_rn(make_float2(__uint_as_float(ra[2 * e]),
                                                            __uint_as_float(ra[2 * e + 1])),
                                                sl2x2, nms2);
                    const float2 x = fwd_poly_pair<POLY>(e)
                                         ? poly_exp2_x2<true>(a)
                                         : make_float2(fast_exp2(a.x), fast_exp2(a.y));
                    cs = __fadd2_rn(cs, x);
                    pk[e] = pack_bf16(x.x, x.y);
                  }
                } else {
#pragma unroll
                  for (int e = 0; e < 16; ++e) {
                    if (2 * e >= rem) {  // (also the unloaded half of an x16 chunk)
                      pk[e] = 0u;
                      continue;
                    }
                    const float2 a = __ffma2_rn(make_float2(__uint_as_float(ra[2 * e]),
                                                            __uint_as_float(ra[2 * e + 1])),
                                                sl2x2, nms2);
                    const float2 x = make_float2(2 * e < rem ? fast_exp2(a.x) : 0.f,
                                                 2 * e + 1 < rem ? fast_exp2(a.y) : 0.f);
                    cs = __fadd2_rn(cs, x);
                    pk[e] = pack_bf16(x.x, x.y);
                  }
                }
                return cs;
              };
              auto chunk_max = [&]() {
                float m0 = -FLT_MAX, m1 = -FLT_MAX, m2 = -FLT_MAX, m3 = -FLT_MAX;
                if (rem >= 32) {
#pragma unroll
                  for (int e = 0; e < 32; e += 8) {
                    m0 = fmax3f(m0, __uint_as_float(ra[e]), __uint_as_float(ra[e + 1]));
                    m1 = fmax3f(m1, __uint_as_float(ra[e + 2]), __uint_as_float(ra[e + 3]));
                    m2 = fmax3f(m2, __uint_as_float(ra[e + 4]), __uint_as_float(ra[e + 5]));
                    m3 = fmax3f(m3, __uint_as_float(ra[e + 6]), __uint_as_float(ra[e + 7]));
                  }
                } else {
#pragma unroll
                  for (int e = 0; e < 32; ++e)
                    if (e < rem) m0 = fmaxf(m0, __uint_as_float(ra[e]));
                }
                return fmaxf(fmaxf(m0, m1), fmaxf(m2, m3)) * sl2;
              };
              const bool first_chunk = j == 0 && ch == 0;
              if (first_chunk) ms = chunk_max();
              float2 cs = chunk_exp(ms);
              if (!first_chunk) {
                const bool up = cs.x + cs.y > 4294967296.0f;
                if (__any_sync(0xffffffffu, up)) {  // rare: rescale, redo the chunk
                  const float ms_new = up ? fmaxf(ms, chunk_max()) : ms;
                  const float f = fast_exp2(ms - ms_new);  // 1 on lanes without overflow
                  sum2 = __fmul2_rn(sum2, make_float2(f, f));
                  tmem_st_wait();
                  if (ch == 1) {  // this block's first P chunk
                    uint32_t q16[16];
                    tmem_ld_32x32_x16(tS, q16);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                      q16[e] = pack_bf16(bf16_lo(q16[e]) * f, bf16_hi(q16[e]) * f);
                    tmem_st_32x32_x16(tS, q16);
                  }
                  if (j > 0) {  // O = P V of this tile's earlier blocks, once complete
                    const int gp = g - 1;
                    mbar_wait(&pb[PD + gp % kRingSlots], (gp / kRingSlots) & 1);
                    tc_fence_after();
                    for (int hf = 0; hf < 2; ++hf) {
                      uint32_t o32[32];
                      tmem_ld_32x32(tO + uint32_t(hf * 32), o32);
                      tmem_ld_wait_regs(o32);
#pragma unroll
                      for (int e = 0; e < 32; ++e)
                        o32[e] = __float_as_uint(__uint_as_float(o32[e]) * f);
                      tmem_st_32x32_x32(tO + uint32_t(hf * 32), o32);
                    }
                  }
                  ms = ms_new;
                  cs = chunk_exp(ms);
                }
              }
              sum2 = __fadd2_rn(sum2, cs);
              tmem_st_32x32_x16(tS + uint32_t(16 * ch), pk);
            }
          }
          if (j == 0 && k > 0) {  // O(k-1): read out before PV(k, 0) may overwrite it
            mbar_wait(&pb[OF], (k - 1) & 1);
            tc_fence_after();
            if (prev_live) emit_o();
          }
          if (live) tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&pb[PF + g % kRingSlots]);
          EPS_TRACE(c == 0 && g < 60 && warp == 4 && lane == 0, 832 + g * 3 + 1);
        }
        const float sum = sum2.x + sum2.y;
        if (live && q < p.T) p.lse[int64_t(bh) * p.T + q] = (ms + __log2f(sum)) * kLn2;
        prev_live = live;
        prev_inv = 1.f / sum;
        prev_row = row0;
        prev_b = b;
        prev_col = h * kD;
      }
    }
    if (k > 0) {  // the last tile's O
      mbar_wait(&pb[OF], (k - 1) & 1);
      tc_fence_after();
      if (prev_live) emit_o();
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 3) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

size_t fwd_ring_smem(int T) {
  const int Tr = (T + kTile - 1) / kTile * kTile;
  return 2 * size_t(3 * Tr) * kRowBytes + 8 * size_t(kStageBytes) + 1024 + 1024;
}

size_t fwd_smem(int) {
  return size_t(kTile + 2 * kFwdRing * kChunk) * kRowBytes + 1024 + 128;
}
size_t bwd_dq_smem(int) {
  return size_t(2 * kTile + 2 * kBwdRing * kChunk) * kRowBytes + 1024 + 128;
}
size_t bwd_dkdv_smem(int Tp) {
  return size_t(2 * kTile + 2 * kBwdRing * kChunk) * kRowBytes + size_t(2 * Tp) * 4 + 1024 + 128;
}

template <typename K>
bool ensure_smem(K kern, size_t bytes) {
  // the attribute is per kernel; set it once per (host thread, kernel, size)
  thread_local std::unordered_map<const void*, size_t> done;
  const void* key = reinterpret_cast<const void*>(kern);
  auto it = done.find(key);
  if (it != done.end() && it->second >= bytes) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)) !=
      cudaSuccess)
    return false;
  done[key] = bytes;
  return true;
}

}  // namespace attn_tc

// Entry points used by attention.cu's C ABI for head_dim 64, T <= 384.
bool attn_tc_supported(int T, int head_dim) { return head_dim == 64 && T >= 1 && T <= 384; }

static int g_trace_on = 0;

// Pairs of exps per 32-key chunk computed on the FMA pipe in the forward
// (attn_fwd_persistent_tc_kernel<POLY>): 4 of 16 measured best (0.173 ->
// 0.168 ms at ViT-B/16 b400; 6: 0.171, 8: 0.176, 10: 0.182).  EPS_ATTN_POLY=0
// selects the all-SFU variant for A/B runs.
static int fwd_poly_mode() {
  static const int mode = [] {
    const char* e = std::getenv("EPS_ATTN_POLY");
    return e == nullptr ? 4 : std::atoi(e);
  }();
  return mode;
}

// Forward kernel for T <= 256 (EPS_ATTN_FWD, for A/B runs; unset = by T):
// 0 = the round-1 attn_fwd_persistent_tc_kernel, 1 = attn_fwd_ring_tc_kernel,
// 2 = the ring kernel without the in-order tensor-pipe assumption, 3 = the
// persistent kernel's V2 softmax.
static int fwd_kernel_mode() {
  static const int mode = [] {
    const char* e = std::getenv("EPS_ATTN_FWD");
    return e == nullptr ? -1 : std::atoi(e);
  }();
  return mode;
}

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
  p.trace = g_trace_on;
  p.dbg = [] {
    const char* e = std::getenv("EPS_ATTN_DBG");
    return e == nullptr ? 0 : std::atoi(e);
  }();
  if (T <= 2 * kTile) {
    const bool poly = fwd_poly_mode() != 0;
    const int heads = B * H;
    const int grid = heads < sm_count() ? heads : sm_count();
    // default: the ring kernel for T <= 128 (one query tile), the persistent
    // V2 kernel above (measured: ring 0.0162 vs 0.0177 ms at BERT-large-128,
    // persistent V2 faster at ViT-B/16 T = 197)
    const int mode = fwd_kernel_mode() >= 0 ? fwd_kernel_mode() : (T <= kTile ? 1 : 3);
    if (mode == 0 || mode == 3) {
      const size_t sp = fwd_persistent_smem(T);
      auto kern = mode == 0 ? (poly ? attn_fwd_persistent_tc_kernel<4, false>
                                    : attn_fwd_persistent_tc_kernel<0, false>)
                            : (poly ? attn_fwd_persistent_tc_kernel<4, true>
                                    : attn_fwd_persistent_tc_kernel<0, true>);
      if (!ensure_smem(kern, sp)) return EPS_ECUDA;
      count_launch();
      if (launch_k(kern, dim3(grid), dim3(kFwdThreads), sp, st, 1, m, p, heads) != cudaSuccess)
        return EPS_ECUDA;
      return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
    }
    // O rows leave through per-warp 32-row TMA stores (rows >= T clipped)
    CUtensorMap mo;
    if (!make_map_3d(&mo, out, int64_t(H) * kD, T, B, int64_t(H) * kD, int64_t(T) * H * kD, kD,
                     32, CU_TENSOR_MAP_SWIZZLE_128B))
      return EPS_ECUDA;
    const size_t sp = fwd_ring_smem(T);
    auto kern = mode == 2
                    ? (poly ? attn_fwd_ring_tc_kernel<4, false> : attn_fwd_ring_tc_kernel<0, false>)
                    : (poly ? attn_fwd_ring_tc_kernel<4, true> : attn_fwd_ring_tc_kernel<0, true>);
    if (!ensure_smem(kern, sp)) return EPS_ECUDA;
    count_launch();
    if (launch_k(kern, dim3(grid), dim3(kFwdThreads), sp, st, 1, m, mo, p, heads) != cudaSuccess)
      return EPS_ECUDA;
    return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
  }
  const size_t smem = fwd_smem(Tp);
  if (!ensure_smem(attn_fwd_tc_kernel, smem)) return EPS_ECUDA;
  dim3 grid((T + kTile - 1) / kTile, B * H);
  count_launch();
  attn_fwd_tc_kernel<<<grid, kThreads, smem, st>>>(m, p);
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}


// D = rowsum(dO * O) per (row, head) -> drow [rows, H] (one warp per row).
__global__ void attn_rowdot_kernel(const uint16_t* __restrict__ out,
                                   const uint16_t* __restrict__ dout, float* __restrict__ drow,
                                   int64_t rows, int H) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int nv = H * 8;  // 16-byte vectors per row (8 per head)
  const uint4* o4 = reinterpret_cast<const uint4*>(out + row * H * attn_tc::kD);
  const uint4* d4 = reinterpret_cast<const uint4*>(dout + row * H * attn_tc::kD);
  for (int i0 = 0; i0 < nv; i0 += 32) {
    const int i = i0 + lane;
    float s = 0.f;
    if (i < nv) {
      const uint4 a = __ldg(o4 + i), d = __ldg(d4 + i);
      s = bf16_lo(a.x) * bf16_lo(d.x) + bf16_hi(a.x) * bf16_hi(d.x) + bf16_lo(a.y) * bf16_lo(d.y) +
          bf16_hi(a.y) * bf16_hi(d.y) + bf16_lo(a.z) * bf16_lo(d.z) + bf16_hi(a.z) * bf16_hi(d.z) +
          bf16_lo(a.w) * bf16_lo(d.w) + bf16_hi(a.w) * bf16_hi(d.w);
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (i < nv && (lane & 7) == 0) drow[row * H + (i >> 3)] = s;
  }
}


// dQ = sum over the key-tile slices of the UNIT kernel's bf16 partials,
// rounded to bf16 into dqkv's Q columns, plus the Q bias column sums (of the
// rounded values).  A thread owns one 8-column vector of a row; the block
// (192 threads = 2 rows of 96 vectors at HD = 768) strides over rows, so each
// thread's column sums stay in registers until one block reduction.
__global__ void attn_dq_reduce_kernel(const uint16_t* __restrict__ part, int64_t slice, int nslices,
                                      uint16_t* __restrict__ dq, int64_t ld_out, int64_t rows,
                                      int HD, float* __restrict__ dbias) {
  extern __shared__ float red[];  // [blockDim.x / nv][HD]
  const int nv = HD / 8;
  const int v = threadIdx.x % nv, rsub = threadIdx.x / nv, rper = blockDim.x / nv;
  float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int64_t r = int64_t(blockIdx.x) * rper + rsub; r < rows; r += int64_t(gridDim.x) * rper) {
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int s = 0; s < nslices; ++s) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(part + s * slice + r * HD) + v);
      a[0] += bf16_lo(w.x), a[1] += bf16_hi(w.x), a[2] += bf16_lo(w.y), a[3] += bf16_hi(w.y);
      a[4] += bf16_lo(w.z), a[5] += bf16_hi(w.z), a[6] += bf16_lo(w.w), a[7] += bf16_hi(w.w);
    }
    const uint4 o = make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]),
                               pack_bf16(a[6], a[7]));
    *(reinterpret_cast<uint4*>(dq + r * ld_out) + v) = o;
    cs[0] += bf16_lo(o.x), cs[1] += bf16_hi(o.x), cs[2] += bf16_lo(o.y), cs[3] += bf16_hi(o.y);
    cs[4] += bf16_lo(o.z), cs[5] += bf16_hi(o.z), cs[6] += bf16_lo(o.w), cs[7] += bf16_hi(o.w);
  }
  if (dbias == nullptr) return;
#pragma unroll
  for (int i = 0; i < 8; ++i) red[rsub * HD + v * 8 + i] = cs[i];
  __syncthreads();
  for (int c = threadIdx.x; c < HD; c += blockDim.x) {
    float t = 0.f;
    for (int q = 0; q < rper; ++q) t += red[q * HD + c];
    atomicAdd(dbias + c, t);
  }
}

// grow-only device scratch for the UNIT kernel's dQ partials
static void* dq_partial_scratch(size_t bytes) {
  static void* buf = nullptr;
  static size_t have = 0;
  if (bytes > have) {
    if (buf != nullptr) cudaFree(buf);
    buf = nullptr;
    have = 0;
    if (cudaMalloc(&buf, bytes) != cudaSuccess) return nullptr;
    have = bytes;
  }
  return buf;
}

// The fused backward (one kernel; D = rowsum(dO * O) precomputed) covers
// T <= 384: whole heads for T <= 256, (head, key tile) units above.
// EPS_ATTN_BWD=split selects the round-1 two-kernel path for 256 < T <= 384.
static bool bwd_unit_on() {
  static const bool on = [] {
    const char* e = std::getenv("EPS_ATTN_BWD");
    return e == nullptr || std::string(e) != "split";
  }();
  return on;
}

// Paired heads for T <= 128 (EPS_ATTN_BWD_PAIRS=1 enables).  Off by default:
// measured slower at BERT-large-128 b64 (0.0478 -> 0.052 ms): 512 pair units
// on 148 SMs balance worse (3.46 per SM) than 1024 heads (6.92).
static bool bwd_pairs_on() {
  static const bool on = [] {
    const char* e = std::getenv("EPS_ATTN_BWD_PAIRS");
    return e != nullptr && std::atoi(e) != 0;
  }();
  return on;
}

bool attn_bwd_fused_supported(int T, int head_dim) {
  return head_dim == 64 && T >= 1 &&
         T <= (bwd_unit_on() ? 3 * attn_tc::kTile : 2 * attn_tc::kTile);
}

// drow: precomputed D [B*T, H] (fused path) or nullptr (computed here into
// dsum, which then holds it in the same layout).
int attn_bwd_tc(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv,
                float* dbias, float* dsum, const float* drow, int B, int T, int H, float scale,
                cudaStream_t st) {
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
  if (attn_bwd_fused_supported(T, kD)) {
    if (drow == nullptr) {
      const int64_t rows = int64_t(B) * T;
      count_launch();
      attn_rowdot_kernel<<<unsigned((rows + 7) / 8), 256, 0, st>>>(
          static_cast<const uint16_t*>(out), static_cast<const uint16_t*>(dout), dsum, rows, H);
      drow = dsum;
    }
    p.drow = drow;
    p.trace = g_trace_on;
    CUtensorMap mdq;
    if (!make_map_3d(&mdq, dqkv, W, T, B, W, int64_t(T) * W, kD, kChunk, CU_TENSOR_MAP_SWIZZLE_128B))
      return EPS_ECUDA;
    const size_t sf = bwd_fused_smem(T);
    const int heads = B * H;
    if (T > 2 * kTile) {  // (head, key tile) units + the dQ slice reduction
      const int64_t R = int64_t(B) * T;
      uint16_t* part = static_cast<uint16_t*>(dq_partial_scratch(size_t(3 * R * WO) * 2));
      if (part == nullptr) return EPS_ECUDA;
      CUtensorMap mdqp;
      if (!make_map_3d(&mdqp, part, WO, T, 3 * B, WO, int64_t(T) * WO, kD, kChunk,
                       CU_TENSOR_MAP_SWIZZLE_128B))
        return EPS_ECUDA;
      auto kern = attn_bwd_fused_tc_kernel<3, true>;
      if (!ensure_smem(kern, sf)) return EPS_ECUDA;
      const int units = 3 * heads;
      const int grid = units < sm_count() ? units : sm_count();
      count_launch();
      if (launch_k(kern, dim3(grid), dim3(kBwdThreads), sf, st, 1, mq, mo, mdq, mdqp, p, heads) !=
          cudaSuccess)
        return EPS_ECUDA;
      const int threads = int(2 * (WO / 8));  // two rows per block iteration
      count_launch();
      attn_dq_reduce_kernel<<<sm_count() * 2, threads, size_t(2 * WO) * 4, st>>>(
          part, R * WO, 3, static_cast<uint16_t*>(dqkv), W, R, int(WO), dbias);
      return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
    }
    // T <= 128 with an even head count: pairs of heads per work unit (PH)
    const bool ph = T <= kTile && heads % 2 == 0 && bwd_pairs_on();
    const int units = ph ? heads / 2 : heads;
    const int grid = units < sm_count() ? units : sm_count();
    auto kern = ph ? attn_bwd_fused_tc_kernel<2, false, true>
                   : T <= kTile ? attn_bwd_fused_tc_kernel<1> : attn_bwd_fused_tc_kernel<2>;
    const size_t sfk = ph ? bwd_fused_smem(2 * kTile) : sf;
    if (!ensure_smem(kern, sfk)) return EPS_ECUDA;
    count_launch();
    if (launch_k(kern, dim3(grid), dim3(kBwdThreads), sfk, st, 1, mq, mo, mdq, mdq, p, heads) !=
        cudaSuccess)
      return EPS_ECUDA;
    return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
  }
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

extern "C" int eps_attn_trace_enable(int on) {
  eps_k::g_trace_on = on;
  return EPS_OK;
}

extern "C" int eps_attn_trace_read(long long* out, int n) {
  if (n > 1024) n = 1024;
  return cudaMemcpyFromSymbol(out, eps_k::attn_tc::g_attn_trace, size_t(n) * sizeof(long long)) ==
                 cudaSuccess
             ? EPS_OK
             : EPS_ECUDA;
}
