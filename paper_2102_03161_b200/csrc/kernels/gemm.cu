// Persistent, warp-specialised tcgen05 GEMM for the transformer block
// contractions (QKV, out-proj, FC1, FC2 and their dgrad / wgrad).
//
//   C[M,N] = sum_k A(m,k) * B(n,k)      bf16 operands, fp32 accumulation
//
// Operands may be K-major ([rows][K], K contiguous) or MN-major ([K][rows])
// so one kernel covers forward (A=X, B=W, both K-major), dgrad (B=W read
// MN-major) and wgrad (A=dY^T, B=X^T, both MN-major, contraction over the
// token rows) without any transpose copies.
//
// Roles (320 threads, one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: 128B-swizzled A/B k-blocks into a STAGES ring
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..9  epilogue, two warps per TMEM lane quarter taking alternate
//               32-column chunks: tcgen05.ld -> fused bias / GELU / dGELU /
//               residual / column-sum -> swizzled smem -> TMA store (or TMA
//               reduce-add); double-buffered TMEM accumulators so the epilogue
//               of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>

#include "eps_capi.h"
#include "ptx.cuh"
#include "tma_host.cuh"

namespace eps_k {

constexpr int kBM = 128;
constexpr int kBK = 64;  // one 128B swizzle atom of bf16 along K
// Warp roles: EW epilogue warps (8 by default), then the TMA producer and the
// MMA issuer on the two highest warp ids -- the SMSP arbiter favours higher
// warp ids, so the single-warp roles are not starved of issue slots by the
// busy epilogue warps.
constexpr int kMnChunk = 64;  // MN extent of one swizzle atom (MN-major operands)

struct GemmArgs {
  int M, N, K;
  int tiles_m, tiles_n, splits;
  int k_blocks_per_split;
  int epi;
  void* C;
  int64_t ldc;
  const float* bias;
  void* aux;
  float* colsum;
  unsigned long long* prof;  // diagnostics (eps_gemm_prof): wait-cycle counters, else null
};

// EPIB: per-epilogue-warp smem bytes.  4 KB: output staging only (aux inputs
// come through registers); 8 KB: 2 KB output + a 3-deep 2 KB TMA ring for the
// aux input (residual / GELU pre-activation), used with BN = 192 so the
// mainloop ring still keeps 4 stages.
//
// PAIR: a cluster of two CTAs computes one 256 x BN tile with cta_group::2
// MMAs (M = 256): each CTA stages its 128 rows of A and BN/2 rows of B, so a
// stage is 16 KB + BN*64 B per CTA instead of 16 KB + BN*128 B, and the even
// CTA issues the MMAs for both.
template <int BN, int STAGES, bool A_MN, bool B_MN, int EPIB, bool PAIR = false, int EW = 8>
struct GemmCfg {
  static constexpr int kBRows = PAIR ? BN / 2 : BN;  // B rows staged by this CTA
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = kBRows * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // double-buffered accumulator (2 x BN columns), allocation rounded to a power of two
  static constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;
  static constexpr size_t kSmem = size_t(STAGES) * kStageBytes + EW * size_t(EPIB) /*epilogue*/ +
                                  1024 /*align*/ + 1024 /*barriers*/;
  static constexpr uint32_t kIdesc = umma_idesc_bf16(PAIR ? 2 * kBM : kBM, BN, A_MN, B_MN);
};

// Byte offset of the UMMA_K=16 slice kk inside one k-block tile.
template <bool MN>
__device__ __forceinline__ uint32_t k_slice_offset(int kk) {
  return MN ? uint32_t(kk) * 16u * 128u  // 16 K-rows of 128 B
            : uint32_t(kk) * 32u;        // 16 bf16 along the swizzled row
}

template <bool MN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int kk) {
  // K-major: 8-row atoms 1024 B apart (SBO); LBO unused for swizzled K-major.
  // MN-major: 64-wide MN chunks kBK*128 B apart (LBO), 8-K-row groups 1024 B apart (SBO).
  return MN ? umma_sdesc(base + k_slice_offset<true>(kk), kBK * 128, 1024)
            : umma_sdesc(base + k_slice_offset<false>(kk), 16, 1024);
}

template <int BN, bool MN>
__device__ __forceinline__ void load_operand(void* dst, const CUtensorMap* map, uint64_t* bar,
                                             int row0, int k0) {
  if constexpr (MN) {
#pragma unroll
    for (int j = 0; j < BN / kMnChunk; ++j)
      tma_load_2d(static_cast<char*>(dst) + j * (kBK * 128), map, bar, row0 + j * kMnChunk, k0);
  } else {
    tma_load_2d(dst, map, bar, k0, row0);
  }
}

template <int ROWS, bool MN>
__device__ __forceinline__ void load_operand_pair(void* dst, const CUtensorMap* map,
                                                  uint32_t bar_leader, int row0, int k0) {
  if constexpr (MN) {
#pragma unroll
    for (int j = 0; j < ROWS / kMnChunk; ++j)
      tma_load_2d_pair(static_cast<char*>(dst) + j * (kBK * 128), map, bar_leader,
                       row0 + j * kMnChunk, k0);
  } else {
    tma_load_2d_pair(dst, map, bar_leader, k0, row0);
  }
}

// ---- epilogue ----------------------------------------------------------------
// Two warps per TMEM lane quarter (32 output rows) walk alternate 32-column
// chunks of each tile.  Outputs are staged in a per-warp swizzled smem ring
// (EPIB bytes per warp) and written with TMA stores (TMA reduce-add for fp32
// accumulation): coalesced, asynchronous global traffic.  Element-wise inputs
// (residual / gelu' / attention output) arrive through a per-warp TMA ring
// (EPIB >= 8 KB) or, on the 4 KB configurations, straight into registers one
// chunk ahead of use.
constexpr int kChunkBf16 = 2048;  // 32x32 bf16

__device__ __forceinline__ bool epi_reads_aux(int epi) {
  return epi == EPS_EPI_BIAS_RESID_BF16 || epi == EPS_EPI_DGELU_BF16 ||
         epi == EPS_EPI_RESID_BF16 || epi == EPS_EPI_ROWDOT_BF16 || epi == EPS_EPI_MUL_BF16;
}

__device__ __forceinline__ void stage_bf16(uint32_t base, int lane, const float (&v)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q)
    st_shared_v4(base + swz64(lane, q), pack_bf16(v[8 * q + 0], v[8 * q + 1]),
                 pack_bf16(v[8 * q + 2], v[8 * q + 3]), pack_bf16(v[8 * q + 4], v[8 * q + 5]),
                 pack_bf16(v[8 * q + 6], v[8 * q + 7]));
}

// Column sums of a staged 32x32 bf16 chunk (SWIZZLE_64B rows), read back
// column-wise -- cheaper than a register transpose, and it sums exactly the
// stored (rounded) values.
// Lane l sums columns 4(l%8)..+3
// over rows l/8, l/8 + 4, ... (eight 8-byte loads, two wavefronts each), the
// four row groups meet with two shuffle rounds; lanes 0..7 then add their
// float4 to global memory with one vector reduction each (8 per chunk
// instead of 32 scalar atomics -- the bias-gradient targets are shared by
// every CTA on the same column tile, so fewer L2 atomic ops matter).
__device__ __forceinline__ float4 staged_colsum4_bf16(uint32_t base, int lane) {
  const int g = lane & 7, h = lane >> 3;
  const uint32_t q = uint32_t(g >> 1), half_off = uint32_t((g & 1) * 8);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int r = 4 * j + h;
    uint32_t w0, w1;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];"
                 : "=r"(w0), "=r"(w1)
                 : "r"(base + uint32_t(r * 64) + ((q ^ uint32_t((r >> 1) & 3)) << 4) + half_off));
    s.x += bf16_lo(w0);
    s.y += bf16_hi(w0);
    s.z += bf16_lo(w1);
    s.w += bf16_hi(w1);
  }
#pragma unroll
  for (int o = 8; o <= 16; o <<= 1) {
    s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
    s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    s.z += __shfl_xor_sync(0xffffffffu, s.z, o);
    s.w += __shfl_xor_sync(0xffffffffu, s.w, o);
  }
  return s;
}

__device__ __forceinline__ void red_add_v4(float* addr, float4 v) {
  asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}

__device__ __forceinline__ void stage_f32(uint32_t base, int lane, const float (&v)[32]) {
#pragma unroll
  for (int q = 0; q < 8; ++q)
    st_shared_v4(base + swz128(lane, q), __float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                 __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
}

// One row's 32 bf16 aux values (64 B) of chunk `col0`; zero past M / N.
__device__ __forceinline__ void load_aux_row(const uint16_t* aux, int64_t ld, int row, int M,
                                             int col0, int N, uint4 (&dst)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) dst[q] = make_uint4(0u, 0u, 0u, 0u);
  if (row < M) {
    const uint4* src = reinterpret_cast<const uint4*>(aux + int64_t(row) * ld + col0);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (col0 + 8 * q < N) dst[q] = src[q];
  }
}

__device__ __forceinline__ void read_aux_smem(uint32_t base, int lane, float (&a)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 w = ld_shared_v4(base + swz64(lane, q));
    a[8 * q + 0] = bf16_lo(w.x);
    a[8 * q + 1] = bf16_hi(w.x);
    a[8 * q + 2] = bf16_lo(w.y);
    a[8 * q + 3] = bf16_hi(w.y);
    a[8 * q + 4] = bf16_lo(w.z);
    a[8 * q + 5] = bf16_hi(w.z);
    a[8 * q + 6] = bf16_lo(w.w);
    a[8 * q + 7] = bf16_hi(w.w);
  }
}

__device__ __forceinline__ void unpack_aux(const uint4 (&w)[4], float (&a)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    a[8 * q + 0] = bf16_lo(w[q].x);
    a[8 * q + 1] = bf16_hi(w[q].x);
    a[8 * q + 2] = bf16_lo(w[q].y);
    a[8 * q + 3] = bf16_hi(w[q].y);
    a[8 * q + 4] = bf16_lo(w[q].z);
    a[8 * q + 5] = bf16_hi(w[q].z);
    a[8 * q + 6] = bf16_lo(w[q].w);
    a[8 * q + 7] = bf16_hi(w[q].w);
  }
}

constexpr int kAuxDepthMax = 7;  // barrier slots per epilogue warp

std::atomic<int>& gemm_pair_mode();

// EW: epilogue warps (a multiple of 4: EW / 4 warps per TMEM lane quarter,
// taking every (EW / 4)-th 32-column chunk of a tile).
template <int BN, int STAGES, bool A_MN, bool B_MN, int EPIB, bool PAIR, int EW>
__global__ void __launch_bounds__(64 + 32 * EW, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_c,
                   const __grid_constant__ CUtensorMap map_x, const GemmArgs args) {
  using Cfg = GemmCfg<BN, STAGES, A_MN, B_MN, EPIB, PAIR, EW>;
  constexpr int kEpiWarps = EW, kTmaWarp = EW, kMmaWarp = EW + 1;
  constexpr int kParts = EW / 4;  // epilogue warps per TMEM lane quarter
  static_assert(EW % 4 == 0 && kAuxDepthMax * EW * 8 + 256 <= 1024, "epilogue warps");
  // aux TMA ring depth: the per-warp epilogue area minus one 2 KB out slot
  constexpr int kAuxDepth = EPIB >= 8192 ? (EPIB - 2048) / 2048 : 1;
  static_assert(kAuxDepth <= kAuxDepthMax, "aux ring");
  // PAIR: rank 0 / 1 of the CTA pair; work is distributed over pairs.
  const int rank = PAIR ? int(cluster_ctarank()) : 0;
  const bool leader = rank == 0;
  const int cta0 = PAIR ? int(blockIdx.x) >> 1 : int(blockIdx.x);
  const int ncta = PAIR ? int(gridDim.x) >> 1 : int(gridDim.x);
  constexpr int kTileM = PAIR ? 2 * kBM : kBM;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* epi_area = smem + STAGES * Cfg::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_area + kEpiWarps * EPIB);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* aux_full = tmem_empty + 2;  // [kEpiWarps][kAuxDepthMax]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux_full + kAuxDepthMax * kEpiWarps);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  pdl_launch_dependents();

  if (warp == kTmaWarp && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    tma_prefetch(&map_c);
    tma_prefetch(&map_x);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tmem_full[s], 1);
      mbar_init(&tmem_empty[s], PAIR ? 2 * kEpiWarps : kEpiWarps);  // both CTAs' epilogues
    }
    for (int s = 0; s < kAuxDepthMax * kEpiWarps; ++s) mbar_init(&aux_full[s], 1);
    mbar_fence_init();
  }
  if (warp == kMmaWarp) {
    if constexpr (PAIR) tmem_alloc_pair(tmem_slot, Cfg::kTmemCols);
    else tmem_alloc(tmem_slot, Cfg::kTmemCols);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // the peer's barriers are initialised
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_wait();  // the predecessor grid's outputs are complete (PDL launch)

  const int tiles = args.tiles_m * args.tiles_n;
  const int units = tiles * args.splits;
  const int kblocks_total = (args.K + kBK - 1) / kBK;

  // diagnostics: cycles each role spends waiting, summed over CTAs (eps_gemm_prof)
  long long pw_slot = 0, pw_full = 0, pw_empty = 0, pw_tfull = 0, pw_store = 0;
  const long long p_t0 = args.prof ? clock64() : 0;
  if (warp == kTmaWarp) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cta0; u < units; u += ncta) {
        const int split = u / tiles;
        const int t = u - split * tiles;
        const int m0 = (t / args.tiles_n) * kTileM + rank * kBM;
        const int n0 = (t % args.tiles_n) * BN + rank * Cfg::kBRows;
        const int kb0 = split * args.k_blocks_per_split;
        const int kb1 = min(kb0 + args.k_blocks_per_split, kblocks_total);
        for (int kb = kb0; kb < kb1; ++kb) {
          const long long w0 = args.prof ? clock64() : 0;
          mbar_wait(&empty[stage], phase ^ 1);
          if (args.prof) pw_slot += clock64() - w0;
          uint8_t* sa = ring + stage * Cfg::kStageBytes;
          uint8_t* sb = sa + Cfg::kABytes;
          if constexpr (PAIR) {
            // both CTAs' bytes land on the leader's full barrier
            if (leader) mbar_expect_tx(&full[stage], 2 * Cfg::kStageBytes);
            load_operand_pair<kBM, A_MN>(sa, &map_a, leader_addr(&full[stage]), m0, kb * kBK);
            load_operand_pair<Cfg::kBRows, B_MN>(sb, &map_b, leader_addr(&full[stage]), n0,
                                                 kb * kBK);
          } else {
            mbar_expect_tx(&full[stage], Cfg::kStageBytes);
            load_operand<kBM, A_MN>(sa, &map_a, &full[stage], m0, kb * kBK);
            load_operand<BN, B_MN>(sb, &map_b, &full[stage], n0, kb * kBK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0 && leader) {  // PAIR: the even CTA issues for both
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = cta0; u < units; u += ncta) {
        const int split = u / tiles;
        const int kb0 = split * args.k_blocks_per_split;
        const int kb1 = min(kb0 + args.k_blocks_per_split, kblocks_total);
        long long w0 = args.prof ? clock64() : 0;
        mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
        if (args.prof) pw_empty += clock64() - w0;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + uint32_t(acc * BN);
        for (int kb = kb0; kb < kb1; ++kb) {
          if (args.prof) w0 = clock64();
          mbar_wait(&full[stage], phase);
          if (args.prof) pw_full += clock64() - w0;
          tc_fence_after();
          const uint32_t sa = smem_addr(ring + stage * Cfg::kStageBytes);
          const uint32_t sb = sa + Cfg::kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            if constexpr (PAIR)
              tc_mma_pair(d_tmem, operand_desc<A_MN>(sa, kk), operand_desc<B_MN>(sb, kk),
                          Cfg::kIdesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            else
              tc_mma_bf16(d_tmem, operand_desc<A_MN>(sa, kk), operand_desc<B_MN>(sb, kk),
                          Cfg::kIdesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          if constexpr (PAIR) tc_commit_pair(&empty[stage]);
          else tc_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (PAIR) tc_commit_pair(&tmem_full[acc]);
        else tc_commit(&tmem_full[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int ew = warp;             // 0..7
    const int quarter = warp & 3;    // TMEM lane quarter this warp may access
    const int part = ew >> 2;        // this warp takes chunks part, part+kParts, ...
    uint8_t* my_area = epi_area + ew * EPIB;
    const uint32_t area_s = smem_addr(my_area);
    const int epi = args.epi;
    const bool aux_in = epi_reads_aux(epi);
    const bool aux_tma = aux_in && EPIB >= 8192;  // aux through the TMA ring
    const bool f32_out = epi == EPS_EPI_STORE_F32 || epi == EPS_EPI_ACCUM_F32;
    // Per-warp out ring: GELU (2 outputs) and fp32 chunks take 4 KB, bf16 2 KB;
    // with the aux TMA ring: one 2 KB out slot + kAuxDepth 2 KB aux slots.
    const bool two_out = epi == EPS_EPI_BIAS_GELU_BF16 || epi == EPS_EPI_BIAS_GELU2_BF16;
    const int out_bytes = (two_out || f32_out) ? 4096 : 2048;
    const int n_out = aux_tma ? 1 : EPIB / out_bytes;
    const uint16_t* auxp = static_cast<const uint16_t*>(args.aux);
    uint64_t* my_aux_bar = aux_full + kAuxDepthMax * ew;
    const uint32_t aux_s = area_s + kChunkBf16;
    // TMA prefetch cursor over this warp's (tile, chunk) stream: c = part, part+kParts, ...
    // Tile coordinates are decoded once per tile (integer division is a
    // ~20-instruction sequence and lane 0 runs this once per chunk).
    int pf_u = cta0, pf_c = part, pf_row = 0, pf_col = 0, pf_chunks = -1;
    uint32_t pf_n = 0, use_n = 0;
    auto pf_decode = [&]() {
      const int tt = pf_u % tiles;
      const int mt = tt / args.tiles_n, nt = tt - mt * args.tiles_n;
      pf_row = mt * kTileM + rank * kBM + quarter * 32;
      pf_col = nt * BN;
      pf_chunks = min(BN / 32, (args.N - pf_col + 31) / 32);
    };
    auto tma_prefetch_until = [&](uint32_t limit) {
      while (pf_n < limit) {
        if (pf_chunks < 0 && pf_u < units) pf_decode();
        while (pf_u < units && pf_c >= pf_chunks) {
          pf_u += ncta;
          pf_c = part;
          if (pf_u < units) pf_decode();
        }
        if (pf_u >= units) return;
        const uint32_t slot = pf_n % kAuxDepth;
        fence_proxy_async_smem();
        mbar_expect_tx(&my_aux_bar[slot], kChunkBf16);
        tma_load_2d(my_area + kChunkBf16 * (1 + slot), &map_x, &my_aux_bar[slot],
                    pf_col + pf_c * 32, pf_row);
        ++pf_n;
        pf_c += kParts;
      }
    };
    if (aux_tma && lane == 0) tma_prefetch_until(kAuxDepth);

    // Pull a tile's aux rows (this lane's row, this warp's chunks) into L2
    // one tile ahead, so the register loads below hit L2 instead of HBM.
    auto prefetch_aux = [&](int uu) {
      if (!aux_in || aux_tma || uu >= units) return;
      const int tt = uu % tiles;
      const int pn0 = (tt % args.tiles_n) * BN;
      const int prow = (tt / args.tiles_n) * kTileM + rank * kBM + quarter * 32 + lane;
      if (prow >= args.M) return;
      const int pch = min(BN / 32, (args.N - pn0 + 31) / 32);
      for (int c = part; c < pch; c += kParts) prefetch_l2(auxp + int64_t(prow) * args.ldc + pn0 + c * 32);
    };
    prefetch_aux(cta0);

    uint32_t out_n = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = cta0; u < units; u += ncta) {
      const int split = u / tiles;
      const int t = u - split * tiles;
      const int m0 = (t / args.tiles_n) * kTileM + rank * kBM;
      const int n0 = (t % args.tiles_n) * BN;
      const int row0 = m0 + quarter * 32;
      const int my_row = row0 + lane;
      const int chunks = min(BN / 32, (args.N - n0 + 31) / 32);
      prefetch_aux(u + ncta);
      uint4 xa[4];
      if (aux_in && !aux_tma && part < chunks)
        load_aux_row(auxp, args.ldc, my_row, args.M, n0 + part * 32, args.N, xa);
      const long long w0 = args.prof ? clock64() : 0;
      mbar_wait(&tmem_full[acc], acc_phase);
      if (args.prof) pw_tfull += clock64() - w0;
      tc_fence_after();
      const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
#pragma unroll 1
      for (int c = part; c < chunks; c += kParts) {
        const int col0 = n0 + c * 32;
        const int valid = min(32, args.N - col0);
        uint32_t raw[32];
        tmem_ld_32x32(taddr + uint32_t(c * 32), raw);
        uint4 xn[4];
        if (aux_in && !aux_tma && c + kParts < chunks)
          load_aux_row(auxp, args.ldc, my_row, args.M, col0 + 32 * kParts, args.N, xn);
        tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(raw[j]);
        float x[32];
        if (aux_tma) {
          const uint32_t slot = use_n % kAuxDepth;
          mbar_wait(&my_aux_bar[slot], (use_n / kAuxDepth) & 1);
          read_aux_smem(aux_s + slot * kChunkBf16, lane, x);
          ++use_n;
          __syncwarp();  // every lane has read the slot before it is refilled
          if (lane == 0) tma_prefetch_until(use_n + kAuxDepth);
        } else if (aux_in) {
          unpack_aux(xa, x);
        }
        // element-wise work on column pairs (packed fp32 pipe, bit-identical to scalar)
        float2* v2 = reinterpret_cast<float2*>(v);
        float2* x2 = reinterpret_cast<float2*>(x);
        if (args.bias != nullptr) {
          const float4* b4 = reinterpret_cast<const float4*>(args.bias + col0);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 b = (q * 4 < valid) ? __ldg(b4 + q) : make_float4(0.f, 0.f, 0.f, 0.f);
            v2[2 * q] = __fadd2_rn(v2[2 * q], make_float2(b.x, b.y));
            v2[2 * q + 1] = __fadd2_rn(v2[2 * q + 1], make_float2(b.z, b.w));
          }
        }
        // reuse an out slot only after its previous TMA store has read it
        if (lane == 0) {
          const long long w0 = args.prof ? clock64() : 0;
          if (n_out == 1) bulk_wait_read<0>();
          else bulk_wait_read<1>();
          if (args.prof) pw_store += clock64() - w0;
        }
        __syncwarp();
        const uint32_t out_off = (out_n % uint32_t(n_out)) * uint32_t(out_bytes);
        const uint32_t out_s = area_s + out_off;
        switch (epi) {
          case EPS_EPI_BIAS_GELU_BF16:
            stage_bf16(out_s + kChunkBf16, lane, v);  // pre-activation -> map_x
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = gelu_f(v[j]);
            stage_bf16(out_s, lane, v);
            break;
          case EPS_EPI_BIAS_RESID_BF16:
          case EPS_EPI_RESID_BF16:
#pragma unroll
            for (int j = 0; j < 16; ++j) v2[j] = __fadd2_rn(v2[j], x2[j]);
            stage_bf16(out_s, lane, v);
            break;
          case EPS_EPI_BIAS_GELU2_BF16:
#pragma unroll
            for (int j = 0; j < 16; ++j) gelu_and_grad_f2(v2[j], v2[j], x2[j]);
            stage_bf16(out_s + kChunkBf16, lane, x);  // gelu' -> map_x
            stage_bf16(out_s, lane, v);
            break;
          case EPS_EPI_DGELU_BF16:
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] *= gelu_grad_f(x[j]);
            stage_bf16(out_s, lane, v);  // bias-gradient sums read the staged values back
            break;
          case EPS_EPI_MUL_BF16:
#pragma unroll
            for (int j = 0; j < 16; ++j) v2[j] = __fmul2_rn(v2[j], x2[j]);
            stage_bf16(out_s, lane, v);
            break;
          case EPS_EPI_ROWDOT_BF16: {
            // this lane's row: partial dot of the stored (bf16) values with
            // aux over the chunk's 32 columns; the two chunks of a 64-column
            // group come from the two warps of this lane quarter
            float dot = 0.f;
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              pk[j] = pack_bf16(v[2 * j], v[2 * j + 1]);
              dot = fmaf(bf16_lo(pk[j]), x[2 * j], dot);
              dot = fmaf(bf16_hi(pk[j]), x[2 * j + 1], dot);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
              st_shared_v4(out_s + swz64(lane, q), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2],
                           pk[4 * q + 3]);
            if (my_row < args.M)
              atomicAdd(args.colsum + int64_t(my_row) * (args.N >> 6) + (col0 >> 6), dot);
            break;
          }
          default:
            if (f32_out) stage_f32(out_s, lane, v);
            else stage_bf16(out_s, lane, v);
            break;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (epi == EPS_EPI_ACCUM_F32) {
            tma_reduce_add_2d(&map_c, my_area + out_off, col0, row0);
          } else {
            tma_store_2d(&map_c, my_area + out_off, col0, row0);
            if (two_out) tma_store_2d(&map_x, my_area + out_off + kChunkBf16, col0, row0);
          }
          bulk_commit();
        }
        ++out_n;
        if ((epi == EPS_EPI_DGELU_BF16 || epi == EPS_EPI_MUL_BF16) && args.colsum != nullptr) {
          // rows past M were zero-filled by TMA (and aux zeroed), so they contribute 0
          const float4 cs = staged_colsum4_bf16(out_s, lane);
          if (lane < 8) {
            float* dst = args.colsum + col0 + 4 * lane;
            if (4 * lane + 3 < valid) {
              red_add_v4(dst, cs);
            } else {
              if (4 * lane < valid) atomicAdd(dst, cs.x);
              if (4 * lane + 1 < valid) atomicAdd(dst + 1, cs.y);
              if (4 * lane + 2 < valid) atomicAdd(dst + 2, cs.z);
            }
          }
        }
        if (aux_in && !aux_tma) {
#pragma unroll
          for (int q = 0; q < 4; ++q) xa[q] = xn[q];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_remote(&tmem_empty[acc], 0u);
        else mbar_arrive(&tmem_empty[acc]);
      }
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait<0>();
  }

  if (args.prof != nullptr && lane == 0) {
    // [0] span of the MMA warp, [1] its tmem_empty waits, [2] its full waits,
    // [3] producer slot waits, [4] epilogue warp 0 tmem_full waits, [5] its
    // store-slot waits, [6] epilogue warp 0 span
    const long long span = clock64() - p_t0;
    if (warp == kMmaWarp && (!PAIR || leader)) {
      atomicAdd(args.prof + 0, (unsigned long long)span);
      atomicAdd(args.prof + 1, (unsigned long long)pw_empty);
      atomicAdd(args.prof + 2, (unsigned long long)pw_full);
    } else if (warp == kTmaWarp && (!PAIR || leader)) {
      atomicAdd(args.prof + 3, (unsigned long long)pw_slot);
    } else if (warp == 0 && (!PAIR || leader)) {
      atomicAdd(args.prof + 4, (unsigned long long)pw_tfull);
      atomicAdd(args.prof + 5, (unsigned long long)pw_store);
      atomicAdd(args.prof + 6, (unsigned long long)span);
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // no remote traffic targets an exited CTA
  if (warp == kMmaWarp) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem_base, Cfg::kTmemCols);
    else tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

// ---- host side -------------------------------------------------------------

template <int BN, int STAGES, bool A_MN, bool B_MN, int EPIB = 4096, bool PAIR = false,
          int EW = 8>
int launch(const void* A, const void* B, int64_t lda, int64_t ldb, GemmArgs args,
           cudaStream_t stream) {
  using Cfg = GemmCfg<BN, STAGES, A_MN, B_MN, EPIB, PAIR, EW>;
  auto kern = gemm_tc_kernel<BN, STAGES, A_MN, B_MN, EPIB, PAIR, EW>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(Cfg::kSmem)) != cudaSuccess)
      return EPS_ECUDA;
    configured = true;
  }
  CUtensorMap ma, mb, mc, mx;
  const auto SW128 = CU_TENSOR_MAP_SWIZZLE_128B;
  const auto SW64 = CU_TENSOR_MAP_SWIZZLE_64B;
  // A(m,k): K-major -> [M][K]; MN-major -> [K][M].  Likewise B(n,k).
  const bool ok_a = A_MN ? make_map(&ma, A, false, args.M, args.K, lda, 64, kBK, SW128)
                         : make_map(&ma, A, false, args.K, args.M, lda, 64, kBM, SW128);
  const bool ok_b = B_MN ? make_map(&mb, B, false, args.N, args.K, ldb, 64, kBK, SW128)
                         : make_map(&mb, B, false, args.K, args.N, ldb, 64, Cfg::kBRows, SW128);
  const bool f32 = args.epi == EPS_EPI_STORE_F32 || args.epi == EPS_EPI_ACCUM_F32;
  const bool ok_c = make_map(&mc, args.C, f32, args.N, args.M, args.ldc, 32, 32, f32 ? SW128 : SW64);
  // aux: GELU pre-activation output (TMA store); residual / pre-activation
  // inputs are read with plain loads.
  const void* xptr = args.aux != nullptr ? args.aux : args.C;
  const bool ok_x = make_map(&mx, xptr, false, args.N, args.M, args.ldc, 32, 32, SW64);
  if (!ok_a || !ok_b || !ok_c || !ok_x) return EPS_ECUDA;
  const int units = args.tiles_m * args.tiles_n * args.splits;
  const int workers = PAIR ? sm_count() / 2 : sm_count();
  const int grid = (units < workers ? units : workers) * (PAIR ? 2 : 1);
  count_launch();
  if (launch_k(kern, dim3(grid), dim3(64 + 32 * EW), Cfg::kSmem, stream, PAIR ? 2 : 1, ma, mb, mc, mx,
               args) != cudaSuccess)
    return EPS_ECUDA;
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

// CTA-pair tiles on (1, default; EPS_GEMM_PAIR=0 in the environment or
// eps_gemm_pair_mode(0) turns them off for A/B comparisons).
// Diagnostics: a device buffer of 7 u64 wait-cycle counters every GEMM launch
// adds to (eps_gemm_prof; null = off, the default).
std::atomic<unsigned long long*>& gemm_prof_buf() {
  static std::atomic<unsigned long long*> buf{nullptr};
  return buf;
}

// Epilogue warps of the pair-tile aux / two-output GEMMs forced by
// EPS_GEMM_EW (8 or 12; 0 = per-epilogue default).
int gemm_epi_warps() {
  static const int ew = [] {
    const char* e = std::getenv("EPS_GEMM_EW");
    return e == nullptr ? 0 : std::atoi(e);
  }();
  return ew;
}

// Utilisation-based tile width for M < 4096 (1, default; EPS_GEMM_SMALL=0
// keeps the fixed choice, for A/B runs).
bool gemm_small_tiles() {
  static const bool on = [] {
    const char* e = std::getenv("EPS_GEMM_SMALL");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

std::atomic<int>& gemm_pair_mode() {
  static std::atomic<int> mode{[] {
    const char* e = std::getenv("EPS_GEMM_PAIR");
    return e == nullptr ? 1 : std::atoi(e);
  }()};
  return mode;
}

}  // namespace eps_k

extern "C" int eps_pdl_mode(int mode) {
  if (mode >= 0) eps_k::pdl_mode().store(mode);
  return eps_k::pdl_mode().load();
}

extern "C" int eps_gemm_prof(void* counters) {
  eps_k::gemm_prof_buf().store(static_cast<unsigned long long*>(counters));
  return EPS_OK;
}

extern "C" int eps_gemm_pair_mode(int mode) {
  if (mode >= 0) eps_k::gemm_pair_mode().store(mode);
  return eps_k::gemm_pair_mode().load();
}

extern "C" int eps_gemm_bf16(int a_mn_major, int b_mn_major, int epilogue, const void* A,
                             const void* B, void* C, const float* bias, void* aux,
                             float* colsum, int64_t M, int64_t N, int64_t K, int64_t lda,
                             int64_t ldb, int64_t ldc, int split_k, void* stream) {
  using namespace eps_k;
  if (M <= 0 || N <= 0 || K <= 0 || N % 8 != 0 || lda % 8 != 0 || ldb % 8 != 0 ||
      ldc % 8 != 0 || M > (int64_t(1) << 31) || epilogue < 0 || epilogue > EPS_EPI_MUL_BF16)
    return EPS_EINVAL;
  if (epilogue == EPS_EPI_ROWDOT_BF16 && (N % 64 != 0 || colsum == nullptr)) return EPS_EINVAL;
  const bool auto_split = split_k == 0 && epilogue == EPS_EPI_ACCUM_F32;
  if (split_k < 1) split_k = 1;
  const bool needs_aux = epilogue == EPS_EPI_BIAS_GELU_BF16 || epilogue == EPS_EPI_BIAS_RESID_BF16 ||
                         epilogue == EPS_EPI_BIAS_GELU2_BF16 || epilogue == EPS_EPI_MUL_BF16 ||
                         epilogue == EPS_EPI_DGELU_BF16 || epilogue == EPS_EPI_RESID_BF16 ||
                         epilogue == EPS_EPI_ROWDOT_BF16;
  if (needs_aux && aux == nullptr) return EPS_EINVAL;
  if ((epilogue == EPS_EPI_BIAS_BF16 || epilogue == EPS_EPI_BIAS_GELU_BF16 ||
       epilogue == EPS_EPI_BIAS_GELU2_BF16 ||
       epilogue == EPS_EPI_BIAS_RESID_BF16) && bias == nullptr)
    return EPS_EINVAL;
  if (split_k > 1 && epilogue != EPS_EPI_ACCUM_F32) return EPS_EINVAL;
  GemmArgs args{};
  args.M = int(M);
  args.N = int(N);
  args.K = int(K);
  args.epi = epilogue;
  args.C = C;
  args.ldc = ldc;
  args.bias = (epilogue == EPS_EPI_BIAS_BF16 || epilogue == EPS_EPI_BIAS_GELU_BF16 ||
               epilogue == EPS_EPI_BIAS_GELU2_BF16 ||
               epilogue == EPS_EPI_BIAS_RESID_BF16) ? bias : nullptr;
  args.aux = aux;
  args.colsum = colsum;
  args.prof = gemm_prof_buf().load();
  const int kblocks = int((K + kBK - 1) / kBK);
  // CTA pairs (256-row tiles, cta_group::2) for every GEMM with enough rows
  // and a 256-multiple N (all ViT-B / BERT block GEMMs at full batch);
  // EPS_GEMM_PAIR=0 forces single-CTA tiles (A/B comparisons).
  // Below ~4K rows without a K split (a pipeline micro-batch of <= 20 ViT
  // samples) single CTAs balance the few tiles better (measured at 17 and 34
  // samples); weight gradients (split-K over the token rows) always have
  // enough units.
  const bool pair = gemm_pair_mode() != 0 && N % 256 == 0 &&
                    (M >= 4096 || (auto_split && M >= 512));
  const int64_t tile_m = pair ? 2 * kBM : kBM;
  if (auto_split) {
    // wgrad: few output tiles, long contraction over token rows.  Pick the
    // split s minimising waves(s) * (k-blocks per split + 7): a unit's fixed
    // cost (fill, drain, fp32 tile reduce-add) is ~7 k-blocks of MMA (fit of
    // BERT-large-128 FC weight gradients, 64 pair tiles x 128 k-blocks, split
    // 1..8: 0.0519 / 0.053 / 0.0572 / 0.0604 ms; the former "+ 1" picked 8).
    // Each split keeps >= 4 k-blocks.
    const int64_t tiles = ((M + tile_m - 1) / tile_m) * ((N + 255) / 256);
    const int64_t sms = pair ? sm_count() / 2 : sm_count();  // concurrent tile workers
    const int cap = std::max(1, std::min(16, kblocks / 4));
    double best = 1e30;
    for (int sk = 1; sk <= cap; ++sk) {
      const double waves = double((tiles * sk + sms - 1) / sms);
      const double cost = waves * (double(kblocks) / sk + 7.0);
      if (cost < best - 1e-12) {
        best = cost;
        split_k = sk;
      }
    }
  }
  if (split_k > kblocks) split_k = kblocks;
  args.k_blocks_per_split = (kblocks + split_k - 1) / split_k;
  args.splits = (kblocks + args.k_blocks_per_split - 1) / args.k_blocks_per_split;
  args.tiles_m = int((M + tile_m - 1) / tile_m);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int key = (a_mn_major ? 2 : 0) | (b_mn_major ? 1 : 0);
  const bool aux_or_two = epilogue == EPS_EPI_BIAS_RESID_BF16 || epilogue == EPS_EPI_DGELU_BF16 ||
                          epilogue == EPS_EPI_RESID_BF16 || epilogue == EPS_EPI_ROWDOT_BF16 ||
                          epilogue == EPS_EPI_MUL_BF16 || epilogue == EPS_EPI_BIAS_GELU2_BF16;
  if (pair) {
    // 256 x 256 pair tiles; a CTA stages 32 KB per k-block, so 6 stages fit
    // beside the 4 KB-per-warp epilogue staging, or 5 beside the 8 KB aux ring.
    args.tiles_n = int(N / 256);
    if (aux_or_two) {
      // The GELU + GELU' (FC1 forward) and gelu'-product + column-sum (FC2
      // dgrad) epilogues are issue-latency bound: 12 epilogue warps (3 per
      // TMEM lane quarter) with 4 operand stages beat 8 warps with 5 stages
      // (ViT-B b400: 0.381 -> 0.363 ms, 0.352 -> 0.340 ms); the residual /
      // row-dot epilogues and K = 3072 mainloops prefer the fifth stage
      // (+2..7 % with 12 warps).  EPS_GEMM_EW = 8 / 12 forces either.
      const int ew = gemm_epi_warps() != 0 ? gemm_epi_warps()
                     : (epilogue == EPS_EPI_BIAS_GELU2_BF16 || epilogue == EPS_EPI_MUL_BF16) ? 12
                                                                                             : 8;
      if (ew == 12) {
        switch (key) {
          case 0: return launch<256, 4, false, false, 8192, true, 12>(A, B, lda, ldb, args, st);
          case 1: return launch<256, 4, false, true, 8192, true, 12>(A, B, lda, ldb, args, st);
          case 2: return launch<256, 4, true, false, 8192, true, 12>(A, B, lda, ldb, args, st);
          default: return launch<256, 4, true, true, 8192, true, 12>(A, B, lda, ldb, args, st);
        }
      }
      switch (key) {
        case 0: return launch<256, 5, false, false, 8192, true>(A, B, lda, ldb, args, st);
        case 1: return launch<256, 5, false, true, 8192, true>(A, B, lda, ldb, args, st);
        case 2: return launch<256, 5, true, false, 8192, true>(A, B, lda, ldb, args, st);
        default: return launch<256, 5, true, true, 8192, true>(A, B, lda, ldb, args, st);
      }
    }
    switch (key) {
      case 0: return launch<256, 6, false, false, 4096, true>(A, B, lda, ldb, args, st);
      case 1: return launch<256, 6, false, true, 4096, true>(A, B, lda, ldb, args, st);
      case 2: return launch<256, 6, true, false, 4096, true>(A, B, lda, ldb, args, st);
      default: return launch<256, 6, true, true, 4096, true>(A, B, lda, ldb, args, st);
    }
  }
  // Epilogues that read an aux input (residual, GELU pre-activation) are
  // latency-bound on it: BN = 192 tiles free smem for a 3-deep TMA aux ring.
  const bool aux_epi = epilogue == EPS_EPI_BIAS_RESID_BF16 || epilogue == EPS_EPI_DGELU_BF16 ||
                       epilogue == EPS_EPI_RESID_BF16 || epilogue == EPS_EPI_ROWDOT_BF16 ||
                       epilogue == EPS_EPI_MUL_BF16;
  const bool ring_epi = aux_epi || epilogue == EPS_EPI_BIAS_GELU2_BF16;
  // Few tiles (M < 4096 rows: a K = 8 pipeline micro-batch of <= 20 ViT
  // samples; single-CTA tiles): pick the tile width that keeps the most SMs
  // busy over whole waves -- e.g. M = 3546, N = 768: 256-wide tiles give 84
  // tiles (57 % of the SMs), 192-wide 112 (76 %): FC1 / QKV dgrad at b18
  // 0.0211 -> 0.0195 ms, 0.0173 -> 0.0161 ms.
  int bn_small = 0;
  if (split_k == 1 && M < 4096 && gemm_small_tiles()) {
    const int64_t tm = (M + kBM - 1) / kBM;
    const int64_t sms = sm_count();
    double best = -1.0;
    for (int bn : {256, 192, 128}) {
      if (ring_epi && bn == 256) continue;  // the aux ring needs the 192 / 128 smem layout
      if (N < bn && bn != 128) continue;
      const int64_t tiles = tm * ((N + bn - 1) / bn);
      const int64_t waves = (tiles + sms - 1) / sms;
      // useful columns per wave slot (the last tile column may be partial),
      // times the MMA efficiency of the width: a single-CTA M = 128, K = 16
      // MMA never takes fewer than ~89 cycles (tools/mma_rate.cu), i.e. 72 %
      // of the math rate at N = 128 (measured: 128-wide GELU2 / MUL tiles at
      // b18 lose to 192-wide despite 91 % vs 76 % wave utilisation)
      const double eff = std::min(1.0, (bn / 2.0) / 89.0);
      const double util =
          eff * double(M) * double(N) / (double(waves * sms) * double(kBM) * bn);
      if (util > best + 0.02) {
        best = util;
        bn_small = bn;
      }
    }
  }
  if (bn_small == 128 && ring_epi) {
    args.tiles_n = int((N + 127) / 128);
    switch (key) {
      case 0: return launch<128, 4, false, false, 8192>(A, B, lda, ldb, args, st);
      case 1: return launch<128, 4, false, true, 8192>(A, B, lda, ldb, args, st);
      case 2: return launch<128, 4, true, false, 8192>(A, B, lda, ldb, args, st);
      default: return launch<128, 4, true, true, 8192>(A, B, lda, ldb, args, st);
    }
  }
  // Two-output GELU forward: BN = 192 leaves 8 KB per epilogue warp, i.e. two
  // 4 KB (gelu, gelu') staging slots, so a chunk's stores drain while the
  // next chunk is computed.
  if ((ring_epi && N >= 192) || bn_small == 192) {
    args.tiles_n = int((N + 191) / 192);
    switch (key) {
      case 0: return launch<192, 4, false, false, 8192>(A, B, lda, ldb, args, st);
      case 1: return launch<192, 4, false, true, 8192>(A, B, lda, ldb, args, st);
      case 2: return launch<192, 4, true, false, 8192>(A, B, lda, ldb, args, st);
      default: return launch<192, 4, true, true, 8192>(A, B, lda, ldb, args, st);
    }
  }
  // BN = 256 when N fills it; 128 otherwise (fewer wasted MMA columns).
  const bool wide = bn_small != 0 ? bn_small == 256 : (N % 256 == 0 || N >= 1024);
  const int bn = wide ? 256 : 128;
  args.tiles_n = int((N + bn - 1) / bn);
  if (wide) {
    switch (key) {
      case 0: return launch<256, 4, false, false>(A, B, lda, ldb, args, st);
      case 1: return launch<256, 4, false, true>(A, B, lda, ldb, args, st);
      case 2: return launch<256, 4, true, false>(A, B, lda, ldb, args, st);
      default: return launch<256, 4, true, true>(A, B, lda, ldb, args, st);
    }
  }
  switch (key) {
    case 0: return launch<128, 6, false, false>(A, B, lda, ldb, args, st);
    case 1: return launch<128, 6, false, true>(A, B, lda, ldb, args, st);
    case 2: return launch<128, 6, true, false>(A, B, lda, ldb, args, st);
    default: return launch<128, 6, true, true>(A, B, lda, ldb, args, st);
  }
}
