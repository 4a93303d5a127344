// Multi-head self-attention over a packed QKV activation, forward and
// backward, bf16 tensor-core MMA (m16n8k16, fp32 accumulate) with the
// softmax kept on chip (flash-attention style: the [T,T] score matrix is
// never written to HBM; the forward stores only the row log-sum-exp).
//
// Layout: qkv [B*T, 3*H*dh]: columns [0,Hdh) = Q, [Hdh,2Hdh) = K,
// [2Hdh,3Hdh) = V, head h at h*dh within each; out [B*T, H*dh].
// T is arbitrary (197, 65, 128, 384 ...): rows past T are zero-filled in
// smem and masked out of the softmax.
//
// Backward = D pre-pass (rowsum(dO * O)) + a dK/dV kernel (key-block
// outer loop, recomputes P^T) + a dQ kernel (query-block outer loop), so no
// atomics are needed on dQ/dK/dV.  Both also emit the column sums of their
// dq / dk / dv slices = the QKV bias gradient.
#include <cuda_runtime.h>

#include <cfloat>

#include "eps_capi.h"
#include "ptx.cuh"

namespace eps_k {

constexpr int kAttWarps = 4;  // 4 warps x 16 rows = 64-row blocks
constexpr int kBlk = 64;

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %2, 0;\n"
      " @p cp.async.cg.shared.global [%0], [%1], 16;\n"
      " @!p st.shared.v4.b32 [%0], {0, 0, 0, 0};\n}\n" ::"r"(dst),
      "l"(src), "r"(int(pred)));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Smem tile of `rows` x DH bf16 with a padded pitch (DH + 8) so ldmatrix row
// addresses fall in distinct banks.
template <int DH>
struct Tile {
  static constexpr int kPitch = DH + 8;
  static constexpr int kBytesPerRow = kPitch * 2;
};

// Copy rows [r0, r0+rows) of one head slice (column offset col, row pitch
// ld elements) into smem, zero-filling rows >= T.
template <int DH>
__device__ __forceinline__ void load_tile(uint32_t smem, const uint16_t* base, int64_t ld,
                                          int col, int r0, int rows, int T) {
  constexpr int kVec = DH / 8;  // 16B vectors per row
  for (int i = threadIdx.x; i < rows * kVec; i += blockDim.x) {
    const int r = i / kVec, v = i % kVec;
    const bool ok = r0 + r < T;
    const uint16_t* src = base + int64_t(ok ? r0 + r : 0) * ld + col + v * 8;
    cp_async16(smem + uint32_t(r * Tile<DH>::kBytesPerRow + v * 16), src, ok);
  }
}

// A operand (16 rows x 16 k) at (row0, k0) of a padded tile.
template <int DH>
__device__ __forceinline__ void lda_frag(uint32_t tile, int row0, int k0, uint32_t (&a)[4]) {
  const int lane = threadIdx.x & 31;
  ldsm_x4(tile + uint32_t((row0 + (lane & 15)) * Tile<DH>::kBytesPerRow + (k0 + 8 * (lane >> 4)) * 2), a);
}
// B operand pair for S = X Y^T: Y stored [n][k]; returns b-frags for n-tile
// (n0..n0+7) and k-steps k0, k0+16: r[0],r[1] = step k0; r[2],r[3] = step k0+16.
template <int DH>
__device__ __forceinline__ void ldb_nk(uint32_t tile, int n0, int k0, uint32_t (&r)[4]) {
  const int lane = threadIdx.x & 31;
  ldsm_x4(tile + uint32_t((n0 + (lane & 7)) * Tile<DH>::kBytesPerRow + (k0 + 8 * (lane >> 3)) * 2), r);
}
// B operand for O = P V: V stored [k][n]; returns b-frags for k-step k0
// (16 rows) and n-tiles n0, n0+8: r[0],r[1] -> n0; r[2],r[3] -> n0+8.
template <int DH>
__device__ __forceinline__ void ldb_kn(uint32_t tile, int k0, int n0, uint32_t (&r)[4]) {
  const int lane = threadIdx.x & 31;
  ldsm_x4_t(tile + uint32_t((k0 + (lane & 7) + 8 * ((lane >> 3) & 1)) * Tile<DH>::kBytesPerRow +
                            (n0 + 8 * (lane >> 4)) * 2),
            r);
}

// ---------------------------------------------------------------------------
// Forward: grid (B*H, ceil(T/64)); each warp owns 16 query rows and streams
// 64-key blocks with an online softmax.
template <int DH>
__global__ void __launch_bounds__(kAttWarps * 32)
    attn_fwd_kernel(const uint16_t* __restrict__ qkv, uint16_t* __restrict__ out,
                    float* __restrict__ lse, int T, int H, float scale_log2) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int q0 = blockIdx.y * kBlk;
  const int64_t ld = int64_t(3) * H * DH;
  const uint16_t* base = qkv + int64_t(b) * T * ld;
  const int Tp = (T + kBlk - 1) / kBlk * kBlk;
  const uint32_t sQ = smem_addr(sm);
  const uint32_t sK = sQ + kBlk * Tile<DH>::kBytesPerRow;
  const uint32_t sV = sK + Tp * Tile<DH>::kBytesPerRow;
  load_tile<DH>(sQ, base, ld, h * DH, q0, kBlk, T);
  load_tile<DH>(sK, base, ld, H * DH + h * DH, 0, Tp, T);
  load_tile<DH>(sV, base, ld, 2 * H * DH + h * DH, 0, Tp, T);
  cp_async_wait_all();
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int r0 = warp * 16;
  uint32_t qa[DH / 16][4];
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) lda_frag<DH>(sQ, r0, kk * 16, qa[kk]);

  float o[DH / 8][4];
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_lo = -FLT_MAX, m_hi = -FLT_MAX, l_lo = 0.f, l_hi = 0.f;

  for (int kb = 0; kb < Tp; kb += kBlk) {
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; kk += 2) {
        uint32_t bf[4];
        ldb_nk<DH>(sK, kb + j * 8, kk * 16, bf);
        mma16816(s[j], qa[kk], bf[0], bf[1]);
        if (kk + 1 < DH / 16) mma16816(s[j], qa[kk + 1], bf[2], bf[3]);
      }
    }
    // scale into log2 domain, mask keys >= T, online softmax
    float mx_lo = m_lo, mx_hi = m_hi;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int key = kb + j * 8 + 2 * t4;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool ok = key + (e & 1) < T;
        s[j][e] = ok ? s[j][e] * scale_log2 : -FLT_MAX;
      }
      mx_lo = fmaxf(mx_lo, fmaxf(s[j][0], s[j][1]));
      mx_hi = fmaxf(mx_hi, fmaxf(s[j][2], s[j][3]));
    }
#pragma unroll
    for (int o2 = 1; o2 <= 2; o2 <<= 1) {
      mx_lo = fmaxf(mx_lo, __shfl_xor_sync(0xffffffffu, mx_lo, o2));
      mx_hi = fmaxf(mx_hi, __shfl_xor_sync(0xffffffffu, mx_hi, o2));
    }
    const float c_lo = exp2f(m_lo - mx_lo), c_hi = exp2f(m_hi - mx_hi);
    m_lo = mx_lo;
    m_hi = mx_hi;
    float sum_lo = 0.f, sum_hi = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      s[j][0] = exp2f(s[j][0] - m_lo);
      s[j][1] = exp2f(s[j][1] - m_lo);
      s[j][2] = exp2f(s[j][2] - m_hi);
      s[j][3] = exp2f(s[j][3] - m_hi);
      sum_lo += s[j][0] + s[j][1];
      sum_hi += s[j][2] + s[j][3];
    }
    l_lo = l_lo * c_lo + sum_lo;
    l_hi = l_hi * c_hi + sum_hi;
#pragma unroll
    for (int j = 0; j < DH / 8; ++j) {
      o[j][0] *= c_lo;
      o[j][1] *= c_lo;
      o[j][2] *= c_hi;
      o[j][3] *= c_hi;
    }
    // O += P V ; P from registers (C layout of n-tiles 2i, 2i+1 == A layout)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t pa[4];
      pa[0] = pack_bf16(s[2 * i][0], s[2 * i][1]);
      pa[1] = pack_bf16(s[2 * i][2], s[2 * i][3]);
      pa[2] = pack_bf16(s[2 * i + 1][0], s[2 * i + 1][1]);
      pa[3] = pack_bf16(s[2 * i + 1][2], s[2 * i + 1][3]);
#pragma unroll
      for (int j = 0; j < DH / 8; j += 2) {
        uint32_t bf[4];
        ldb_kn<DH>(sV, kb + i * 16, j * 8, bf);
        mma16816(o[j], pa, bf[0], bf[1]);
        mma16816(o[j + 1], pa, bf[2], bf[3]);
      }
    }
  }
#pragma unroll
  for (int o2 = 1; o2 <= 2; o2 <<= 1) {
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, o2);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, o2);
  }
  const float inv_lo = 1.f / l_lo, inv_hi = 1.f / l_hi;
  const int row_lo = q0 + r0 + g, row_hi = row_lo + 8;
  const int64_t ldo = int64_t(H) * DH;
  uint16_t* ob = out + int64_t(b) * T * ldo + h * DH;
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) {
    const int col = j * 8 + 2 * t4;
    if (row_lo < T)
      *reinterpret_cast<uint32_t*>(ob + int64_t(row_lo) * ldo + col) =
          pack_bf16(o[j][0] * inv_lo, o[j][1] * inv_lo);
    if (row_hi < T)
      *reinterpret_cast<uint32_t*>(ob + int64_t(row_hi) * ldo + col) =
          pack_bf16(o[j][2] * inv_hi, o[j][3] * inv_hi);
  }
  if (t4 == 0) {
    // natural-log LSE of the scaled scores
    float* lb = lse + int64_t(bh) * T;
    if (row_lo < T) lb[row_lo] = (m_lo + __log2f(l_lo)) * 0.69314718055994531f;
    if (row_hi < T) lb[row_hi] = (m_hi + __log2f(l_hi)) * 0.69314718055994531f;
  }
}

// D[b,h,t] = sum_d dO[b,t,h,d] * O[b,t,h,d]   (one warp per (row, head))
template <int DH>
__global__ void attn_bwd_dot_kernel(const uint16_t* __restrict__ o, const uint16_t* __restrict__ dout,
                                    float* __restrict__ dsum, int B, int T, int H) {
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= int64_t(B) * T * H) return;
  const int h = int(w % H);
  const int64_t row = w / H;  // b*T + t
  const int64_t off = row * H * DH + h * DH;
  float s = 0.f;
  for (int d = lane * 2; d < DH; d += 64) {
    const uint32_t a = *reinterpret_cast<const uint32_t*>(o + off + d);
    const uint32_t c = *reinterpret_cast<const uint32_t*>(dout + off + d);
    s += bf16_lo(a) * bf16_lo(c) + bf16_hi(a) * bf16_hi(c);
  }
#pragma unroll
  for (int x = 16; x > 0; x >>= 1) s += __shfl_xor_sync(0xffffffffu, s, x);
  if (lane == 0) {
    const int b = int(row / T), t = int(row % T);
    dsum[(int64_t(b) * H + h) * T + t] = s;
  }
}

// Column sums over the 16 rows of a warp's C fragments (rows g, g+8 of
// n-tile j), accumulated into dbias[col0 + j*8 + 2*t4 + {0,1}].
template <int NT>
__device__ __forceinline__ void frag_colsum(const float (&c)[NT][4], float* dbias, int row_lo,
                                            int row_hi, int T) {
  const int lane = threadIdx.x & 31, t4 = lane & 3;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    float a = (row_lo < T ? c[j][0] : 0.f) + (row_hi < T ? c[j][2] : 0.f);
    float b2 = (row_lo < T ? c[j][1] : 0.f) + (row_hi < T ? c[j][3] : 0.f);
#pragma unroll
    for (int x = 4; x < 32; x <<= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, x);
      b2 += __shfl_xor_sync(0xffffffffu, b2, x);
    }
    if (lane < 4 && dbias != nullptr) {
      atomicAdd(dbias + j * 8 + 2 * t4, a);
      atomicAdd(dbias + j * 8 + 2 * t4 + 1, b2);
    }
  }
}

template <int NT>
__device__ __forceinline__ void store_frag_rows(uint16_t* base, int64_t ld, const float (&c)[NT][4],
                                                float scale, int row_lo, int row_hi, int T) {
  const int t4 = threadIdx.x & 3;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int col = j * 8 + 2 * t4;
    if (row_lo < T)
      *reinterpret_cast<uint32_t*>(base + int64_t(row_lo) * ld + col) =
          pack_bf16(c[j][0] * scale, c[j][1] * scale);
    if (row_hi < T)
      *reinterpret_cast<uint32_t*>(base + int64_t(row_hi) * ld + col) =
          pack_bf16(c[j][2] * scale, c[j][3] * scale);
  }
}

// dK / dV: grid (B*H, ceil(T/64)); warp owns 16 keys, loops over query blocks.
//   S^T = K Q^T, P^T = exp(S^T*scale - lse[q]), dV += P^T dO,
//   dP^T = V dO^T, dS^T = P^T * (dP^T - D[q]), dK += dS^T Q * scale.
template <int DH>
__global__ void __launch_bounds__(kAttWarps * 32)
    attn_bwd_dkdv_kernel(const uint16_t* __restrict__ qkv, const uint16_t* __restrict__ dout,
                         const float* __restrict__ lse, const float* __restrict__ dsum,
                         uint16_t* __restrict__ dqkv, float* __restrict__ dbias, int T, int H,
                         float scale) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int k0 = blockIdx.y * kBlk;
  const int64_t ld = int64_t(3) * H * DH, ldo = int64_t(H) * DH;
  const uint16_t* base = qkv + int64_t(b) * T * ld;
  const uint16_t* dob = dout + int64_t(b) * T * ldo;
  const int Tp = (T + kBlk - 1) / kBlk * kBlk;
  constexpr int RB = Tile<DH>::kBytesPerRow;
  const uint32_t sK = smem_addr(sm);
  const uint32_t sV = sK + kBlk * RB;
  const uint32_t sQ = sV + kBlk * RB;
  const uint32_t sO = sQ + Tp * RB;  // dO
  float* sL = reinterpret_cast<float*>(sm + (2 * kBlk + 2 * Tp) * RB);
  float* sD = sL + Tp;
  load_tile<DH>(sK, base, ld, H * DH + h * DH, k0, kBlk, T);
  load_tile<DH>(sV, base, ld, 2 * H * DH + h * DH, k0, kBlk, T);
  load_tile<DH>(sQ, base, ld, h * DH, 0, Tp, T);
  load_tile<DH>(sO, dob, ldo, h * DH, 0, Tp, T);
  for (int i = threadIdx.x; i < Tp; i += blockDim.x) {
    sL[i] = i < T ? lse[int64_t(bh) * T + i] : 0.f;
    sD[i] = i < T ? dsum[int64_t(bh) * T + i] : 0.f;
  }
  cp_async_wait_all();
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int r0 = warp * 16;  // local key rows
  uint32_t ka[DH / 16][4], va[DH / 16][4];
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) {
    lda_frag<DH>(sK, r0, kk * 16, ka[kk]);
    lda_frag<DH>(sV, r0, kk * 16, va[kk]);
  }
  float dk[DH / 8][4], dv[DH / 8][4];
#pragma unroll
  for (int j = 0; j < DH / 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[j][e] = dv[j][e] = 0.f;
  const float l2e = 1.4426950408889634f;

  for (int qb = 0; qb < Tp; qb += kBlk) {
    float st[8][4], dp[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) st[j][e] = dp[j][e] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; kk += 2) {
        uint32_t bq[4], bo[4];
        ldb_nk<DH>(sQ, qb + j * 8, kk * 16, bq);
        ldb_nk<DH>(sO, qb + j * 8, kk * 16, bo);
        mma16816(st[j], ka[kk], bq[0], bq[1]);
        mma16816(dp[j], va[kk], bo[0], bo[1]);
        if (kk + 1 < DH / 16) {
          mma16816(st[j], ka[kk + 1], bq[2], bq[3]);
          mma16816(dp[j], va[kk + 1], bo[2], bo[3]);
        }
      }
    }
    // P^T and dS^T (columns = queries)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int q = qb + j * 8 + 2 * t4 + (e & 1);
        const float p = q < T ? exp2f((st[j][e] * scale - sL[q]) * l2e) : 0.f;
        st[j][e] = p;
        dp[j][e] = p * (dp[j][e] - sD[q]);
      }
    }
    // dV += P^T dO ; dK += dS^T Q   (k = queries)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t pa[4], sa[4];
      pa[0] = pack_bf16(st[2 * i][0], st[2 * i][1]);
      pa[1] = pack_bf16(st[2 * i][2], st[2 * i][3]);
      pa[2] = pack_bf16(st[2 * i + 1][0], st[2 * i + 1][1]);
      pa[3] = pack_bf16(st[2 * i + 1][2], st[2 * i + 1][3]);
      sa[0] = pack_bf16(dp[2 * i][0], dp[2 * i][1]);
      sa[1] = pack_bf16(dp[2 * i][2], dp[2 * i][3]);
      sa[2] = pack_bf16(dp[2 * i + 1][0], dp[2 * i + 1][1]);
      sa[3] = pack_bf16(dp[2 * i + 1][2], dp[2 * i + 1][3]);
#pragma unroll
      for (int j = 0; j < DH / 8; j += 2) {
        uint32_t bo[4], bq[4];
        ldb_kn<DH>(sO, qb + i * 16, j * 8, bo);
        ldb_kn<DH>(sQ, qb + i * 16, j * 8, bq);
        mma16816(dv[j], pa, bo[0], bo[1]);
        mma16816(dv[j + 1], pa, bo[2], bo[3]);
        mma16816(dk[j], sa, bq[0], bq[1]);
        mma16816(dk[j + 1], sa, bq[2], bq[3]);
      }
    }
  }
  const int row_lo = k0 + r0 + g, row_hi = row_lo + 8;
  uint16_t* out_b = dqkv + int64_t(b) * T * ld;
#pragma unroll
  for (int j = 0; j < DH / 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[j][e] *= scale;
  store_frag_rows<DH / 8>(out_b + H * DH + h * DH, ld, dk, 1.f, row_lo, row_hi, T);
  store_frag_rows<DH / 8>(out_b + 2 * H * DH + h * DH, ld, dv, 1.f, row_lo, row_hi, T);
  if (dbias != nullptr) {
    // bias grads are sums of the stored (bf16) values
#pragma unroll
    for (int j = 0; j < DH / 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        dk[j][e] = __bfloat162float(__float2bfloat16_rn(dk[j][e]));
        dv[j][e] = __bfloat162float(__float2bfloat16_rn(dv[j][e]));
      }
    frag_colsum<DH / 8>(dk, dbias + H * DH + h * DH, row_lo, row_hi, T);
    frag_colsum<DH / 8>(dv, dbias + 2 * H * DH + h * DH, row_lo, row_hi, T);
  }
}

// dQ: grid (B*H, ceil(T/64)); warp owns 16 queries, loops over key blocks.
//   S = Q K^T, P = exp(S*scale - lse), dP = dO V^T, dS = P*(dP - D), dQ += dS K * scale.
template <int DH>
__global__ void __launch_bounds__(kAttWarps * 32)
    attn_bwd_dq_kernel(const uint16_t* __restrict__ qkv, const uint16_t* __restrict__ dout,
                       const float* __restrict__ lse, const float* __restrict__ dsum,
                       uint16_t* __restrict__ dqkv, float* __restrict__ dbias, int T, int H,
                       float scale) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int q0 = blockIdx.y * kBlk;
  const int64_t ld = int64_t(3) * H * DH, ldo = int64_t(H) * DH;
  const uint16_t* base = qkv + int64_t(b) * T * ld;
  const uint16_t* dob = dout + int64_t(b) * T * ldo;
  const int Tp = (T + kBlk - 1) / kBlk * kBlk;
  constexpr int RB = Tile<DH>::kBytesPerRow;
  const uint32_t sQ = smem_addr(sm);
  const uint32_t sO = sQ + kBlk * RB;
  const uint32_t sK = sO + kBlk * RB;
  const uint32_t sV = sK + Tp * RB;
  load_tile<DH>(sQ, base, ld, h * DH, q0, kBlk, T);
  load_tile<DH>(sO, dob, ldo, h * DH, q0, kBlk, T);
  load_tile<DH>(sK, base, ld, H * DH + h * DH, 0, Tp, T);
  load_tile<DH>(sV, base, ld, 2 * H * DH + h * DH, 0, Tp, T);
  cp_async_wait_all();
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int r0 = warp * 16;
  const int row_lo = q0 + r0 + g, row_hi = row_lo + 8;
  const float L_lo = row_lo < T ? lse[int64_t(bh) * T + row_lo] : 0.f;
  const float L_hi = row_hi < T ? lse[int64_t(bh) * T + row_hi] : 0.f;
  const float D_lo = row_lo < T ? dsum[int64_t(bh) * T + row_lo] : 0.f;
  const float D_hi = row_hi < T ? dsum[int64_t(bh) * T + row_hi] : 0.f;
  uint32_t qa[DH / 16][4], oa[DH / 16][4];
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) {
    lda_frag<DH>(sQ, r0, kk * 16, qa[kk]);
    lda_frag<DH>(sO, r0, kk * 16, oa[kk]);
  }
  float dq[DH / 8][4];
#pragma unroll
  for (int j = 0; j < DH / 8; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
  const float l2e = 1.4426950408889634f;

  for (int kb = 0; kb < Tp; kb += kBlk) {
    float s[8][4], dp[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int e = 0; e < 4; ++e) s[j][e] = dp[j][e] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int kk = 0; kk < DH / 16; kk += 2) {
        uint32_t bk[4], bv[4];
        ldb_nk<DH>(sK, kb + j * 8, kk * 16, bk);
        ldb_nk<DH>(sV, kb + j * 8, kk * 16, bv);
        mma16816(s[j], qa[kk], bk[0], bk[1]);
        mma16816(dp[j], oa[kk], bv[0], bv[1]);
        if (kk + 1 < DH / 16) {
          mma16816(s[j], qa[kk + 1], bk[2], bk[3]);
          mma16816(dp[j], oa[kk + 1], bv[2], bv[3]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kb + j * 8 + 2 * t4 + (e & 1);
        const bool hi = e >= 2;
        const float p = key < T ? exp2f((s[j][e] * scale - (hi ? L_hi : L_lo)) * l2e) : 0.f;
        dp[j][e] = p * (dp[j][e] - (hi ? D_hi : D_lo));
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t sa[4];
      sa[0] = pack_bf16(dp[2 * i][0], dp[2 * i][1]);
      sa[1] = pack_bf16(dp[2 * i][2], dp[2 * i][3]);
      sa[2] = pack_bf16(dp[2 * i + 1][0], dp[2 * i + 1][1]);
      sa[3] = pack_bf16(dp[2 * i + 1][2], dp[2 * i + 1][3]);
#pragma unroll
      for (int j = 0; j < DH / 8; j += 2) {
        uint32_t bk[4];
        ldb_kn<DH>(sK, kb + i * 16, j * 8, bk);
        mma16816(dq[j], sa, bk[0], bk[1]);
        mma16816(dq[j + 1], sa, bk[2], bk[3]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < DH / 8; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) dq[j][e] = __bfloat162float(__float2bfloat16_rn(dq[j][e] * scale));
  uint16_t* out_b = dqkv + int64_t(b) * T * ld;
  store_frag_rows<DH / 8>(out_b + h * DH, ld, dq, 1.f, row_lo, row_hi, T);
  if (dbias != nullptr) frag_colsum<DH / 8>(dq, dbias + h * DH, row_lo, row_hi, T);
}

template <int DH>
size_t fwd_smem(int T) {
  const int Tp = (T + kBlk - 1) / kBlk * kBlk;
  return size_t(kBlk + 2 * Tp) * Tile<DH>::kBytesPerRow;
}
template <int DH>
size_t bwd_smem(int T) {
  const int Tp = (T + kBlk - 1) / kBlk * kBlk;
  return size_t(2 * kBlk + 2 * Tp) * Tile<DH>::kBytesPerRow + size_t(2 * Tp) * sizeof(float);
}

template <int DH>
int attn_fwd_launch(const void* qkv, void* out, float* lse, int B, int T, int H, float scale,
                    cudaStream_t st) {
  const size_t smem = fwd_smem<DH>(T);
  if (smem > 227 * 1024) return EPS_EINVAL;
  cudaFuncSetAttribute(attn_fwd_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  dim3 grid(B * H, (T + kBlk - 1) / kBlk);
  count_launch(); attn_fwd_kernel<DH><<<grid, kAttWarps * 32, smem, st>>>(
      static_cast<const uint16_t*>(qkv), static_cast<uint16_t*>(out), lse, T, H,
      scale * 1.4426950408889634f);
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

template <int DH>
int attn_bwd_launch(const void* qkv, const void* out, const void* dout, const float* lse,
                    void* dqkv, float* dbias, float* dsum, int B, int T, int H, float scale,
                    cudaStream_t st) {
  const size_t smem = bwd_smem<DH>(T);
  if (smem > 227 * 1024) return EPS_EINVAL;
  const int64_t warps = int64_t(B) * T * H;
  count_launch(); attn_bwd_dot_kernel<DH><<<unsigned((warps * 32 + 255) / 256), 256, 0, st>>>(
      static_cast<const uint16_t*>(out), static_cast<const uint16_t*>(dout), dsum, B, T, H);
  cudaFuncSetAttribute(attn_bwd_dkdv_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(smem));
  cudaFuncSetAttribute(attn_bwd_dq_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(smem));
  dim3 grid(B * H, (T + kBlk - 1) / kBlk);
  count_launch(); attn_bwd_dkdv_kernel<DH><<<grid, kAttWarps * 32, smem, st>>>(
      static_cast<const uint16_t*>(qkv), static_cast<const uint16_t*>(dout), lse, dsum,
      static_cast<uint16_t*>(dqkv), dbias, T, H, scale);
  count_launch(); attn_bwd_dq_kernel<DH><<<grid, kAttWarps * 32, smem, st>>>(
      static_cast<const uint16_t*>(qkv), static_cast<const uint16_t*>(dout), lse, dsum,
      static_cast<uint16_t*>(dqkv), dbias, T, H, scale);
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}

bool attn_tc_supported(int T, int head_dim);
int attn_fwd_tc(const void* qkv, void* out, float* lse, int B, int T, int H, float scale,
                cudaStream_t st);
int attn_bwd_tc(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv,
                float* dbias, float* dsum, const float* drow, int B, int T, int H, float scale,
                cudaStream_t st);
bool attn_bwd_fused_supported(int T, int head_dim);

}  // namespace eps_k

// head_dim 64, T <= 384: tcgen05/TMEM kernels (attention_tc.cu); head_dim 32
// (the tiny ViT): the mma.sync kernels above.
extern "C" int eps_attn_fwd(const void* qkv, void* out, float* lse, int batch, int tokens,
                            int heads, int head_dim, float scale, void* stream) {
  using namespace eps_k;
  auto st = static_cast<cudaStream_t>(stream);
  if (batch < 1 || tokens < 1 || heads < 1) return EPS_EINVAL;
  if (attn_tc_supported(tokens, head_dim))
    return attn_fwd_tc(qkv, out, lse, batch, tokens, heads, scale, st);
  switch (head_dim) {
    case 32: return attn_fwd_launch<32>(qkv, out, lse, batch, tokens, heads, scale, st);
    case 64: return attn_fwd_launch<64>(qkv, out, lse, batch, tokens, heads, scale, st);
    default: return EPS_EINVAL;
  }
}

// dsum_workspace: fp32 [batch*heads*tokens] scratch for rowsum(dO*O).
extern "C" int eps_attn_bwd_ws(const void* qkv, const void* out, const void* dout,
                               const float* lse, void* dqkv, float* dbias_qkv,
                               float* dsum_workspace, int batch, int tokens, int heads,
                               int head_dim, float scale, void* stream) {
  using namespace eps_k;
  auto st = static_cast<cudaStream_t>(stream);
  if (batch < 1 || tokens < 1 || heads < 1) return EPS_EINVAL;
  if (attn_tc_supported(tokens, head_dim))
    return attn_bwd_tc(qkv, out, dout, lse, dqkv, dbias_qkv, dsum_workspace, nullptr, batch,
                       tokens, heads, scale, st);
  switch (head_dim) {
    case 32:
      return attn_bwd_launch<32>(qkv, out, dout, lse, dqkv, dbias_qkv, dsum_workspace, batch,
                                 tokens, heads, scale, st);
    case 64:
      return attn_bwd_launch<64>(qkv, out, dout, lse, dqkv, dbias_qkv, dsum_workspace, batch,
                                 tokens, heads, scale, st);
    default:
      return EPS_EINVAL;
  }
}

extern "C" int eps_attn_bwd_uses_rowdot(int tokens, int head_dim) {
  return eps_k::attn_bwd_fused_supported(tokens, head_dim) ? 1 : 0;
}

extern "C" int eps_attn_bwd_rowdot(const void* qkv, const void* out, const void* dout,
                                   const float* lse, const float* dsum_rows, void* dqkv,
                                   float* dbias_qkv, float* dsum_workspace, int batch, int tokens,
                                   int heads, int head_dim, float scale, void* stream) {
  using namespace eps_k;
  if (batch < 1 || tokens < 1 || heads < 1) return EPS_EINVAL;
  if (!attn_bwd_fused_supported(tokens, head_dim))
    return eps_attn_bwd_ws(qkv, out, dout, lse, dqkv, dbias_qkv, dsum_workspace, batch, tokens,
                           heads, head_dim, scale, stream);
  if (dsum_rows == nullptr) return EPS_EINVAL;
  return attn_bwd_tc(qkv, out, dout, lse, dqkv, dbias_qkv, dsum_workspace, dsum_rows, batch,
                     tokens, heads, scale, static_cast<cudaStream_t>(stream));
}
