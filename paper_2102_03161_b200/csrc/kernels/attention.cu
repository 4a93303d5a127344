// Multi-head self-attention C entry points over a packed QKV activation.
//
// Layout: qkv [B*T, 3*H*dh]: columns [0,Hdh) = Q, [Hdh,2Hdh) = K,
// [2Hdh,3Hdh) = V, head h at h*dh within each; out [B*T, H*dh]; lse [B,H,T].
// Every supported shape runs on the tcgen05 / TMEM kernels of attention_tc.cu:
// head_dim 64 directly, head_dim 32 (the tiny ViT) on heads zero-padded to 64
// (below); T <= 384.  Other shapes return EPS_EINVAL (no fallback path; the
// round-1 mma.sync kernels were retired in round 2).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "eps_capi.h"
#include "ptx.cuh"

namespace eps_k {

bool attn_tc_supported(int T, int head_dim);
int attn_fwd_tc(const void* qkv, void* out, float* lse, int B, int T, int H, float scale,
                cudaStream_t st);
int attn_bwd_tc(const void* qkv, const void* out, const void* dout, const float* lse, void* dqkv,
                float* dbias, float* dsum, const float* drow, int B, int T, int H, float scale,
                cudaStream_t st);
bool attn_bwd_fused_supported(int T, int head_dim);

// ---- head_dim 32 on the tcgen05 kernels ------------------------------------
// The tiny ViT's 32-wide heads run through the head_dim 64 tcgen05 kernels
// with every head's columns zero-padded to 64: Q K^T and dP are unchanged by
// the zero columns, P V / dQ / dK / dV get zero upper halves that are dropped
// again (the softmax scale stays the caller's 1 / sqrt(32)).  The pad / unpad
// copies are HBM-trivial at the tiny ViT's size (64 x 65 rows).
__global__ void head_pad_kernel(const uint16_t* __restrict__ src, uint16_t* __restrict__ dst,
                                int64_t rows, int groups, int pad) {
  // one thread per 16-byte vector of the 64-wide layout: (row, group, v < 8)
  const int64_t n = rows * groups * 8;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int v = int(i & 7);
    const int64_t rg = i >> 3;
    const int64_t r = rg / groups;
    const int g = int(rg - r * groups);
    const int64_t wide = (r * groups + g) * 64 + v * 8, narrow = (r * groups + g) * 32 + v * 8;
    if (pad) {
      *reinterpret_cast<uint4*>(dst + wide) =
          v < 4 ? *reinterpret_cast<const uint4*>(src + narrow) : make_uint4(0u, 0u, 0u, 0u);
    } else if (v < 4) {
      *reinterpret_cast<uint4*>(dst + narrow) = *reinterpret_cast<const uint4*>(src + wide);
    }
  }
}
__global__ void head_unpad_add_f32_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                          int groups) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < groups * 32) dst[i] += src[(i >> 5) * 64 + (i & 31)];
}
int head_pad(const void* src, void* dst, int64_t rows, int groups, bool pad, cudaStream_t st) {
  const int64_t n = rows * groups * 8;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, 148 * 16));
  count_launch();
  head_pad_kernel<<<blocks, 256, 0, st>>>(static_cast<const uint16_t*>(src),
                                          static_cast<uint16_t*>(dst), rows, groups, pad ? 1 : 0);
  return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
}
// grow-only device scratch for the padded operands (cudaFree / cudaMalloc
// synchronise the device; growth happens once per size)
void* pad_scratch(size_t bytes) {
  static void* p = nullptr;
  static size_t have = 0;
  if (bytes > have) {
    if (p != nullptr) cudaFree(p);
    p = nullptr;
    have = 0;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    have = bytes;
  }
  return p;
}

}  // namespace eps_k

// head_dim 64, T <= 384: tcgen05/TMEM kernels (attention_tc.cu); head_dim 32
// (the tiny ViT), T <= 384: the same kernels on zero-padded heads (above).
extern "C" int eps_attn_fwd(const void* qkv, void* out, float* lse, int batch, int tokens,
                            int heads, int head_dim, float scale, void* stream) {
  using namespace eps_k;
  auto st = static_cast<cudaStream_t>(stream);
  if (batch < 1 || tokens < 1 || heads < 1) return EPS_EINVAL;
  if (attn_tc_supported(tokens, head_dim))
    return attn_fwd_tc(qkv, out, lse, batch, tokens, heads, scale, st);
  if (head_dim == 32 && attn_tc_supported(tokens, 64)) {
    const int64_t R = int64_t(batch) * tokens;
    uint16_t* q64 = static_cast<uint16_t*>(pad_scratch(size_t(R) * 4 * heads * 64 * 2));
    if (q64 == nullptr) return EPS_ECUDA;
    uint16_t* o64 = q64 + R * 3 * heads * 64;
    int rc = head_pad(qkv, q64, R, 3 * heads, true, st);
    if (rc == EPS_OK) rc = attn_fwd_tc(q64, o64, lse, batch, tokens, heads, scale, st);
    if (rc == EPS_OK) rc = head_pad(o64, out, R, heads, false, st);
    return rc;
  }
  return EPS_EINVAL;
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
  if (head_dim == 32 && attn_tc_supported(tokens, 64)) {
    // padded qkv | out | dout | dqkv (bf16), then dbias (fp32 [3 H 64])
    const int64_t R = int64_t(batch) * tokens, W3 = 3 * int64_t(heads) * 64, W1 = heads * 64;
    const size_t bf = size_t(R) * size_t(2 * W3 + 2 * W1) * 2;
    uint16_t* q64 = static_cast<uint16_t*>(pad_scratch(bf + size_t(W3) * 4));
    if (q64 == nullptr) return EPS_ECUDA;
    uint16_t* o64 = q64 + R * W3;
    uint16_t* do64 = o64 + R * W1;
    uint16_t* dq64 = do64 + R * W1;
    float* db64 = reinterpret_cast<float*>(dq64 + R * W3);
    int rc = head_pad(qkv, q64, R, 3 * heads, true, st);
    if (rc == EPS_OK) rc = head_pad(out, o64, R, heads, true, st);
    if (rc == EPS_OK) rc = head_pad(dout, do64, R, heads, true, st);
    if (rc == EPS_OK && cudaMemsetAsync(db64, 0, size_t(W3) * 4, st) != cudaSuccess) rc = EPS_ECUDA;
    if (rc == EPS_OK)
      rc = attn_bwd_tc(q64, o64, do64, lse, dq64, dbias_qkv != nullptr ? db64 : nullptr,
                       dsum_workspace, nullptr, batch, tokens, heads, scale, st);
    if (rc == EPS_OK) rc = head_pad(dq64, dqkv, R, 3 * heads, false, st);
    if (rc == EPS_OK && dbias_qkv != nullptr) {
      count_launch();
      head_unpad_add_f32_kernel<<<(3 * heads * 32 + 255) / 256, 256, 0, st>>>(db64, dbias_qkv,
                                                                            3 * heads);
      rc = cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA;
    }
    return rc;
  }
  return EPS_EINVAL;
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
