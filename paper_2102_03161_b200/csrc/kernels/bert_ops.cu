// BERT front end and heads (HBM / latency-bound helpers around the GEMMs):
//   * embedding sum  E[b,t] = word[tok] + pos[t] + type[seg]  (fp32 tables ->
//     bf16 rows; the embedding LayerNorm is the regular LN kernel) and its
//     backward (row scatter-add of dE into the three fp32 gradient tables);
//   * SQuAD span loss: per sample, softmax over the T positions of the
//     start and end logit columns, CE averaged over the two, gradient back;
//   * tanh forward / backward for the pooler.
#include <cuda_runtime.h>

#include "eps_capi.h"
#include "ptx.cuh"

namespace eps_k {

__global__ void bert_embed_fwd_kernel(const int64_t* __restrict__ tok,
                                      const int64_t* __restrict__ seg,
                                      const float* __restrict__ word, const float* __restrict__ pos,
                                      const float* __restrict__ type, uint16_t* __restrict__ out,
                                      int64_t rows, int T, int64_t d) {
  const int64_t per_row = d / 4;
  const int64_t total = rows * per_row;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / per_row, c = (i - r * per_row) * 4;
    const int t = int(r % T);
    const float4 w = *reinterpret_cast<const float4*>(word + tok[r] * d + c);
    const float4 p = *reinterpret_cast<const float4*>(pos + int64_t(t) * d + c);
    const float4 y = *reinterpret_cast<const float4*>(type + seg[r] * d + c);
    *reinterpret_cast<uint2*>(out + r * d + c) =
        make_uint2(pack_bf16(w.x + p.x + y.x, w.y + p.y + y.y),
                   pack_bf16(w.z + p.z + y.z, w.w + p.w + y.w));
  }
}

__global__ void bert_embed_bwd_kernel(const uint16_t* __restrict__ de,
                                      const int64_t* __restrict__ tok,
                                      const int64_t* __restrict__ seg, float* __restrict__ dword,
                                      float* __restrict__ dpos, float* __restrict__ dtype,
                                      int64_t rows, int T, int64_t d) {
  const int64_t per_row = d / 4;
  const int64_t total = rows * per_row;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / per_row, c = (i - r * per_row) * 4;
    const int t = int(r % T);
    const uint2 g = *reinterpret_cast<const uint2*>(de + r * d + c);
    const float a = bf16_lo(g.x), b = bf16_hi(g.x), e = bf16_lo(g.y), f = bf16_hi(g.y);
    red_add_v4(dword + tok[r] * d + c, a, b, e, f);
    red_add_v4(dpos + int64_t(t) * d + c, a, b, e, f);
    red_add_v4(dtype + seg[r] * d + c, a, b, e, f);
  }
}

// One block per sample; columns 0 (start) and 1 (end) of logits[b*T + t].
__global__ void span_xent_kernel(const uint16_t* __restrict__ logits,
                                 const int64_t* __restrict__ start,
                                 const int64_t* __restrict__ end, uint16_t* __restrict__ dlogits,
                                 float* __restrict__ loss_sum, float* __restrict__ dbias, int T,
                                 int ld, float grad_scale) {
  const int b = blockIdx.x;
  __shared__ float red[2][32];
  __shared__ float stat[2][2];  // max, sum per column
  const uint16_t* L = logits + int64_t(b) * T * ld;
  uint16_t* dL = dlogits + int64_t(b) * T * ld;
  auto val = [&](int t, int col) { return __bfloat162float(__ushort_as_bfloat16(L[int64_t(t) * ld + col])); };
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int col = 0; col < 2; ++col) {
    float m = -3.0e38f;
    for (int t = threadIdx.x; t < T; t += blockDim.x) m = fmaxf(m, val(t, col));
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[col][warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      float mm = red[col][0];
      for (int w = 1; w < nw; ++w) mm = fmaxf(mm, red[col][w]);
      stat[col][0] = mm;
    }
    __syncthreads();
    float s = 0.f;
    for (int t = threadIdx.x; t < T; t += blockDim.x) s += __expf(val(t, col) - stat[col][0]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __syncthreads();
    if (lane == 0) red[col][warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      float ss = 0.f;
      for (int w = 0; w < nw; ++w) ss += red[col][w];
      stat[col][1] = ss;
    }
    __syncthreads();
  }
  const int64_t ys = start[b], ye = end[b];
  float c0 = 0.f, c1 = 0.f;
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    const float p0 = __expf(val(t, 0) - stat[0][0]) / stat[0][1];
    const float p1 = __expf(val(t, 1) - stat[1][0]) / stat[1][1];
    const float g0 = 0.5f * grad_scale * (p0 - (t == ys ? 1.f : 0.f));
    const float g1 = 0.5f * grad_scale * (p1 - (t == ye ? 1.f : 0.f));
    const uint16_t h0 = __bfloat16_as_ushort(__float2bfloat16_rn(g0));
    const uint16_t h1 = __bfloat16_as_ushort(__float2bfloat16_rn(g1));
    dL[int64_t(t) * ld + 0] = h0;
    dL[int64_t(t) * ld + 1] = h1;
    for (int c = 2; c < ld; ++c) dL[int64_t(t) * ld + c] = 0;
    c0 += __bfloat162float(__ushort_as_bfloat16(h0));
    c1 += __bfloat162float(__ushort_as_bfloat16(h1));
  }
  for (int o = 16; o > 0; o >>= 1) {
    c0 += __shfl_xor_sync(0xffffffffu, c0, o);
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
  }
  if (lane == 0) {
    atomicAdd(dbias + 0, c0);
    atomicAdd(dbias + 1, c1);
  }
  if (threadIdx.x == 0) {
    const float ls = stat[0][0] + __logf(stat[0][1]) - val(int(ys), 0);
    const float le = stat[1][0] + __logf(stat[1][1]) - val(int(ye), 1);
    atomicAdd(loss_sum, 0.5f * (ls + le));
  }
}

__global__ void tanh_fwd_kernel(const uint16_t* __restrict__ x, uint16_t* __restrict__ y,
                                int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __bfloat16_as_ushort(__float2bfloat16_rn(tanhf(__bfloat162float(__ushort_as_bfloat16(x[i])))));
}

__global__ void tanh_bwd_kernel(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ y,
                                uint16_t* __restrict__ dx, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float t = __bfloat162float(__ushort_as_bfloat16(y[i]));
    const float g = __bfloat162float(__ushort_as_bfloat16(dy[i]));
    dx[i] = __bfloat16_as_ushort(__float2bfloat16_rn(g * (1.f - t * t)));
  }
}

inline int grid_for(int64_t work) {
  const int64_t blocks = (work + 255) / 256;
  return int(blocks < 148 * 16 ? (blocks > 0 ? blocks : 1) : 148 * 16);
}

inline int launched() { return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA; }

}  // namespace eps_k

extern "C" int eps_bert_embed_fwd(const int64_t* tokens, const int64_t* segments,
                                  const float* word, const float* pos, const float* type,
                                  void* out, int batch, int tokens_per_sample, int64_t d,
                                  void* stream) {
  using namespace eps_k;
  if (batch < 1 || tokens_per_sample < 1 || d % 4 != 0) return EPS_EINVAL;
  const int64_t rows = int64_t(batch) * tokens_per_sample;
  count_launch();
  bert_embed_fwd_kernel<<<grid_for(rows * d / 4), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      tokens, segments, word, pos, type, static_cast<uint16_t*>(out), rows, tokens_per_sample, d);
  return launched();
}

extern "C" int eps_bert_embed_bwd(const void* d_embed, const int64_t* tokens,
                                  const int64_t* segments, float* dword, float* dpos,
                                  float* dtype, int batch, int tokens_per_sample, int64_t d,
                                  void* stream) {
  using namespace eps_k;
  if (batch < 1 || tokens_per_sample < 1 || d % 4 != 0) return EPS_EINVAL;
  const int64_t rows = int64_t(batch) * tokens_per_sample;
  count_launch();
  bert_embed_bwd_kernel<<<grid_for(rows * d / 4), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(d_embed), tokens, segments, dword, dpos, dtype, rows,
      tokens_per_sample, d);
  return launched();
}

extern "C" int eps_span_xent(const void* logits, const int64_t* start, const int64_t* end,
                             void* dlogits, float* loss_sum, float* dbias, int batch,
                             int tokens_per_sample, int ld, float grad_scale, void* stream) {
  using namespace eps_k;
  if (batch < 1 || tokens_per_sample < 1 || ld < 2) return EPS_EINVAL;
  count_launch();
  span_xent_kernel<<<batch, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(logits), start, end, static_cast<uint16_t*>(dlogits), loss_sum,
      dbias, tokens_per_sample, ld, grad_scale);
  return launched();
}

extern "C" int eps_tanh_fwd(const void* x, void* y, int64_t n, void* stream) {
  using namespace eps_k;
  if (n < 0) return EPS_EINVAL;
  if (n == 0) return EPS_OK;
  count_launch();
  tanh_fwd_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(x), static_cast<uint16_t*>(y), n);
  return launched();
}

extern "C" int eps_tanh_bwd(const void* dy, const void* y, void* dx, int64_t n, void* stream) {
  using namespace eps_k;
  if (n < 0) return EPS_EINVAL;
  if (n == 0) return EPS_OK;
  count_launch();
  tanh_bwd_kernel<<<grid_for(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(dy), static_cast<const uint16_t*>(y), static_cast<uint16_t*>(dx),
      n);
  return launched();
}
