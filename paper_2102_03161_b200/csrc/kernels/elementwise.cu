// HBM-bound kernels around the transformer blocks: ViT frontend (patchify
// with optional nearest upsampling, token assembly and its backward),
// softmax cross-entropy head, fused optimizers, the freeze test's segmented
// gradient sum-of-squares, and the AutoCache HBM store gather / scatter.
#include <cuda_runtime.h>

#include "eps_capi.h"
#include "ptx.cuh"

namespace eps_k {

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline int ok_or_cuda() { return cudaGetLastError() == cudaSuccess ? EPS_OK : EPS_ECUDA; }

// ---- ViT frontend -------------------------------------------------------------
// patches[b*P + p, (c*ps + kh)*ps + kw] = img[b, c, y, x] (Conv2d weight order),
// y = (ph*ps + kh) * in / out (nearest) when the stored image is smaller.
// Four consecutive kw per thread (ps % 4 == 0): one float4 in, 8 B out.
__global__ void patchify_kernel(const float* __restrict__ img, uint16_t* __restrict__ out,
                                int batch, int channels, int in_side, int out_side, int ps) {
  const int per_side = out_side / ps;
  const int patches = per_side * per_side;
  const int row_len = channels * ps * ps;  // patch vector length
  const int64_t total4 = int64_t(batch) * patches * row_len / 4;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total4;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = i * 4;
    const int64_t row = e / row_len;
    const int col = int(e % row_len);
    const int b = int(row / patches), p = int(row % patches);
    const int c = col / (ps * ps), kh = (col / ps) % ps, kw0 = col % ps;
    const int py = (p / per_side) * ps + kh, px0 = (p % per_side) * ps + kw0;
    const float* src = img + (int64_t(b) * channels + c) * in_side * in_side;
    float v[4];
    if (in_side == out_side) {
      const float4 a = *reinterpret_cast<const float4*>(src + int64_t(py) * in_side + px0);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else {
      const int sy = py * in_side / out_side;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        v[j] = __ldg(src + int64_t(sy) * in_side + (px0 + j) * in_side / out_side);
    }
    *reinterpret_cast<uint2*>(out + e) = make_uint2(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]));
  }
}

// x[b, 0] = cls + pos[0]; x[b, 1 + p] = tok[b*P + p] + pos[1 + p]   (8 bf16 / thread)
__global__ void assemble_kernel(const uint16_t* __restrict__ tok, const float* __restrict__ cls,
                                const float* __restrict__ pos, uint16_t* __restrict__ x,
                                int batch, int tokens, int d) {
  const int64_t total8 = int64_t(batch) * tokens * d / 8;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total8;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = i * 8;
    const int64_t row = e / d;
    const int col = int(e % d);
    const int b = int(row / tokens), t = int(row % tokens);
    float v[8];
    if (t == 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldg(cls + col + j);
    } else {
      const uint4 w =
          *reinterpret_cast<const uint4*>(tok + (int64_t(b) * (tokens - 1) + t - 1) * d + col);
      v[0] = bf16_lo(w.x); v[1] = bf16_hi(w.x); v[2] = bf16_lo(w.y); v[3] = bf16_hi(w.y);
      v[4] = bf16_lo(w.z); v[5] = bf16_hi(w.z); v[6] = bf16_lo(w.w); v[7] = bf16_hi(w.w);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] += __ldg(pos + int64_t(t) * d + col + j);
    *reinterpret_cast<uint4*>(x + e) = make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]),
                                                  pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
  }
}

// Backward of assemble: dpos[t] += sum_b dx[b,t]; dcls += sum_b dx[b,0];
// dtok[b*P+p] = dx[b,1+p] (optional) -- assemble_bwd_split_kernel below.

// ---- softmax cross-entropy -------------------------------------------------------
// One warp per row: loss_sum += lse - z[label]; dz = (softmax - onehot) / B;
// dbias (optional) += column sums of dz.
__global__ void xent_kernel(const uint16_t* __restrict__ logits, const int64_t* __restrict__ labels,
                            uint16_t* __restrict__ dlogits, float* __restrict__ loss_sum,
                            float* __restrict__ dbias, int batch, int classes, int ld,
                            float grad_scale) {
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (row >= batch) return;
  const uint16_t* z = logits + int64_t(row) * ld;
  float m = -INFINITY;
  for (int c = lane; c < classes; c += 32) m = fmaxf(m, __uint_as_float(uint32_t(z[c]) << 16));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float s = 0.f;
  for (int c = lane; c < classes; c += 32) s += __expf(__uint_as_float(uint32_t(z[c]) << 16) - m);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float lse = m + __logf(s);
  const int64_t y = labels[row];
  if (lane == 0) atomicAdd(loss_sum, lse - __uint_as_float(uint32_t(z[y]) << 16));
  const float inv_b = grad_scale;
  for (int c = lane; c < ld; c += 32) {
    float g = 0.f;  // padding columns (c >= classes) carry no gradient
    if (c < classes) {
      const float p = __expf(__uint_as_float(uint32_t(z[c]) << 16) - lse);
      g = (p - (c == y ? 1.0f : 0.0f)) * inv_b;
    }
    const __nv_bfloat16 gb = __float2bfloat16_rn(g);
    dlogits[int64_t(row) * ld + c] = *reinterpret_cast<const uint16_t*>(&gb);
    if (dbias != nullptr && c < classes) atomicAdd(dbias + c, __bfloat162float(gb));
  }
}

// ---- optimizers -------------------------------------------------------------------
__global__ void sgd_kernel(float* __restrict__ p, uint16_t* __restrict__ pb, float* __restrict__ g,
                           float* __restrict__ mom, int64_t n, float lr, float mu, float wd) {
  const int64_t n4 = n / 4;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    float4 pv = reinterpret_cast<float4*>(p)[i];
    float4 gv = reinterpret_cast<float4*>(g)[i];
    float4 mv = reinterpret_cast<float4*>(mom)[i];
    float* pp = &pv.x;
    float* gg = &gv.x;
    float* mm = &mv.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float gr = gg[j] + wd * pp[j];
      mm[j] = mu * mm[j] + gr;
      pp[j] -= lr * mm[j];
    }
    reinterpret_cast<float4*>(p)[i] = pv;
    reinterpret_cast<float4*>(mom)[i] = mv;
    reinterpret_cast<float4*>(g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    reinterpret_cast<uint2*>(pb)[i] = make_uint2(pack_bf16(pv.x, pv.y), pack_bf16(pv.z, pv.w));
  }
  for (int64_t i = n4 * 4 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float gr = g[i] + wd * p[i];
    mom[i] = mu * mom[i] + gr;
    p[i] -= lr * mom[i];
    g[i] = 0.f;
    const __nv_bfloat16 b = __float2bfloat16_rn(p[i]);
    pb[i] = *reinterpret_cast<const uint16_t*>(&b);
  }
}

__global__ void adamw_kernel(float* __restrict__ p, uint16_t* __restrict__ pb, float* __restrict__ g,
                             float* __restrict__ m, float* __restrict__ v, int64_t n, float lr,
                             float b1, float b2, float eps, float wd, float c1, float c2) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float gr = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gr;
    const float vi = b2 * v[i] + (1.f - b2) * gr * gr;
    m[i] = mi;
    v[i] = vi;
    float pv = p[i] * (1.f - lr * wd);
    pv -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
    p[i] = pv;
    g[i] = 0.f;
    const __nv_bfloat16 b = __float2bfloat16_rn(pv);
    pb[i] = *reinterpret_cast<const uint16_t*>(&b);
  }
}

// ---- freeze test: segmented sum of squares ---------------------------------------
// Segment s = flat[off[s], off[s+1]).  Block b handles one fixed 64K-element
// chunk of one segment (table in the kernel argument) and writes its fp64
// partial; a second pass sums each segment's partials in chunk order, so
// the result is bit-reproducible run to run.
constexpr int kMaxSeg = 64;
constexpr int64_t kNormChunk = 1 << 16;
struct SegTable {
  int64_t off[kMaxSeg + 1];
  int first_block[kMaxSeg + 1];
  int n;
};

__global__ void sqnorm_partial_kernel(const float* __restrict__ flat, SegTable t,
                                      double* __restrict__ partial) {
  int s = 0;
  while (s + 1 < t.n && int(blockIdx.x) >= t.first_block[s + 1]) ++s;
  const int64_t lo = t.off[s] + int64_t(blockIdx.x - t.first_block[s]) * kNormChunk;
  const int64_t hi = min(lo + kNormChunk, t.off[s + 1]);
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const float v = flat[i];
    acc += double(v) * double(v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) b += ws[w];
    partial[blockIdx.x] = b;
  }
}

__global__ void sqnorm_final_kernel(const double* __restrict__ partial, SegTable t,
                                    double* __restrict__ out) {
  const int s = threadIdx.x;
  if (s >= t.n) return;
  double acc = 0.0;
  for (int b = t.first_block[s]; b < t.first_block[s + 1]; ++b) acc += partial[b];
  out[s] = acc;
}

// ---- AutoCache store ----------------------------------------------------------------
__global__ void cache_copy_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                  const int64_t* __restrict__ ids, int64_t row_bytes,
                                  bool gather) {
  const int r = blockIdx.y;
  const int64_t key = ids[r];
  const uint4* s = reinterpret_cast<const uint4*>(src + (gather ? key : r) * row_bytes);
  uint4* d = reinterpret_cast<uint4*>(dst + (gather ? r : key) * row_bytes);
  const int64_t n16 = row_bytes / 16;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += int64_t(gridDim.x) * blockDim.x)
    d[i] = s[i];
}

// AutoCache store sharded over the ranks of a node (one shard per GPU, rows
// [r * rows_per_shard, (r + 1) * rows_per_shard) on rank r, every shard
// mapped into every rank over CUDA IPC): sample `key` lives at row
// key % rows_per_shard of shard key / rows_per_shard, so a gather reads a
// peer GPU's HBM over NVLink (and a scatter writes it) inside this one
// kernel -- no store replication, broadcast or all-reduce.
__global__ void cache_copy_sharded_kernel(const uint64_t* __restrict__ shards,
                                          int64_t rows_per_shard, uint8_t* __restrict__ local,
                                          const int64_t* __restrict__ ids, int64_t row_bytes,
                                          bool gather) {
  const int r = blockIdx.y;
  const int64_t key = ids[r];
  uint8_t* remote = reinterpret_cast<uint8_t*>(shards[key / rows_per_shard]) +
                    (key % rows_per_shard) * row_bytes;
  const uint4* s = reinterpret_cast<const uint4*>(gather ? remote : local + r * row_bytes);
  uint4* d = reinterpret_cast<uint4*>(gather ? local + r * row_bytes : remote);
  const int64_t n16 = row_bytes / 16;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += int64_t(gridDim.x) * blockDim.x)
    d[i] = s[i];
}

// Background gather for the host tier's prefetch window: a few CTAs walk all
// (row, 16-byte) pairs with four independent 16-byte loads in flight per
// thread (enough outstanding host-link reads for full PCIe rate from ~8 SMs),
// so the copy overlaps the compute kernels instead of flooding every SM.
__global__ void __launch_bounds__(256) cache_gather_bg_kernel(
    const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, const int64_t* __restrict__ ids,
    int n, int64_t row_bytes) {
  const int64_t n16 = row_bytes / 16, total = n16 * n;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; base < total;
       base += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = base + u * stride;
      if (i < total) {
        const int64_t r = i / n16, c = i - r * n16;
        v[u] = reinterpret_cast<const uint4*>(src + ids[r] * row_bytes)[c];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = base + u * stride;
      if (i < total) {
        const int64_t r = i / n16, c = i - r * n16;
        reinterpret_cast<uint4*>(dst + r * row_bytes)[c] = v[u];
      }
    }
  }
}

__global__ void rows_copy_kernel(const uint16_t* __restrict__ src, int64_t src_stride,
                                 uint16_t* __restrict__ dst, int64_t dst_stride, int rows,
                                 int64_t d) {
  const int r = blockIdx.y;
  if (r >= rows) return;
  const uint4* s = reinterpret_cast<const uint4*>(src + r * src_stride);
  uint4* o = reinterpret_cast<uint4*>(dst + r * dst_stride);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < d / 8;
       i += int64_t(gridDim.x) * blockDim.x)
    o[i] = s[i];
}

__global__ void colsum_kernel(const uint16_t* __restrict__ x, float* __restrict__ out,
                              int64_t rows, int64_t cols, int64_t rows_per_block) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int64_t r0 = int64_t(blockIdx.y) * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) s += __uint_as_float(uint32_t(x[r * cols + c]) << 16);
  atomicAdd(out + c, s);
}

// Row-per-block variants (no 64-bit divisions per element): one block per
// patch row / token row, one thread per 4 (patchify) or 8 (assemble) columns.
__global__ void patchify_rows_kernel(const float* __restrict__ img, uint16_t* __restrict__ out,
                                     int channels, int side, int ps) {
  const int per_side = side / ps, patches = per_side * per_side;
  const int row = blockIdx.x;  // b * patches + p
  const int b = row / patches, p = row - b * patches;
  const int col = threadIdx.x * 4;  // within channels * ps * ps
  const int c = col / (ps * ps), rem = col - c * ps * ps, kh = rem / ps, kw0 = rem - kh * ps;
  const int py = (p / per_side) * ps + kh, px0 = (p % per_side) * ps + kw0;
  const float4 a = __ldg(reinterpret_cast<const float4*>(
      img + (int64_t(b) * channels + c) * side * side + int64_t(py) * side + px0));
  *reinterpret_cast<uint2*>(out + int64_t(row) * channels * ps * ps + col) =
      make_uint2(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w));
}

__global__ void assemble_rows_kernel(const uint16_t* __restrict__ tok, const float* __restrict__ cls,
                                     const float* __restrict__ pos, uint16_t* __restrict__ x,
                                     int tokens, int d) {
  const int row = blockIdx.x;  // b * tokens + t
  const int b = row / tokens, t = row - b * tokens;
  const int col = threadIdx.x * 8;
  float v[8];
  if (t == 0) {
    const float4 c0 = __ldg(reinterpret_cast<const float4*>(cls + col));
    const float4 c1 = __ldg(reinterpret_cast<const float4*>(cls + col) + 1);
    v[0] = c0.x; v[1] = c0.y; v[2] = c0.z; v[3] = c0.w;
    v[4] = c1.x; v[5] = c1.y; v[6] = c1.z; v[7] = c1.w;
  } else {
    const uint4 w = *reinterpret_cast<const uint4*>(tok + (int64_t(b) * (tokens - 1) + t - 1) * d + col);
    v[0] = bf16_lo(w.x); v[1] = bf16_hi(w.x); v[2] = bf16_lo(w.y); v[3] = bf16_hi(w.y);
    v[4] = bf16_lo(w.z); v[5] = bf16_hi(w.z); v[6] = bf16_lo(w.w); v[7] = bf16_hi(w.w);
  }
  const float4 p0 = __ldg(reinterpret_cast<const float4*>(pos + int64_t(t) * d + col));
  const float4 p1 = __ldg(reinterpret_cast<const float4*>(pos + int64_t(t) * d + col) + 1);
  v[0] += p0.x; v[1] += p0.y; v[2] += p0.z; v[3] += p0.w;
  v[4] += p1.x; v[5] += p1.y; v[6] += p1.z; v[7] += p1.w;
  *reinterpret_cast<uint4*>(x + int64_t(row) * d + col) =
      make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]),
                 pack_bf16(v[6], v[7]));
}

// Backward of assemble (block = token t, 256-col slab, batch slice z), batch split over gridDim.z slices with 4 independent
// accumulators per thread (the sequential 400-sample loop was latency-bound).
__global__ void assemble_bwd_split_kernel(const uint16_t* __restrict__ dx, float* __restrict__ dcls,
                                          float* __restrict__ dpos, uint16_t* __restrict__ dtok,
                                          int batch, int tokens, int d) {
  const int t = blockIdx.x;
  const int col = blockIdx.y * blockDim.x + threadIdx.x;
  if (col >= d) return;
  const int per = (batch + gridDim.z - 1) / gridDim.z;
  const int b0 = blockIdx.z * per, b1 = min(batch, b0 + per);
  float s[4] = {0.f, 0.f, 0.f, 0.f};
  int b = b0;
  for (; b + 4 <= b1; b += 4) {
    uint16_t raw[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) raw[u] = dx[(int64_t(b + u) * tokens + t) * d + col];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      s[u] += __uint_as_float(uint32_t(raw[u]) << 16);
      if (dtok != nullptr && t > 0) dtok[(int64_t(b + u) * (tokens - 1) + t - 1) * d + col] = raw[u];
    }
  }
  for (; b < b1; ++b) {
    const uint16_t raw = dx[(int64_t(b) * tokens + t) * d + col];
    s[0] += __uint_as_float(uint32_t(raw) << 16);
    if (dtok != nullptr && t > 0) dtok[(int64_t(b) * (tokens - 1) + t - 1) * d + col] = raw;
  }
  const float sum = (s[0] + s[1]) + (s[2] + s[3]);
  if (dpos != nullptr) atomicAdd(dpos + int64_t(t) * d + col, sum);
  if (t == 0 && dcls != nullptr) atomicAdd(dcls + col, sum);
}

}  // namespace eps_k

using namespace eps_k;

extern "C" int eps_patchify(const float* images, void* patches, int batch, int channels,
                            int image, int patch, void* stream) {
  // `image` packs (stored side << 16) | model side when they differ.
  const int out_side = image & 0xFFFF;
  const int in_side = (image >> 16) ? (image >> 16) : out_side;
  if (patch % 4 != 0 || out_side % patch != 0) return EPS_EINVAL;
  const int row_len = channels * patch * patch;
  if (in_side == out_side && row_len / 4 <= 1024) {
    const int rows = batch * (out_side / patch) * (out_side / patch);
    count_launch();
    patchify_rows_kernel<<<rows, row_len / 4, 0, static_cast<cudaStream_t>(stream)>>>(
        images, static_cast<uint16_t*>(patches), channels, out_side, patch);
    return ok_or_cuda();
  }
  count_launch(); patchify_kernel<<<num_sms() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      images, static_cast<uint16_t*>(patches), batch, channels, in_side, out_side, patch);
  return ok_or_cuda();
}

extern "C" int eps_vit_assemble(const void* patch_tokens, const float* cls, const float* pos,
                                void* x, int batch, int tokens, int64_t d, void* stream) {
  if (d % 8 != 0) return EPS_EINVAL;
  if (d / 8 <= 1024) {
    count_launch();
    assemble_rows_kernel<<<batch * tokens, int(d / 8), 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint16_t*>(patch_tokens), cls, pos, static_cast<uint16_t*>(x), tokens,
        int(d));
    return ok_or_cuda();
  }
  count_launch(); assemble_kernel<<<num_sms() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(patch_tokens), cls, pos, static_cast<uint16_t*>(x), batch,
      tokens, int(d));
  return ok_or_cuda();
}

extern "C" int eps_vit_assemble_bwd(const void* dx, float* dcls, float* dpos, void* dpatch_tokens,
                                    int batch, int tokens, int64_t d, void* stream) {
  const int splits = batch >= 64 ? 8 : 1;
  dim3 grid(tokens, unsigned((d + 255) / 256), unsigned(splits));
  count_launch();
  assemble_bwd_split_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(dx), dcls, dpos, static_cast<uint16_t*>(dpatch_tokens), batch,
      tokens, int(d));
  return ok_or_cuda();
}

extern "C" int eps_softmax_xent(const void* logits, const int64_t* labels, void* dlogits,
                                float* loss_sum, int batch, int classes, void* stream) {
  count_launch(); xent_kernel<<<(batch + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(logits), labels, static_cast<uint16_t*>(dlogits), loss_sum,
      nullptr, batch, classes, classes, 1.0f / batch);
  return ok_or_cuda();
}

extern "C" int eps_softmax_xent_bias(const void* logits, const int64_t* labels, void* dlogits,
                                     float* loss_sum, float* dbias, int batch, int classes,
                                     int ld, float grad_scale, void* stream) {
  count_launch(); xent_kernel<<<(batch + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(logits), labels, static_cast<uint16_t*>(dlogits), loss_sum,
      dbias, batch, classes, ld, grad_scale);
  return ok_or_cuda();
}

extern "C" int eps_sgd_momentum(float* param, uint16_t* param_bf16, float* grad, float* momentum,
                                int64_t n, float lr, float mu, float weight_decay, void* stream) {
  if (n <= 0) return EPS_OK;
  if ((reinterpret_cast<uintptr_t>(param) | reinterpret_cast<uintptr_t>(grad) |
       reinterpret_cast<uintptr_t>(momentum)) % 16 ||
      reinterpret_cast<uintptr_t>(param_bf16) % 8)
    return EPS_EINVAL;
  count_launch(); sgd_kernel<<<num_sms() * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      param, param_bf16, grad, momentum, n, lr, mu, weight_decay);
  return ok_or_cuda();
}

extern "C" int eps_adamw(float* param, uint16_t* param_bf16, float* grad, float* m, float* v,
                         int64_t n, float lr, float beta1, float beta2, float eps,
                         float weight_decay, int step, void* stream) {
  if (n <= 0) return EPS_OK;
  const float c1 = 1.f - powf(beta1, float(step)), c2 = 1.f - powf(beta2, float(step));
  count_launch(); adamw_kernel<<<num_sms() * 4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      param, param_bf16, grad, m, v, n, lr, beta1, beta2, eps, weight_decay, c1, c2);
  return ok_or_cuda();
}

// Flat-arena form of the segmented reduction: segments are contiguous ranges
// [seg_offsets[s], seg_offsets[s+1]) of one fp32 gradient buffer (host array).
// workspace: >= 8 * ceil(total/65536) + 64 bytes.  out: device double[n_segments].
extern "C" int eps_grad_sqnorm_flat(const float* flat, const int64_t* seg_offsets, int n_segments,
                                    double* out, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  if (n_segments < 1 || n_segments > kMaxSeg) return EPS_EINVAL;
  SegTable t{};
  t.n = n_segments;
  int blocks = 0;
  for (int s = 0; s < n_segments; ++s) {
    t.off[s] = seg_offsets[s];
    t.first_block[s] = blocks;
    const int64_t len = seg_offsets[s + 1] - seg_offsets[s];
    if (len < 0) return EPS_EINVAL;
    blocks += int((len + kNormChunk - 1) / kNormChunk);
  }
  t.off[n_segments] = seg_offsets[n_segments];
  t.first_block[n_segments] = blocks;
  if (workspace_bytes < size_t(blocks) * sizeof(double)) return EPS_ECAPACITY;
  auto st = static_cast<cudaStream_t>(stream);
  double* partial = static_cast<double*>(workspace);
  if (blocks > 0) { count_launch(); sqnorm_partial_kernel<<<blocks, 512, 0, st>>>(flat, t, partial); }
  count_launch(); sqnorm_final_kernel<<<1, 64, 0, st>>>(partial, t, out);
  return ok_or_cuda();
}

extern "C" int eps_grad_sqnorm_segmented(const float* const* tensors, const int64_t* n,
                                         const int* seg, int n_tensors, double* out,
                                         int n_segments, void* workspace, size_t workspace_bytes,
                                         void* stream) {
  // Tensor-list form: tensors must be laid out back to back in one arena in
  // segment order (the executor's layout); validated, then reduced flat.
  if (n_tensors < 1) return EPS_EINVAL;
  int64_t offs[kMaxSeg + 1];
  int cur = -1;
  const float* base = tensors[0];
  int64_t at = 0;
  for (int i = 0; i < n_tensors; ++i) {
    if (tensors[i] != base + at) return EPS_EINVAL;
    if (seg[i] != cur) {
      if (seg[i] != cur + 1 || seg[i] >= n_segments) return EPS_EINVAL;
      cur = seg[i];
      offs[cur] = at;
    }
    at += n[i];
  }
  if (cur != n_segments - 1) return EPS_EINVAL;
  offs[n_segments] = at;
  return eps_grad_sqnorm_flat(base, offs, n_segments, out, workspace, workspace_bytes, stream);
}

extern "C" int eps_cache_gather(const void* store, const int64_t* ids, int n, int64_t row_bytes,
                                void* dst, void* stream) {
  if (n <= 0) return EPS_OK;
  if (row_bytes % 16) return EPS_EINVAL;
  dim3 grid(unsigned(std::min<int64_t>((row_bytes / 16 + 255) / 256, 64)), unsigned(n));
  count_launch(); cache_copy_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(store), static_cast<uint8_t*>(dst), ids, row_bytes, true);
  return ok_or_cuda();
}

// shards: device array of n_shards base pointers (uint64), shard r holding
// sample rows [r * rows_per_shard, (r + 1) * rows_per_shard).
static int cache_sharded(const uint64_t* shards, int64_t rows_per_shard, const int64_t* ids,
                         int n, int64_t row_bytes, void* local, bool gather, void* stream) {
  if (n <= 0) return EPS_OK;
  if (row_bytes % 16 || shards == nullptr || rows_per_shard <= 0) return EPS_EINVAL;
  dim3 grid(unsigned(std::min<int64_t>((row_bytes / 16 + 255) / 256, 64)), unsigned(n));
  count_launch();
  cache_copy_sharded_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      shards, rows_per_shard, static_cast<uint8_t*>(local), ids, row_bytes, gather);
  return ok_or_cuda();
}

extern "C" int eps_cache_gather_sharded(const uint64_t* shards, int64_t rows_per_shard,
                                        const int64_t* ids, int n, int64_t row_bytes, void* dst,
                                        void* stream) {
  return cache_sharded(shards, rows_per_shard, ids, n, row_bytes, dst, true, stream);
}

extern "C" int eps_cache_scatter_sharded(const uint64_t* shards, int64_t rows_per_shard,
                                         const int64_t* ids, int n, int64_t row_bytes,
                                         const void* src, void* stream) {
  return cache_sharded(shards, rows_per_shard, ids, n, row_bytes, const_cast<void*>(src), false,
                       stream);
}

extern "C" int eps_cache_gather_bg(const void* store, const int64_t* ids, int n,
                                   int64_t row_bytes, void* dst, int ctas, void* stream) {
  if (n <= 0) return EPS_OK;
  if (row_bytes % 16 || ctas <= 0) return EPS_EINVAL;
  count_launch();
  cache_gather_bg_kernel<<<ctas, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(store), static_cast<uint8_t*>(dst), ids, n, row_bytes);
  return ok_or_cuda();
}

extern "C" int eps_cache_scatter(void* store, const int64_t* ids, int n, int64_t row_bytes,
                                 const void* src, void* stream) {
  if (n <= 0) return EPS_OK;
  if (row_bytes % 16) return EPS_EINVAL;
  dim3 grid(unsigned(std::min<int64_t>((row_bytes / 16 + 255) / 256, 64)), unsigned(n));
  count_launch(); cache_copy_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src), static_cast<uint8_t*>(store), ids, row_bytes, false);
  return ok_or_cuda();
}

extern "C" int eps_gather_rows(const void* src, int64_t src_stride_rows, void* dst, int rows,
                               int64_t d, int64_t offset_rows, void* stream) {
  if (rows <= 0) return EPS_OK;
  dim3 grid(unsigned((d / 8 + 255) / 256), unsigned(rows));
  count_launch(); rows_copy_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(src) + offset_rows * src_stride_rows, src_stride_rows,
      static_cast<uint16_t*>(dst), d, rows, d);
  return ok_or_cuda();
}

extern "C" int eps_scatter_rows(const void* src, void* dst, int64_t dst_stride_rows, int rows,
                                int64_t d, int64_t offset_rows, void* stream) {
  if (rows <= 0) return EPS_OK;
  dim3 grid(unsigned((d / 8 + 255) / 256), unsigned(rows));
  count_launch(); rows_copy_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(src), d,
      static_cast<uint16_t*>(dst) + offset_rows * dst_stride_rows, dst_stride_rows, rows, d);
  return ok_or_cuda();
}

extern "C" int eps_colsum_bf16(const void* x, float* out, int64_t rows, int64_t cols,
                               void* stream) {
  if (rows <= 0) return EPS_OK;
  const int64_t rpb = 256;
  dim3 grid(unsigned((cols + 255) / 256), unsigned((rows + rpb - 1) / rpb));
  count_launch(); colsum_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint16_t*>(x), out, rows, cols, rpb);
  return ok_or_cuda();
}

// Seeded synthetic data (the native trainer's dataset): element i of a
// stream is a function of (seed, i) only -- SplitMix64 finalisers of the
// counter, Box-Muller for N(0, 1) -- so any grid shape gives the same data.
namespace eps_k {
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__global__ void fill_normal_kernel(float* __restrict__ dst, int64_t n, uint64_t seed) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t a = mix64(seed + 0x9E3779B97F4A7C15ull * uint64_t(2 * i + 1));
    const uint64_t b = mix64(seed + 0x9E3779B97F4A7C15ull * uint64_t(2 * i + 2));
    const float u1 = (float(a >> 40) + 0.5f) * (1.0f / 16777216.0f);  // (0, 1)
    const float u2 = float(b >> 40) * (1.0f / 16777216.0f);
    dst[i] = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
  }
}
__global__ void fill_labels_kernel(int64_t* __restrict__ dst, int64_t n, int64_t classes,
                                   uint64_t seed) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = int64_t(mix64(seed + 0x9E3779B97F4A7C15ull * uint64_t(i + 1)) % uint64_t(classes));
}
}  // namespace eps_k

extern "C" int eps_fill_normal(float* dst, int64_t n, uint64_t seed, void* stream) {
  if (n <= 0) return EPS_OK;
  count_launch();
  eps_k::fill_normal_kernel<<<num_sms() * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(dst, n,
                                                                                          seed);
  return ok_or_cuda();
}

extern "C" int eps_fill_labels(int64_t* dst, int64_t n, int64_t classes, uint64_t seed,
                               void* stream) {
  if (n <= 0 || classes < 1) return n <= 0 ? EPS_OK : EPS_EINVAL;
  count_launch();
  eps_k::fill_labels_kernel<<<num_sms() * 2, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dst, n, classes, seed);
  return ok_or_cuda();
}

// Number of kernels this library has launched in the process so far.
extern "C" unsigned long long eps_launch_count(void) { return eps_k::launch_counter().load(); }
