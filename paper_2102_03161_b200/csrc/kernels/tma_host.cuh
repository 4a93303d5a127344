// Host-side TMA tensor-map construction (cuTensorMapEncodeTiled through the
// runtime's driver entry point, so the library needs no -lcuda).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <unordered_map>

namespace eps_k {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Tensor-map cache.  cuTensorMapEncodeTiled costs ~1-2 us of host time and a
// training step encodes ~600 maps (4 per GEMM): at the small micro-batches of
// a deep pipeline the host would otherwise fall behind the device.  A map is
// a pure function of its encode arguments (pointer, dims, strides, box,
// swizzle), so identical requests return the cached copy.  One cache per host
// thread (one thread drives one GPU); cleared when it grows past 16K entries.
struct MapKey {
  const void* base;
  uint64_t dims[3], strides[2];
  uint32_t box[3];
  uint32_t rank, dtype, swz;
  bool operator==(const MapKey& o) const { return std::memcmp(this, &o, sizeof(MapKey)) == 0; }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(&k);
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof(MapKey) / 8; ++i) h = (h ^ w[i]) * 1099511628211ull;
    return size_t(h);
  }
};
inline bool encode_cached(CUtensorMap* map, CUtensorMapDataType dtype, uint32_t rank,
                          const void* base, const cuuint64_t* dims, const cuuint64_t* strides,
                          const cuuint32_t* box, CUtensorMapSwizzle swz) {
  static_assert(sizeof(MapKey) % 8 == 0, "MapKey hashing");
  MapKey k;
  std::memset(&k, 0, sizeof(k));
  k.base = base;
  for (uint32_t i = 0; i < rank; ++i) {
    k.dims[i] = dims[i];
    k.box[i] = box[i];
    if (i + 1 < rank) k.strides[i] = strides[i];
  }
  k.rank = rank;
  k.dtype = uint32_t(dtype);
  k.swz = uint32_t(swz);
  thread_local std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  auto it = cache.find(k);
  if (it != cache.end()) {
    *map = it->second;
    return true;
  }
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return false;
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  if (fn(map, dtype, rank, const_cast<void*>(base), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 16384) cache.clear();
  cache.emplace(k, *map);
  return true;
}

// 2D tensor map: inner dim `inner` (contiguous), outer dim `outer` with a
// row pitch of `ld` elements; zero fill for out-of-bounds boxes.
inline bool make_map(CUtensorMap* map, const void* base, bool f32, int64_t inner, int64_t outer,
                     int64_t ld, int box_inner, int box_outer, CUtensorMapSwizzle swz) {
  const int esize = f32 ? 4 : 2;
  const cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * esize};
  const cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_outer)};
  return encode_cached(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                       2, base, dims, strides, box, swz);
}

// 3D bf16 map over [outer][mid][inner] with pitches ld_mid (elements between
// consecutive mid rows) and ld_outer (elements between outer slices): rows
// past `mid` inside one outer slice are zero-filled, not read from the next.
inline bool make_map_3d(CUtensorMap* map, const void* base, int64_t inner, int64_t mid,
                        int64_t outer, int64_t ld_mid, int64_t ld_outer, int box_inner,
                        int box_mid, CUtensorMapSwizzle swz) {
  const cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(mid), cuuint64_t(outer)};
  const cuuint64_t strides[2] = {cuuint64_t(ld_mid) * 2, cuuint64_t(ld_outer) * 2};
  const cuuint32_t box[3] = {cuuint32_t(box_inner), cuuint32_t(box_mid), 1u};
  return encode_cached(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, swz);
}

inline int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

}  // namespace eps_k

#include <atomic>
#include <cstdlib>
#include <utility>

namespace eps_k {

// PDL on (1, default) / off (0): EPS_PDL in the environment or eps_pdl_mode().
inline std::atomic<int>& pdl_mode() {
  static std::atomic<int> mode{[] {
    const char* e = std::getenv("EPS_PDL");
    return e == nullptr ? 1 : std::atoi(e);
  }()};
  return mode;
}

// cudaLaunchKernelEx with programmatic stream serialization (the kernel must
// call pdl_wait() before reading or writing global memory) and an optional
// cluster width.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     int cluster_x, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl_mode().load() != 0) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = unsigned(cluster_x);
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = unsigned(n);
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace eps_k
