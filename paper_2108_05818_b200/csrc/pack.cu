// K3 grad pack, K4 grad accumulate, K5 fp32->fp16 cast+pack and K6 optimizer
// state birth for the chunk-managed step on B200 (sm_100a).
//
// K3/K4 realise the BWD "grad overwrite" of
// /root/reference/pkg/src/chunkstar/engine.py:177-190 (a parameter's fp16
// gradient is written over its own slot of the fp16 chunk); K5 realises the
// fp16 chunk materialisation of chunks.py:297-314; K6 the lazy optimizer
// state birth of engine.py:234-240.
//
// Chunk slots are packed gap-free (chunks.py:186-200), so a slot's element
// offset is arbitrary.  Each work item is split into 8-element units; when
// both the destination slot and the source are 16-byte aligned the unit is
// one 128-bit load/store per operand (the GPT layouts here are always
// aligned: every tensor is a multiple of H^2 elements), otherwise the unit
// falls back to element accesses.  Block tile = 256 threads x 2 units.

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>

#include "cs_internal.h"

namespace {

constexpr int kThreads = 256;
// 8-element units per thread and tile: the accumulate reads the slot before
// writing it and needs more reads in flight (4 units, all loads first: 0.85
// -> 0.99 of the copy peak); pack and cast keep 2 units issued in turn
// (0.94; the loads-first form measured 0.90-0.92 for them)
template <int OP>
__host__ __device__ constexpr int units() { return OP == 1 ? 4 : 2; }
template <int OP>
__host__ __device__ constexpr int64_t block_tile() { return (int64_t)kThreads * units<OP>() * 8; }

enum Op { kPack = 0, kAccumulate = 1, kCast = 2 };

// A/B switch for K6 (CS_MASTER_INIT_FUSED=1: the single fused kernel)
const bool g_master_init_split = [] {
  const char* e = getenv("CS_MASTER_INIT_FUSED");
  return !(e && e[0] == '1');
}();

struct PackBatch {
  void* dst[cs::kMaxBatch];
  const void* src[cs::kMaxBatch];
  int64_t n[cs::kMaxBatch];
  int64_t tile_start[cs::kMaxBatch + 1];
  uint8_t vec[cs::kMaxBatch];
  int count;
};

__device__ __forceinline__ int find_item(const int64_t* start, int n, int64_t tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int DT>
__device__ __forceinline__ float to_f(uint16_t h) {
  if (DT == CS_FP16) return __half2float(__ushort_as_half(h));
  return __bfloat162float(__ushort_as_bfloat16(h));
}
template <int DT>
__device__ __forceinline__ uint16_t from_f(float f) {
  if (DT == CS_FP16) return __half_as_ushort(__float2half_rn(f));
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

template <int DT>
__device__ __forceinline__ uint32_t pair_from_f(float a, float b) {
  return (uint32_t)from_f<DT>(a) | ((uint32_t)from_f<DT>(b) << 16);
}

// dst/src as 16-bit element arrays except src of kCast, which is fp32.
template <int OP, int DT>
__device__ __forceinline__ void unit_vec(uint16_t* dst, const void* src, int64_t e) {
  uint4* d = reinterpret_cast<uint4*>(dst + e);
  if (OP == kCast) {
    const float4* s = reinterpret_cast<const float4*>(static_cast<const float*>(src) + e);
    const float4 a = __ldcs(s), b = __ldcs(s + 1);
    __stcs(d, make_uint4(pair_from_f<DT>(a.x, a.y), pair_from_f<DT>(a.z, a.w),
                         pair_from_f<DT>(b.x, b.y), pair_from_f<DT>(b.z, b.w)));
    return;
  }
  const uint4 sv = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(src) + e));
  if (OP == kPack) {
    __stcs(d, sv);
    return;
  }
  const uint4 dv = *d;
  const uint32_t* sw = reinterpret_cast<const uint32_t*>(&sv);
  const uint32_t* dw = reinterpret_cast<const uint32_t*>(&dv);
  uint4 out;
  uint32_t* ow = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float lo = __fadd_rn(to_f<DT>(dw[k] & 0xffff), to_f<DT>(sw[k] & 0xffff));
    const float hi = __fadd_rn(to_f<DT>(dw[k] >> 16), to_f<DT>(sw[k] >> 16));
    ow[k] = pair_from_f<DT>(lo, hi);
  }
  __stcs(d, out);
}

template <int OP, int DT>
__device__ __forceinline__ void elem(uint16_t* dst, const void* src, int64_t e) {
  if (OP == kCast) {
    dst[e] = from_f<DT>(static_cast<const float*>(src)[e]);
  } else if (OP == kPack) {
    dst[e] = static_cast<const uint16_t*>(src)[e];
  } else {
    dst[e] = from_f<DT>(__fadd_rn(to_f<DT>(dst[e]), to_f<DT>(static_cast<const uint16_t*>(src)[e])));
  }
}

// Whole-tile vector path: every unit's loads are issued before any store
// (the slot and the source never alias, but the compiler cannot know), so a
// thread keeps kUnits x 16-32 B of reads in flight.
template <int OP, int DT>
__device__ __forceinline__ void tile_vec(uint16_t* __restrict__ dst, const void* __restrict__ src,
                                         int64_t base) {
  constexpr int kUnits = units<OP>();
  constexpr int W = OP == kCast ? 2 : 1;  // 16-byte source words per unit
  uint4 sv[kUnits][W];
  uint4 dv[kUnits];
#pragma unroll
  for (int u = 0; u < kUnits; ++u) {
    const int64_t e = base + (int64_t)(u * kThreads + threadIdx.x) * 8;
    if (OP == kCast) {
      const uint4* s4 = reinterpret_cast<const uint4*>(static_cast<const float*>(src) + e);
      sv[u][0] = __ldcs(s4);
      sv[u][W - 1] = __ldcs(s4 + (W - 1));
    } else {
      sv[u][0] = __ldcs(reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(src) + e));
    }
    if (OP == kAccumulate) dv[u] = *reinterpret_cast<const uint4*>(dst + e);
  }
#pragma unroll
  for (int u = 0; u < kUnits; ++u) {
    const int64_t e = base + (int64_t)(u * kThreads + threadIdx.x) * 8;
    uint4* d = reinterpret_cast<uint4*>(dst + e);
    if (OP == kPack) {
      __stcs(d, sv[u][0]);
    } else if (OP == kCast) {
      const float4 a = *reinterpret_cast<const float4*>(&sv[u][0]);
      const float4 b = *reinterpret_cast<const float4*>(&sv[u][W - 1]);
      __stcs(d, make_uint4(pair_from_f<DT>(a.x, a.y), pair_from_f<DT>(a.z, a.w),
                           pair_from_f<DT>(b.x, b.y), pair_from_f<DT>(b.z, b.w)));
    } else {
      const uint32_t* sw = reinterpret_cast<const uint32_t*>(&sv[u][0]);
      const uint32_t* dw = reinterpret_cast<const uint32_t*>(&dv[u]);
      uint4 out;
      uint32_t* ow = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float lo = __fadd_rn(to_f<DT>(dw[k] & 0xffff), to_f<DT>(sw[k] & 0xffff));
        const float hi = __fadd_rn(to_f<DT>(dw[k] >> 16), to_f<DT>(sw[k] >> 16));
        ow[k] = pair_from_f<DT>(lo, hi);
      }
      __stcs(d, out);
    }
  }
}

template <int OP, int DT>
__global__ void __launch_bounds__(kThreads) pack_kernel(const __grid_constant__ PackBatch b) {
  const int64_t total = b.tile_start[b.count];
  for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
    const int k = find_item(b.tile_start, b.count, tile);
    uint16_t* dst = static_cast<uint16_t*>(b.dst[k]);
    const void* src = b.src[k];
    const int64_t n = b.n[k];
    const int64_t base = (tile - b.tile_start[k]) * block_tile<OP>();
    if (OP == kAccumulate && b.vec[k] && base + block_tile<OP>() <= n) {
      tile_vec<OP, DT>(dst, src, base);
      continue;
    }
#pragma unroll
    for (int u = 0; u < units<OP>(); ++u) {
      const int64_t e = base + (int64_t)(u * kThreads + threadIdx.x) * 8;
      if (e >= n) continue;
      if (b.vec[k] && e + 8 <= n) {
        unit_vec<OP, DT>(dst, src, e);
      } else {
        const int64_t end = e + 8 < n ? e + 8 : n;
        for (int64_t i = e; i < end; ++i) elem<OP, DT>(dst, src, i);
      }
    }
  }
}

// K6: p32 = float(src) (src fp16/bf16/fp32, may be host-mapped), m = v = 0.
template <int SDT>
__global__ void __launch_bounds__(kThreads)
master_init_kernel(float* __restrict__ p32, float* __restrict__ m, float* __restrict__ v,
                   const void* __restrict__ src, int64_t n, int vec) {
  const int64_t stride = (int64_t)gridDim.x * kThreads * 4;
  for (int64_t e = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * 4; e < n; e += stride) {
    if (vec && e + 4 <= n) {
      float4 f;
      if (SDT == CS_FP32) {
        f = *reinterpret_cast<const float4*>(static_cast<const float*>(src) + e);
      } else {
        const uint2 w = *reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(src) + e);
        f = make_float4(to_f<SDT>(w.x & 0xffff), to_f<SDT>(w.x >> 16),
                        to_f<SDT>(w.y & 0xffff), to_f<SDT>(w.y >> 16));
      }
      __stcs(reinterpret_cast<float4*>(p32 + e), f);
      __stcs(reinterpret_cast<float4*>(m + e), make_float4(0.f, 0.f, 0.f, 0.f));
      __stcs(reinterpret_cast<float4*>(v + e), make_float4(0.f, 0.f, 0.f, 0.f));
    } else {
      for (int64_t i = e; i < e + 4 && i < n; ++i) {
        p32[i] = SDT == CS_FP32 ? static_cast<const float*>(src)[i]
                                : to_f<SDT>(static_cast<const uint16_t*>(src)[i]);
        m[i] = 0.0f;
        v[i] = 0.0f;
      }
    }
  }
}

// p32 = float(src), 4-element vectors (the caller checked alignment), four
// vectors per thread with every load issued before the stores
template <int SDT>
__global__ void __launch_bounds__(kThreads)
widen_kernel(float* __restrict__ p32, const void* __restrict__ src, int64_t n) {
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * kThreads * 4 * U;
  for (int64_t e0 = ((int64_t)blockIdx.x * kThreads * U + threadIdx.x) * 4; e0 < n;
       e0 += stride) {
    float4 f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * kThreads * 4;
      if (e + 4 <= n) {
        if (SDT == CS_FP32) {
          f[u] = __ldcs(reinterpret_cast<const float4*>(static_cast<const float*>(src) + e));
        } else {
          const uint2 w =
              __ldcs(reinterpret_cast<const uint2*>(static_cast<const uint16_t*>(src) + e));
          f[u] = make_float4(to_f<SDT>(w.x & 0xffff), to_f<SDT>(w.x >> 16),
                             to_f<SDT>(w.y & 0xffff), to_f<SDT>(w.y >> 16));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = e0 + (int64_t)u * kThreads * 4;
      if (e + 4 <= n) {
        __stcs(reinterpret_cast<float4*>(p32 + e), f[u]);
      } else {
        for (int64_t i = e; i < n; ++i)
          p32[i] = SDT == CS_FP32 ? static_cast<const float*>(src)[i]
                                  : to_f<SDT>(static_cast<const uint16_t*>(src)[i]);
      }
    }
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int grid_for(int64_t tiles) {
  const int sms = cs_num_sms();
  const int64_t cap = (int64_t)(sms > 0 ? sms : 148) * 8;
  return (int)(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs::set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

template <int OP>
int run_pack(const char* what, const CsPackItem* items, int n_items, int dtype, void* stream) {
  if (n_items < 0 || (n_items > 0 && !items) || (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("%s: invalid argument", what);
    return CS_EINVAL;
  }
  if (n_items > CS_MAX_ITEMS) {
    cs::set_error("%s: %d items > CS_MAX_ITEMS", what, n_items);
    return CS_ETOOMANY;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int first = 0; first < n_items;) {
    PackBatch b;
    b.count = 0;
    int64_t tiles = 0;
    int i = first;
    for (; i < n_items && b.count < cs::kMaxBatch; ++i) {
      const CsPackItem& it = items[i];
      if (it.n < 0 || it.offset < 0 || (it.n > 0 && (!it.chunk || !it.src))) {
        cs::set_error("%s: item %d invalid", what, i);
        return CS_EINVAL;
      }
      if (it.n == 0) continue;
      uint16_t* dst = static_cast<uint16_t*>(it.chunk) + it.offset;
      b.dst[b.count] = dst;
      b.src[b.count] = it.src;
      b.n[b.count] = it.n;
      b.vec[b.count] = aligned16(dst) && aligned16(it.src);
      b.tile_start[b.count] = tiles;
      tiles += (it.n + block_tile<OP>() - 1) / block_tile<OP>();
      ++b.count;
    }
    first = i;  // resume where this batch stopped (zero-length items took no slot)
    b.tile_start[b.count] = tiles;
    if (b.count == 0) continue;
    const int grid = grid_for(tiles);
    if (dtype == CS_FP16) pack_kernel<OP, CS_FP16><<<grid, kThreads, 0, s>>>(b);
    else pack_kernel<OP, CS_BF16><<<grid, kThreads, 0, s>>>(b);
    cs::note_launches(1);
    if (int e = check_launch(what)) return e;
  }
  return 0;
}

}  // namespace

extern "C" int cs_pack(const CsPackItem* items, int n_items, int dtype, int accumulate,
                       void* stream) {
  return accumulate ? run_pack<kAccumulate>("cs_pack(accumulate)", items, n_items, dtype, stream)
                    : run_pack<kPack>("cs_pack", items, n_items, dtype, stream);
}

extern "C" int cs_cast_pack(const CsPackItem* items, int n_items, int dtype, void* stream) {
  return run_pack<kCast>("cs_cast_pack", items, n_items, dtype, stream);
}

extern "C" int cs_master_init(float* p32, float* m, float* v, const void* src, int src_dtype,
                              int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!p32 || !m || !v || !src)) ||
      (src_dtype != CS_FP16 && src_dtype != CS_BF16 && src_dtype != CS_FP32)) {
    cs::set_error("cs_master_init: invalid argument");
    return CS_EINVAL;
  }
  if (n == 0) return 0;
  const uintptr_t need = src_dtype == CS_FP32 ? 15u : 7u;
  const int vec = aligned16(p32) && aligned16(m) && aligned16(v) &&
                  (reinterpret_cast<uintptr_t>(src) & need) == 0;
  const int grid = grid_for((n + kThreads * 4 - 1) / (kThreads * 4));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (vec && g_master_init_split) {
    // m = v = 0 as two write-only memsets and p32 = float(src) as one 1:2
    // stream: interleaving one read and three write streams in one kernel
    // ran at 0.82 of the copy peak (profiles/r02/microbench_c5.jsonl)
    cudaError_t e = cudaMemsetAsync(m, 0, (size_t)n * sizeof(float), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(v, 0, (size_t)n * sizeof(float), s);
    if (e != cudaSuccess) {
      cs::set_error("cs_master_init: memset failed: %s", cudaGetErrorString(e));
      return (int)e;
    }
    if (src_dtype == CS_FP16)
      widen_kernel<CS_FP16><<<grid, kThreads, 0, s>>>(p32, src, n);
    else if (src_dtype == CS_BF16)
      widen_kernel<CS_BF16><<<grid, kThreads, 0, s>>>(p32, src, n);
    else
      widen_kernel<CS_FP32><<<grid, kThreads, 0, s>>>(p32, src, n);
    cs::note_launches(1);
    return check_launch("cs_master_init");
  }
  if (src_dtype == CS_FP16)
    master_init_kernel<CS_FP16><<<grid, kThreads, 0, s>>>(p32, m, v, src, n, vec);
  else if (src_dtype == CS_BF16)
    master_init_kernel<CS_BF16><<<grid, kThreads, 0, s>>>(p32, m, v, src, n, vec);
  else
    master_init_kernel<CS_FP32><<<grid, kThreads, 0, s>>>(p32, m, v, src, n, vec);
  cs::note_launches(1);
  return check_launch("cs_master_init");
}
