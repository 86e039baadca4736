// K1 fused chunk Adam and the device-side step scalars for the chunk-managed
// training step on B200 (sm_100a); K2 (sum of squares) is in sumsq.cu.
//
// K1 realises Engine._adam_event's per-position update
// (/root/reference/pkg/src/chunkstar/engine.py:225-272): it reads the fp16
// grad chunk and the fp32 master/momentum/variance chunks of a position and
// writes fp32 state plus the new fp16 params back into the same fp16 chunk,
// in one pass — 28 B/element of HBM traffic, the algorithmic minimum.
//
// Layout/access: every item is the used prefix [0, n) of one chunk payload
// (chunk bases are allocation-aligned, tensors are packed gap-free, so the
// prefix is one contiguous run).  A block tile is 256 threads x 4 groups x 4
// elements = 4096 elements; in each group a warp touches 32 consecutive
// 4-element groups, so every load/store instruction is a fully coalesced
// 256 B (fp16, 64-bit/lane) or 512 B (fp32, 128-bit/lane) transaction.  All
// 16 groups' loads of a thread are issued before any math (memory-level
// parallelism ~ 14 x 16 B in flight per thread).  Data is touched exactly
// once, so loads/stores carry the streaming (evict-first) policy.  The grid
// is persistent: #SMs x resident blocks, striding over the block tiles of all
// items of the launch (one launch updates every GPU-placed position).

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <math.h>
#include <stdlib.h>

#include "cs_internal.h"

namespace {

constexpr int kThreads = 256;
// K1 data-movement variants, bit-identical results.  Selected once per
// process (CS_ADAM_VARIANT, default kAdamDefault):
//   0  SIMT register-tiled (this file; also the fallback for items whose
//      streams are not 16-byte aligned)
//   1  TMA-staged three-role pipeline (adam_tma.cu), the default
// The round-1 sweep over 25 tilings is recorded in profiles/r01/k1_variants.md.
constexpr int kAdamSimtGroups = 4;   // 4-element groups per thread per block tile
constexpr int kAdamVariantCount = 2;
constexpr int kAdamDefault = 1;

struct AdamBatch {
  CsAdamItem item[cs::kMaxBatch];
  int64_t tile_start[cs::kMaxBatch + 1];  // exclusive prefix of block tiles
  int n;
  float b2, c1, c2, eps, wd, decay;  // scalars formed in double, rounded once
  int adamw;
};

// ---- 16-bit storage helpers (4 elements = 64 bits) -------------------------

template <int DT>
__device__ __forceinline__ float4 widen4(uint2 w);
template <>
__device__ __forceinline__ float4 widen4<CS_FP16>(uint2 w) {
  float2 a = __half22float2(*reinterpret_cast<__half2*>(&w.x));
  float2 b = __half22float2(*reinterpret_cast<__half2*>(&w.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
template <>
__device__ __forceinline__ float4 widen4<CS_BF16>(uint2 w) {
  float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w.x));
  float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

template <int DT>
__device__ __forceinline__ uint2 narrow4(float4 f);
template <>
__device__ __forceinline__ uint2 narrow4<CS_FP16>(float4 f) {
  __half2 a = __floats2half2_rn(f.x, f.y), b = __floats2half2_rn(f.z, f.w);
  return make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
}
template <>
__device__ __forceinline__ uint2 narrow4<CS_BF16>(float4 f) {
  __nv_bfloat162 a = __floats2bfloat162_rn(f.x, f.y), b = __floats2bfloat162_rn(f.z, f.w);
  return make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
}

template <int DT>
__device__ __forceinline__ float widen1(uint16_t h) {
  if (DT == CS_FP16) return __half2float(__ushort_as_half(h));
  return __bfloat162float(__ushort_as_bfloat16(h));
}
template <int DT>
__device__ __forceinline__ uint16_t narrow1(float f) {
  if (DT == CS_FP16) return __half_as_ushort(__float2half_rn(f));
  return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// ---- the Adam element update (every op individually rounded) --------------

struct AdamConsts {
  float grad_scale, neg_step_size, sqrt_bc2;
  float b2, c1, c2, eps, wd, decay;
  bool adamw;
};

// Association of torch.optim.Adam's CPU single-tensor path (lerp_, mul_ +
// addcmul_, addcdiv_), IEEE sqrt/div; see include/chunkstar_b200.h.
__device__ __forceinline__ void adam1(float g16, float& p, float& m, float& v,
                                      const AdamConsts& c) {
  float g = __fmul_rn(g16, c.grad_scale);
  if (c.wd != 0.0f) {
    if (c.adamw) p = __fmul_rn(p, c.decay);
    else g = __fmaf_rn(c.wd, p, g);
  }
  m = __fmaf_rn(c.c1, __fsub_rn(g, m), m);
  v = __fmaf_rn(__fmul_rn(c.c2, g), g, __fmul_rn(v, c.b2));
  const float denom = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), c.sqrt_bc2), c.eps);
  p = __fadd_rn(p, __fdiv_rn(__fmul_rn(c.neg_step_size, m), denom));
}

// A skipped step (non-finite gradients) leaves p32 / m / v untouched, but the
// 16-bit chunk holds the step's gradients (the grad overwrite of
// engine.py:177-190): every element gets its unchanged parameter back,
// p16 = round(p32).  Grid-stride over all items; rare, so plain loads.
template <int DT>
__device__ void restore_params(const CsAdamItem* items, int n_items, const CsStepState* st) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int i = 0; i < n_items; ++i) {
    const CsAdamItem it = items[i];
    uint16_t* q16 = static_cast<uint16_t*>(it.p16);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < it.n; e += stride) {
      const float f = it.p32[e];
      q16[e] = DT == CS_FP16 ? __half_as_ushort(__float2half_rn(f))
                             : __bfloat16_as_ushort(__float2bfloat16_rn(f));
    }
  }
}

__device__ __forceinline__ int find_item(const int64_t* start, int n, int64_t tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <int DT, int G, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
adam_chunks_kernel(const __grid_constant__ AdamBatch b, const CsStepState* __restrict__ st) {
  constexpr int kTile = kThreads * G * 4;
  if (st->skip) {  // non-finite gradients: no update, parameters restored
    restore_params<DT>(b.item, b.n, st);
    return;
  }
  AdamConsts c;
  c.grad_scale = st->grad_scale;
  c.neg_step_size = -st->step_size;
  c.sqrt_bc2 = st->sqrt_bc2;
  c.b2 = b.b2;
  c.c1 = b.c1;
  c.c2 = b.c2;
  c.eps = b.eps;
  c.wd = b.wd;
  c.decay = b.decay;
  c.adamw = b.adamw != 0;

  const int64_t total = b.tile_start[b.n];
  for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
    const int k = find_item(b.tile_start, b.n, tile);
    const CsAdamItem it = b.item[k];
    const int64_t base = (tile - b.tile_start[k]) * kTile;
    uint16_t* __restrict__ p16 = static_cast<uint16_t*>(it.p16);

    if (base + kTile <= it.n) {  // full tile: vector path
      uint2 g[G];
      float4 p[G], m[G], v[G];
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int64_t e = base + (int64_t)(u * kThreads + threadIdx.x) * 4;
        g[u] = __ldcs(reinterpret_cast<const uint2*>(p16 + e));
        p[u] = __ldcs(reinterpret_cast<const float4*>(it.p32 + e));
        m[u] = __ldcs(reinterpret_cast<const float4*>(it.m + e));
        v[u] = __ldcs(reinterpret_cast<const float4*>(it.v + e));
      }
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const float4 gf = widen4<DT>(g[u]);
        adam1(gf.x, p[u].x, m[u].x, v[u].x, c);
        adam1(gf.y, p[u].y, m[u].y, v[u].y, c);
        adam1(gf.z, p[u].z, m[u].z, v[u].z, c);
        adam1(gf.w, p[u].w, m[u].w, v[u].w, c);
        const int64_t e = base + (int64_t)(u * kThreads + threadIdx.x) * 4;
        __stcs(reinterpret_cast<float4*>(it.p32 + e), p[u]);
        __stcs(reinterpret_cast<float4*>(it.m + e), m[u]);
        __stcs(reinterpret_cast<float4*>(it.v + e), v[u]);
        __stcs(reinterpret_cast<uint2*>(p16 + e), narrow4<DT>(p[u]));
      }
    } else {  // the last, partial tile of an item
      for (int u = 0; u < G; ++u) {
        const int64_t e0 = base + (int64_t)(u * kThreads + threadIdx.x) * 4;
        for (int64_t e = e0; e < e0 + 4 && e < it.n; ++e) {
          float pp = it.p32[e], mm = it.m[e], vv = it.v[e];
          adam1(widen1<DT>(p16[e]), pp, mm, vv, c);
          it.p32[e] = pp;
          it.m[e] = mm;
          it.v[e] = vv;
          p16[e] = narrow1<DT>(pp);
        }
      }
    }
  }
}

__global__ void step_state_init_kernel(CsStepState* st, float loss_scale) {
  st->beta1_pow = 1.0;
  st->beta2_pow = 1.0;
  st->step = 0;
  st->loss_scale = loss_scale;
  st->good_steps = 0;
  st->grad_scale = __fdiv_rn(1.0f, loss_scale);
  st->step_size = 0.0f;
  st->sqrt_bc2 = 1.0f;
  st->skip = 0;
  st->grad_norm = 0.0f;
  st->sumsq = 0.0f;
}

// One thread: skip decision, clip coefficient, bias corrections and the
// dynamic loss-scale update, all from the device-resident sumsq.
__global__ void adam_prepare_kernel(CsStepState* st, CsAdamHyper h, float max_norm,
                                    float growth, float backoff, int32_t interval,
                                    int32_t dynamic_scale) {
  const float sumsq = st->sumsq;
  const float ls = st->loss_scale;
  if (!isfinite(sumsq)) {
    st->skip = 1;
    st->grad_norm = sumsq;
    if (dynamic_scale) {
      st->loss_scale = __fmul_rn(ls, backoff);
      st->good_steps = 0;
    }
    return;
  }
  const float norm = __fdiv_rn(__fsqrt_rn(sumsq), ls);
  float clip = 1.0f;
  if (max_norm > 0.0f) clip = fminf(__fdiv_rn(max_norm, __fadd_rn(norm, 1e-6f)), 1.0f);
  st->grad_scale = __fmul_rn(__fdiv_rn(1.0f, ls), clip);
  st->grad_norm = norm;
  st->skip = 0;
  st->step += 1;
  st->beta1_pow = __dmul_rn(st->beta1_pow, h.beta1);
  st->beta2_pow = __dmul_rn(st->beta2_pow, h.beta2);
  st->step_size = (float)__ddiv_rn(h.lr, __dsub_rn(1.0, st->beta1_pow));
  st->sqrt_bc2 = (float)__dsqrt_rn(__dsub_rn(1.0, st->beta2_pow));
  if (dynamic_scale && ++st->good_steps >= interval) {
    st->loss_scale = __fmul_rn(ls, growth);
    st->good_steps = 0;
  }
}

// ---- host side ---------------------------------------------------------------

int g_num_sms = 0;
int g_adam_variant = -1;
int g_adam_blocks_per_sm = 0;

typedef void (*AdamKernel)(const AdamBatch, const CsStepState*);

int adam_variant() {
  if (g_adam_variant < 0) {
    const char* e = getenv("CS_ADAM_VARIANT");
    const int v = e ? atoi(e) : kAdamDefault;
    g_adam_variant = (v >= 0 && v < kAdamVariantCount) ? v : kAdamDefault;
  }
  return g_adam_variant;
}

int num_sms() {
  if (g_num_sms > 0) return g_num_sms;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return -1;
  return g_num_sms;
}

bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

int launch_error(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs::set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

}  // namespace

int cs_adam_chunks_tma(const CsAdamItem* items, int n_items, int dtype, const CsAdamHyper* h,
                       const CsStepState* d_state, void* stream);

extern "C" int cs_num_sms(void) { return num_sms(); }

extern "C" int cs_adam_variant(int v) {
  if (v >= 0 && v < kAdamVariantCount && v != adam_variant()) {
    g_adam_variant = v;
    g_adam_blocks_per_sm = 0;  // occupancy is per kernel
  }
  return adam_variant();
}


extern "C" int cs_adam_chunks(const CsAdamItem* items, int n_items, int dtype,
                              const CsAdamHyper* hyper, const CsStepState* d_state,
                              void* stream) {
  if (n_items < 0 || (n_items > 0 && !items) || !hyper || !d_state ||
      (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_adam_chunks: invalid argument");
    return CS_EINVAL;
  }
  if (n_items > CS_MAX_ITEMS) {
    cs::set_error("cs_adam_chunks: %d items > CS_MAX_ITEMS", n_items);
    return CS_ETOOMANY;
  }
  const int sms = num_sms();
  if (sms <= 0) {
    cs::set_error("cs_adam_chunks: no CUDA device");
    return CS_EINVAL;
  }
  if (adam_variant() == 1) {
    bool ok16 = true;
    for (int i = 0; i < n_items && ok16; ++i)
      ok16 = aligned(items[i].p16, 16) && aligned(items[i].p32, 16) && aligned(items[i].m, 16) &&
             aligned(items[i].v, 16);
    if (ok16) {
      for (int i = 0; i < n_items; ++i) {
        const CsAdamItem& it = items[i];
        if (it.n < 0 || (it.n > 0 && (!it.p16 || !it.p32 || !it.m || !it.v))) {
          cs::set_error("cs_adam_chunks: item %d invalid", i);
          return CS_EINVAL;
        }
      }
      return cs_adam_chunks_tma(items, n_items, dtype, hyper, d_state, stream);
    }
    // bulk copies need 16-byte aligned streams: the SIMT kernel takes the rest
  }
  const int64_t tile_elems = (int64_t)kThreads * kAdamSimtGroups * 4;
  AdamKernel kern = dtype == CS_FP16 ? adam_chunks_kernel<CS_FP16, kAdamSimtGroups, 1>
                                     : adam_chunks_kernel<CS_BF16, kAdamSimtGroups, 1>;
  if (g_adam_blocks_per_sm == 0) {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kThreads, 0);
    g_adam_blocks_per_sm = nb > 0 ? nb : 1;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int first = 0; first < n_items;) {
    AdamBatch b;
    b.n = 0;
    int64_t tiles = 0;
    int i = first;
    for (; i < n_items && b.n < cs::kMaxBatch; ++i) {
      const CsAdamItem& it = items[i];
      if (it.n < 0 || (it.n > 0 && (!it.p16 || !it.p32 || !it.m || !it.v))) {
        cs::set_error("cs_adam_chunks: item %d invalid", i);
        return CS_EINVAL;
      }
      if (!aligned(it.p16, 8) || !aligned(it.p32, 16) || !aligned(it.m, 16) ||
          !aligned(it.v, 16)) {
        cs::set_error("cs_adam_chunks: item %d misaligned (p16 needs 8 B, fp32 16 B)", i);
        return CS_EALIGN;
      }
      if (it.n == 0) continue;  // takes no batch slot
      b.item[b.n] = it;
      b.tile_start[b.n] = tiles;
      tiles += (it.n + tile_elems - 1) / tile_elems;
      ++b.n;
    }
    first = i;  // resume where this batch stopped
    b.tile_start[b.n] = tiles;
    if (b.n == 0) continue;
    b.b2 = (float)hyper->beta2;
    b.c1 = (float)(1.0 - hyper->beta1);
    b.c2 = (float)(1.0 - hyper->beta2);
    b.eps = (float)hyper->eps;
    b.wd = (float)hyper->weight_decay;
    b.decay = (float)(1.0 - hyper->lr * hyper->weight_decay);
    b.adamw = hyper->adamw;
    const int64_t grid64 = (int64_t)sms * g_adam_blocks_per_sm;
    const int grid = (int)(tiles < grid64 ? tiles : grid64);
    kern<<<grid, kThreads, 0, s>>>(b, d_state);
    cs::note_launches(1);
    if (int e = launch_error("cs_adam_chunks")) return e;
  }
  return 0;
}

extern "C" int cs_step_state_init(CsStepState* d_state, float init_loss_scale, void* stream) {
  if (!d_state || !(init_loss_scale > 0.0f)) {
    cs::set_error("cs_step_state_init: invalid argument");
    return CS_EINVAL;
  }
  step_state_init_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_state,
                                                                        init_loss_scale);
  cs::note_launches(1);
  return launch_error("cs_step_state_init");
}

extern "C" int cs_adam_prepare(CsStepState* d_state, const CsAdamHyper* hyper,
                               float max_grad_norm, float growth_factor,
                               float backoff_factor, int32_t growth_interval,
                               int32_t dynamic_scale, void* stream) {
  if (!d_state || !hyper || (dynamic_scale && growth_interval <= 0)) {
    cs::set_error("cs_adam_prepare: invalid argument");
    return CS_EINVAL;
  }
  adam_prepare_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
      d_state, *hyper, max_grad_norm, growth_factor, backoff_factor, growth_interval,
      dynamic_scale);
  cs::note_launches(1);
  return launch_error("cs_adam_prepare");
}
