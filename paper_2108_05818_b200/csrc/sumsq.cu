// K2: sum of squares of the fp16/bf16 gradients, in a canonical order that
// does not depend on where each gradient lives (HBM or host DRAM) or on how
// the items are batched into launches -- so the global norm, the clip
// coefficient and the overflow decision are bit-identical for every
// placement of the same model (no reference counterpart: the simulator has
// no numerics).  The order is the specification below; the device kernels
// here, the host twin (host_adam.cpp cs_grad_sumsq_host) and the C oracle
// (oracle/cs_oracle.c or_grad_sumsq_item) all evaluate exactly it.
//
//   Item g[0..n), zero-padded to whole tiles of 8192 elements.  In tile t,
//   lane tau (0..255), group u (0..3), j (0..7) is element
//   e = 8192 t + (256 u + tau) 8 + j, x = float(g[e]).
//   a_j   = fold over u = 0..3 of  a_j = fl(a_j + fl(x * x)),  a_j = +0 first
//   L_tau = fl(fl(fl(a0 + a1) + fl(a2 + a3)) + fl(fl(a4 + a5) + fl(a6 + a7)))
//   warp w (lanes 32w .. 32w+31): for o = 16, 8, 4, 2, 1:
//           L_l = fl(L_l + L_(l xor o));   P[8 t + w] = L_(32 w)
//   double: D_s = fold over q = s, s + 8192, ... < Q of D_s + (double) P_q,
//           s = 0..8191; each group c of 256 strands (s = 256 c + r) is a tree:
//           for w = 128, 64, ..., 1: D_r = D_r + D_(r+w) (r < w), G_c = D_(256 c);
//           S(item) = fold over c = 0..31 of S + G_c
//   global: sumsq = (float) fold over the item slots 0..N-1 of T = T + S_i
//
// (fl = IEEE fp32 round-to-nearest; +0-padding adds exact zeros, so a tail
// is the same as skipping it.)  Device cost: one pass over the gradients
// (2 B/element; the next tile's four 128-bit loads per thread are in flight
// during the current tile's arithmetic),
// one fp32 partial per (tile, warp) -- 1/1024 of the gradient bytes -- and
// two tiny kernels.

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "cs_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kGroups = 4;
constexpr int64_t kTile = kThreads * kGroups * 8;  // 8192 elements
constexpr int kWarps = kThreads / 32;

struct TileBatch {
  const uint16_t* g[cs::kMaxBatch];
  int64_t n[cs::kMaxBatch];
  int64_t tile_start[cs::kMaxBatch + 1];  // exclusive prefix of tiles in this launch
  int64_t part_start[cs::kMaxBatch];      // first partial of each item (whole call)
  int count;
};

constexpr int kStrandGroups = 32;  // 32 x 256 strands per item

struct ItemBatch {
  int64_t part_start[cs::kMaxBatch];
  int64_t parts[cs::kMaxBatch];
  int slot[cs::kMaxBatch];
  int count;
};

template <int DT>
__device__ __forceinline__ float widen(uint16_t h) {
  if (DT == CS_FP16) return __half2float(__ushort_as_half(h));
  return __bfloat162float(__ushort_as_bfloat16(h));
}

__device__ __forceinline__ int find_item(const int64_t* start, int n, int64_t tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// the thread's 4 x 8 elements of one tile, zero-padded past the item's end
__device__ __forceinline__ void load_tile(const TileBatch& b, int64_t tile, uint4 (&v)[kGroups],
                                          int& k, int64_t& t) {
  k = find_item(b.tile_start, b.count, tile);
  const uint16_t* __restrict__ g = b.g[k];
  const int64_t n = b.n[k];
  t = tile - b.tile_start[k];
  const int64_t base = t * kTile;
  if (base + kTile <= n && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
#pragma unroll
    for (int u = 0; u < kGroups; ++u)
      v[u] = __ldcs(reinterpret_cast<const uint4*>(g + base + (int64_t)(u * kThreads +
                                                                         threadIdx.x) * 8));
  } else {  // last tile of an item (or unaligned)
#pragma unroll
    for (int u = 0; u < kGroups; ++u) {
      const int64_t e0 = base + (int64_t)(u * kThreads + threadIdx.x) * 8;
      uint16_t h[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) h[j] = e0 + j < n ? g[e0 + j] : (uint16_t)0;
      v[u] = make_uint4(h[0] | (uint32_t)h[1] << 16, h[2] | (uint32_t)h[3] << 16,
                        h[4] | (uint32_t)h[5] << 16, h[6] | (uint32_t)h[7] << 16);
    }
  }
}

// Grid-stride over the tiles of the launch; the next tile's loads are issued
// before the current tile's arithmetic and warp reduction (8 x 16 B in
// flight per thread), so the per-tile reduction does not stall the stream.
template <int DT>
__global__ void __launch_bounds__(kThreads)
sumsq_tiles_kernel(const __grid_constant__ TileBatch b, float* __restrict__ partials) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t total = b.tile_start[b.count];
  int64_t tile = blockIdx.x;
  if (tile >= total) return;
  uint4 v[kGroups];
  int k;
  int64_t t;
  load_tile(b, tile, v, k, t);
  while (true) {
    const int64_t next = tile + gridDim.x;
    uint4 vn[kGroups];
    int kn = 0;
    int64_t tn = 0;
    if (next < total) load_tile(b, next, vn, kn, tn);
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = 0.0f;
#pragma unroll
    for (int u = 0; u < kGroups; ++u) {
      const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float x = widen<DT>((uint16_t)(w[j >> 1] >> ((j & 1) * 16)));
        a[j] = __fadd_rn(a[j], __fmul_rn(x, x));
      }
    }
    float L = __fadd_rn(__fadd_rn(__fadd_rn(a[0], a[1]), __fadd_rn(a[2], a[3])),
                        __fadd_rn(__fadd_rn(a[4], a[5]), __fadd_rn(a[6], a[7])));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) L = __fadd_rn(L, __shfl_xor_sync(0xffffffffu, L, o));
    if (lane == 0) partials[b.part_start[k] + t * kWarps + warp] = L;
    if (next >= total) break;
    tile = next;
#pragma unroll
    for (int u = 0; u < kGroups; ++u) v[u] = vn[u];
    k = kn;
    t = tn;
  }
}

// grid (kStrandGroups, items): block c of item k folds strands 256 c + r
__global__ void __launch_bounds__(kThreads)
sumsq_strands_kernel(const __grid_constant__ ItemBatch b, const float* __restrict__ partials,
                     double* __restrict__ groups) {
  __shared__ double red[kThreads];
  const int k = blockIdx.y, c = blockIdx.x;
  const float* p = partials + b.part_start[k];
  double d = 0.0;
  constexpr int64_t kStride = (int64_t)kStrandGroups * kThreads;
  for (int64_t q = (int64_t)c * kThreads + threadIdx.x; q < b.parts[k]; q += kStride)
    d = __dadd_rn(d, (double)p[q]);
  red[threadIdx.x] = d;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] = __dadd_rn(red[threadIdx.x], red[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) groups[(int64_t)k * kStrandGroups + c] = red[0];
}

__global__ void sumsq_items_kernel(const __grid_constant__ ItemBatch b,
                                   const double* __restrict__ groups,
                                   double* __restrict__ item_sums) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= b.count) return;
  double s = 0.0;
  for (int c = 0; c < kStrandGroups; ++c) s = __dadd_rn(s, groups[(int64_t)k * kStrandGroups + c]);
  item_sums[b.slot[k]] = s;
}

__global__ void sumsq_total_kernel(const double* __restrict__ item_sums, int n,
                                   CsStepState* st) {
  double t = 0.0;
  for (int i = 0; i < n; ++i) t = __dadd_rn(t, item_sums[i]);
  st->sumsq = (float)t;
}

int64_t tiles_of(int64_t n) { return (n + kTile - 1) / kTile; }

int launch_error(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs::set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

}  // namespace

namespace {
int64_t partials_of(const CsGradItem* items, int n_items) {
  int64_t parts = 0;
  for (int i = 0; i < n_items; ++i) {
    if (items[i].n < 0) return -1;
    parts += tiles_of(items[i].n) * kWarps;
  }
  return parts;
}
// scratch layout: the fp32 (tile, warp) partials, then (8-byte aligned) one
// launch batch's double strand-group sums
int64_t groups_offset(int64_t parts) { return (parts + 1) & ~(int64_t)1; }
}  // namespace

extern "C" int64_t cs_sumsq_scratch(const CsGradItem* items, int n_items) {
  if (n_items < 0 || (n_items > 0 && !items)) return -1;
  const int64_t parts = partials_of(items, n_items);
  if (parts < 0) return -1;
  const int64_t batch = n_items < cs::kMaxBatch ? n_items : cs::kMaxBatch;
  return groups_offset(parts) + 2 * (int64_t)kStrandGroups * batch;
}

extern "C" int cs_grad_sumsq(const CsGradItem* items, int n_items, int dtype, const int* slots,
                             float* d_scratch, int64_t scratch_elems, double* d_item_sums,
                             void* stream) {
  if (n_items < 0 || (n_items > 0 && (!items || !d_item_sums)) ||
      (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_grad_sumsq: invalid argument");
    return CS_EINVAL;
  }
  if (n_items > CS_MAX_ITEMS) {
    cs::set_error("cs_grad_sumsq: %d items > CS_MAX_ITEMS", n_items);
    return CS_ETOOMANY;
  }
  const int64_t need = cs_sumsq_scratch(items, n_items);
  const int64_t parts_total = partials_of(items, n_items);
  if (need < 0) {
    cs::set_error("cs_grad_sumsq: an item has n < 0");
    return CS_EINVAL;
  }
  if (need > 0 && (!d_scratch || scratch_elems < need)) {
    cs::set_error("cs_grad_sumsq: scratch of %lld floats < %lld needed",
                  (long long)scratch_elems, (long long)need);
    return CS_EINVAL;
  }
  for (int i = 0; i < n_items; ++i) {
    if (items[i].n > 0 && !items[i].g16) {
      cs::set_error("cs_grad_sumsq: item %d has no data", i);
      return CS_EINVAL;
    }
    if ((reinterpret_cast<uintptr_t>(items[i].g16) & 1) != 0) {
      cs::set_error("cs_grad_sumsq: item %d misaligned", i);
      return CS_EALIGN;
    }
    if (slots && slots[i] < 0) {
      cs::set_error("cs_grad_sumsq: item %d has a negative slot", i);
      return CS_EINVAL;
    }
  }
  const int sms = cs_num_sms();
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int64_t part = 0;
  for (int first = 0; first < n_items;) {
    TileBatch tb;
    ItemBatch ib;
    tb.count = 0;
    ib.count = 0;
    int64_t tiles = 0;
    int i = first;
    // both batches are bounded: empty items take an item slot (their S is
    // written as 0) but no tile slot
    for (; i < n_items && tb.count < cs::kMaxBatch && ib.count < cs::kMaxBatch; ++i) {
      const CsGradItem& it = items[i];
      const int64_t nt = tiles_of(it.n);
      ib.part_start[ib.count] = part;
      ib.parts[ib.count] = nt * kWarps;
      ib.slot[ib.count] = slots ? slots[i] : i;
      ++ib.count;
      if (nt > 0) {
        tb.g[tb.count] = static_cast<const uint16_t*>(it.g16);
        tb.n[tb.count] = it.n;
        tb.tile_start[tb.count] = tiles;
        tb.part_start[tb.count] = part;
        ++tb.count;
        tiles += nt;
      }
      part += nt * kWarps;
    }
    first = i;
    tb.tile_start[tb.count] = tiles;
    if (tb.count > 0) {
      const int64_t cap = (int64_t)(sms > 0 ? sms : 148) * 8;
      const int grid = (int)(tiles < cap ? tiles : cap);
      if (dtype == CS_FP16)
        sumsq_tiles_kernel<CS_FP16><<<grid, kThreads, 0, s>>>(tb, d_scratch);
      else
        sumsq_tiles_kernel<CS_BF16><<<grid, kThreads, 0, s>>>(tb, d_scratch);
      cs::note_launches(1);
      if (int e = launch_error("cs_grad_sumsq")) return e;
    }
    double* groups = reinterpret_cast<double*>(d_scratch + groups_offset(parts_total));
    sumsq_strands_kernel<<<dim3(kStrandGroups, ib.count), kThreads, 0, s>>>(ib, d_scratch,
                                                                             groups);
    sumsq_items_kernel<<<(ib.count + 127) / 128, 128, 0, s>>>(ib, groups, d_item_sums);
    cs::note_launches(2);
    if (int e = launch_error("cs_grad_sumsq")) return e;
  }
  return 0;
}

extern "C" int cs_sumsq_finalize(const double* d_item_sums, int n_slots, CsStepState* d_state,
                                 void* stream) {
  if (n_slots < 0 || (n_slots > 0 && !d_item_sums) || !d_state) {
    cs::set_error("cs_sumsq_finalize: invalid argument");
    return CS_EINVAL;
  }
  sumsq_total_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(d_item_sums, n_slots,
                                                                     d_state);
  cs::note_launches(1);
  return launch_error("cs_sumsq_finalize");
}
