// K1 fused chunk Adam, TMA-staged (sm_100a) -- the default K1.
//
// Same arithmetic as adam_chunks_kernel (adam.cu, bit-identical results);
// different data movement.  A persistent CTA per SM runs a STAGES-deep ring
// of shared-memory tiles with three roles:
//
//   producer (one lane)   : wait empty[s] -> mbarrier expect_tx(14·T bytes) ->
//                           cp.async.bulk global->shared of the tile's g16,
//                           p32, m, v (4 bulk copies, complete_tx on full[s])
//   consumers (CW warps)  : wait full[s] -> Adam in shared memory, in place
//                           (p16 written over the g16 slot) -> fence.proxy.async
//                           -> arrive computed[s] and move on to the next tile
//   store warp (one lane) : wait computed[s] -> cp.async.bulk shared->global of
//                           p16, p32, m, v, commit; once the bulk reads of the
//                           previous group are done -> arrive empty[s]
//
// Loads for STAGES tiles are always in flight while the consumers compute and
// the stores drain asynchronously, so the SM keeps ~STAGES·14·T bytes of read
// traffic outstanding with a handful of registers.  Tiles are T elements of
// one item (the used prefix of one chunk position); each item's last n % 8
// elements (bulk copies move multiples of 16 B) are updated by the consumer
// warps straight from global memory.

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "cs_internal.h"

namespace cs_tma {

struct Batch {
  CsAdamItem item[cs::kMaxBatch];
  int64_t tile_start[cs::kMaxBatch + 1];
  int n;
  float b2, c1, c2, eps, wd, decay;
  int adamw;
};

__device__ __forceinline__ uint32_t saddr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(saddr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(saddr(dst)),
      "l"(src), "r"(bytes), "r"(saddr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(saddr(src)), "r"(bytes)
               : "memory");
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

struct Consts {
  float gs, nss, sb, b2, c1, c2, eps, wd, decay;
  double rsb;  // RN_f64(1 / sb), for div_by_sb
  bool adamw;
};

// x / sb rounded to float, bit-identical to __fdiv_rn(x, sb), in three
// instructions instead of the IEEE division sequence (MUFU.RCP, FCHK, Newton
// FFMAs and the slow-path branch).  Why exact: q = RN_f64(x * RN_f64(1/sb)) is
// within ~2^-52 relative of x/sb.  Rounding q to float gives RN_f32(x/sb)
// unless x/sb lies within 2^-52 relative of a float rounding midpoint M.
// x/sb is never exactly on M: M has a 25-bit odd significand, so sb * M needs
// more than 24 bits and cannot equal the float x.  Nor can it be closer to M
// than 2^-49 relative: x - sb*M is a nonzero multiple of ulp(sb)*ulp(M)/2.
// The quotient here is sqrt(v)/sqrt(1 - beta2^t): zero, a normal float, or
// inf/nan, which pass through the conversions unchanged.  No subnormal or
// overflowing results: sqrt(v) >= 2^-75 for v > 0, and sb lies in
// [sqrt(1 - beta2), 1].  tests/test_kernels_gpu.py checks every variant
// against the oracle's IEEE division, at the full bench size too.
__device__ __forceinline__ float div_by_sb(float x, const Consts& c) {
  return __double2float_rn(__dmul_rn((double)x, c.rsb));
}

// same op sequence and rounding as adam.cu's adam1 (torch.optim.Adam association)
__device__ __forceinline__ void adam1(float g16, float& p, float& m, float& v, const Consts& c) {
  float g = __fmul_rn(g16, c.gs);
  if (c.wd != 0.0f) {
    if (c.adamw) p = __fmul_rn(p, c.decay);
    else g = __fmaf_rn(c.wd, p, g);
  }
  m = __fmaf_rn(c.c1, __fsub_rn(g, m), m);
  v = __fmaf_rn(__fmul_rn(c.c2, g), g, __fmul_rn(v, c.b2));
  const float denom = __fadd_rn(div_by_sb(__fsqrt_rn(v), c), c.eps);
  p = __fadd_rn(p, __fdiv_rn(__fmul_rn(c.nss, m), denom));
}

__device__ __forceinline__ int find_item(const int64_t* start, int n, int64_t tile) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Three-role variant: producer warp (bulk loads), 8 consumer warps (math),
// store warp (bulk stores).  Consumers publish a finished stage by arriving on
// computed[s] (count = all consumer threads) and move straight on; only the
// store warp waits for the bulk reads before freeing the stage.
template <int DT, int T, int STAGES, int CW, int U = 1>
__global__ void __launch_bounds__(CW * 32 + 64)
adam_tma3_kernel(const __grid_constant__ Batch b, const CsStepState* __restrict__ st) {
  constexpr int kConsumerWarps = CW;
  constexpr int kConsumers = CW * 32;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int kStageBytes = T * 14;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* computed = empty + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (st->skip) {  // non-finite gradients: no update, p16 = round(p32) restored
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int i = 0; i < b.n; ++i) {
      const CsAdamItem it = b.item[i];
      uint16_t* q16 = static_cast<uint16_t*>(it.p16);
      for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < it.n; e += stride)
        q16[e] = from_f<DT>(it.p32[e]);
    }
    return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&computed[s], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t total = b.tile_start[b.n];
  if (warp >= kConsumerWarps) {
    if (lane != 0) return;
    const bool producer = warp == kConsumerWarps;
    int64_t k = 0;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x, ++k) {
      const int s = (int)(k % STAGES);
      const uint32_t phase = (uint32_t)((k / STAGES) & 1);
      const int i = find_item(b.tile_start, b.n, tile);
      const CsAdamItem it = b.item[i];
      const int64_t e0 = (tile - b.tile_start[i]) * T;
      const int64_t nvec = it.n & ~(int64_t)7;
      const int len = (int)((nvec - e0) < T ? (nvec - e0) : T);
      unsigned char* base = smem + s * kStageBytes;
      if (producer) {
        mbar_wait(&empty[s], phase ^ 1u);
        mbar_expect_tx(&full[s], (uint32_t)len * 14u);
        bulk_load(base, static_cast<const uint16_t*>(it.p16) + e0, len * 2, &full[s]);
        bulk_load(base + T * 2, it.p32 + e0, len * 4, &full[s]);
        bulk_load(base + T * 6, it.m + e0, len * 4, &full[s]);
        bulk_load(base + T * 10, it.v + e0, len * 4, &full[s]);
      } else {
        mbar_wait(&computed[s], phase);
        bulk_store(static_cast<uint16_t*>(it.p16) + e0, base, len * 2);
        bulk_store(it.p32 + e0, base + T * 2, len * 4);
        bulk_store(it.m + e0, base + T * 6, len * 4);
        bulk_store(it.v + e0, base + T * 10, len * 4);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // keep this stage's stores in flight; the previous stage's are read
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        if (k > 0) mbar_arrive(&empty[(int)((k - 1) % STAGES)]);
      }
    }
    if (!producer) {
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      if (k > 0) mbar_arrive(&empty[(int)((k - 1) % STAGES)]);
    }
    return;
  }
  Consts c;
  c.gs = st->grad_scale;
  c.nss = -st->step_size;
  c.sb = st->sqrt_bc2;
  c.rsb = __ddiv_rn(1.0, (double)c.sb);
  c.b2 = b.b2;
  c.c1 = b.c1;
  c.c2 = b.c2;
  c.eps = b.eps;
  c.wd = b.wd;
  c.decay = b.decay;
  c.adamw = b.adamw != 0;
  const int t = threadIdx.x;
  int64_t k = 0;
  for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x, ++k) {
    const int s = (int)(k % STAGES);
    const uint32_t phase = (uint32_t)((k / STAGES) & 1);
    const int i = find_item(b.tile_start, b.n, tile);
    const int64_t e0 = (tile - b.tile_start[i]) * T;
    const int64_t nvec = b.item[i].n & ~(int64_t)7;
    const int len = (int)((nvec - e0) < T ? (nvec - e0) : T);
    unsigned char* base = smem + s * kStageBytes;
    uint16_t* g16 = reinterpret_cast<uint16_t*>(base);
    float* p = reinterpret_cast<float*>(base + T * 2);
    float* m = reinterpret_cast<float*>(base + T * 6);
    float* v = reinterpret_cast<float*>(base + T * 10);
    mbar_wait(&full[s], phase);
    if (U == 1) {
      for (int e = t * 4; e < len; e += kConsumers * 4) {
        uint2 gw = *reinterpret_cast<uint2*>(g16 + e);
        float4 pp = *reinterpret_cast<float4*>(p + e);
        float4 mm = *reinterpret_cast<float4*>(m + e);
        float4 vv = *reinterpret_cast<float4*>(v + e);
        adam1(to_f<DT>(gw.x & 0xffff), pp.x, mm.x, vv.x, c);
        adam1(to_f<DT>(gw.x >> 16), pp.y, mm.y, vv.y, c);
        adam1(to_f<DT>(gw.y & 0xffff), pp.z, mm.z, vv.z, c);
        adam1(to_f<DT>(gw.y >> 16), pp.w, mm.w, vv.w, c);
        *reinterpret_cast<float4*>(p + e) = pp;
        *reinterpret_cast<float4*>(m + e) = mm;
        *reinterpret_cast<float4*>(v + e) = vv;
        gw.x = (uint32_t)from_f<DT>(pp.x) | ((uint32_t)from_f<DT>(pp.y) << 16);
        gw.y = (uint32_t)from_f<DT>(pp.z) | ((uint32_t)from_f<DT>(pp.w) << 16);
        *reinterpret_cast<uint2*>(g16 + e) = gw;
      }
    } else {
      // U groups of 4 per thread per pass: every smem load issued before the
      // math, U*4 independent update chains for the schedulers (low-clock ILP)
      for (int e0 = t * 4; e0 < len; e0 += kConsumers * 4 * U) {
        uint2 gw[U];
        float4 pp[U], mm[U], vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * kConsumers * 4;
          if (e < len) {
            gw[u] = *reinterpret_cast<uint2*>(g16 + e);
            pp[u] = *reinterpret_cast<float4*>(p + e);
            mm[u] = *reinterpret_cast<float4*>(m + e);
            vv[u] = *reinterpret_cast<float4*>(v + e);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * kConsumers * 4;
          if (e < len) {
            adam1(to_f<DT>(gw[u].x & 0xffff), pp[u].x, mm[u].x, vv[u].x, c);
            adam1(to_f<DT>(gw[u].x >> 16), pp[u].y, mm[u].y, vv[u].y, c);
            adam1(to_f<DT>(gw[u].y & 0xffff), pp[u].z, mm[u].z, vv[u].z, c);
            adam1(to_f<DT>(gw[u].y >> 16), pp[u].w, mm[u].w, vv[u].w, c);
            *reinterpret_cast<float4*>(p + e) = pp[u];
            *reinterpret_cast<float4*>(m + e) = mm[u];
            *reinterpret_cast<float4*>(v + e) = vv[u];
            uint2 o;
            o.x = (uint32_t)from_f<DT>(pp[u].x) | ((uint32_t)from_f<DT>(pp[u].y) << 16);
            o.y = (uint32_t)from_f<DT>(pp[u].z) | ((uint32_t)from_f<DT>(pp[u].w) << 16);
            *reinterpret_cast<uint2*>(g16 + e) = o;
          }
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive(&computed[s]);
  }
  for (int i = blockIdx.x; i < b.n; i += gridDim.x) {
    const CsAdamItem it = b.item[i];
    const int64_t e = (it.n & ~(int64_t)7) + t;
    if (t < 8 && e < it.n) {
      uint16_t* q16 = static_cast<uint16_t*>(it.p16);
      float pp = it.p32[e], mm = it.m[e], vv = it.v[e];
      adam1(to_f<DT>(q16[e]), pp, mm, vv, c);
      it.p32[e] = pp;
      it.m[e] = mm;
      it.v[e] = vv;
      q16[e] = from_f<DT>(pp);
    }
  }
}

template <int DT, int T, int STAGES, int CW, int U = 1>
int launch(const CsAdamItem* items, int n_items, const CsAdamHyper* h,
           const CsStepState* d_state, cudaStream_t stream, int ctas_per_sm) {
  constexpr int kSmem = STAGES * T * 14 + 3 * STAGES * 8;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(adam_tma3_kernel<DT, T, STAGES, CW, U>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    configured = true;
  }
  const int sms = cs_num_sms();
  for (int first = 0; first < n_items;) {
    Batch b;
    b.n = 0;
    int64_t tiles = 0;
    int i = first;
    for (; i < n_items && b.n < cs::kMaxBatch; ++i) {
      const CsAdamItem& it = items[i];
      if (it.n == 0) continue;  // takes no batch slot
      b.item[b.n] = it;
      b.tile_start[b.n] = tiles;
      tiles += ((it.n & ~(int64_t)7) + T - 1) / T;
      ++b.n;
    }
    first = i;  // resume where this batch stopped (zero-length items took no slot)
    b.tile_start[b.n] = tiles;
    if (b.n == 0) continue;
    b.b2 = (float)h->beta2;
    b.c1 = (float)(1.0 - h->beta1);
    b.c2 = (float)(1.0 - h->beta2);
    b.eps = (float)h->eps;
    b.wd = (float)h->weight_decay;
    b.decay = (float)(1.0 - h->lr * h->weight_decay);
    b.adamw = h->adamw;
    int64_t grid = (int64_t)sms * ctas_per_sm;
    const int64_t need = tiles > b.n ? tiles : b.n;  // every item's tail needs a CTA
    if (grid > need) grid = need;
    adam_tma3_kernel<DT, T, STAGES, CW, U><<<(int)grid, CW * 32 + 64, kSmem, stream>>>(b, d_state);
    cs::note_launches(1);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      cs::set_error("cs_adam_chunks(tma): launch failed: %s", cudaGetErrorString(e));
      return (int)e;
    }
  }
  return 0;
}

}  // namespace cs_tma

// Entry used by cs_adam_chunks for the TMA-staged K1 (variant 1, see adam.cu):
// 5120-element tiles x 3 stages (215 KB of the 227 KB of shared memory),
// 20 consumer warps, 1 CTA per SM.  The A/B sweep over tile size, stage count
// and consumer warps that chose it is in profiles/r01/k1_variants.md.
int cs_adam_chunks_tma(const CsAdamItem* items, int n_items, int dtype, const CsAdamHyper* h,
                       const CsStepState* d_state, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == CS_FP16)
    return cs_tma::launch<CS_FP16, 5120, 3, 20>(items, n_items, h, d_state, s, 1);
  return cs_tma::launch<CS_BF16, 5120, 3, 20>(items, n_items, h, d_state, s, 1);
}
