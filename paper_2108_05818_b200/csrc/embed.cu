// GPU-placed embedding operator (the GPU branch of PatrickStar's device-aware
// operator placement, /root/reference/pkg/src/chunkstar/profiler.py:70-74,
// engine.py:214-219).  Same semantics as the host operator
// (host_embed.cpp, cs_embed_*_host), so a run's numerics do not depend on
// where the plan puts the embedding:
//
//   fwd: out[i,:] = round(float(wte[tok[i],:]) + float(wpe[i % S,:]))
//   bwd: gwte[v,:] = round(sum over tokens i with tok[i]==v, ascending i, of
//        float(dout[i,:])), zero for rows no token hits;
//        gwpe[s,:] = round(sum over b ascending of float(dout[b*S+s,:])).
//   bwd with accumulate (the tied LM head already wrote its dW over wte — the
//   grad overwrite of engine.py:177-190 — and the lookup adds to it, K4's
//   slot += src semantics fused in): gwte[v,:] = round(float(gwte[v,:]) +
//   float(round(sum))).
//
// The backward replaces a sort + segmented-reduce + scatter pipeline with ONE
// kernel: the caller passes the token positions stably sorted by token id
// (`order`) and each row's range in it (`row_start`, V+1 entries); CTA r < V
// owns vocabulary row r, CTA V+s owns position row s.  Each thread owns 8
// columns (one 128-bit vector), accumulates in fp32 registers and writes the
// row once: dout is read twice (rows via `order`, positions), gwte/gwpe are
// written once — HBM-bound, 2 x n*H*2 + (V+S)*H*2 bytes.

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "cs_internal.h"

namespace {

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
__device__ __forceinline__ void acc8(float* a, const uint4& w) {
  const uint32_t* u = reinterpret_cast<const uint32_t*>(&w);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    a[2 * k] = __fadd_rn(a[2 * k], to_f<DT>(u[k] & 0xffff));
    a[2 * k + 1] = __fadd_rn(a[2 * k + 1], to_f<DT>(u[k] >> 16));
  }
}

template <int DT>
__device__ __forceinline__ uint4 pack8(const float* a) {
  uint4 o;
  uint32_t* u = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    u[k] = (uint32_t)from_f<DT>(a[2 * k]) | ((uint32_t)from_f<DT>(a[2 * k + 1]) << 16);
  return o;
}

// grid-stride over vectors of the [n, H] output; 128-bit loads/stores
template <int DT>
__global__ void embed_fwd_kernel(const int64_t* __restrict__ tok, int64_t n, int S, int H,
                                 int64_t V, const uint4* __restrict__ wte,
                                 const uint4* __restrict__ wpe, uint4* __restrict__ out) {
  const int hv = H / 8;
  const int64_t total = n * hv;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / hv;
    const int c = (int)(q - i * hv);
    const int64_t t = tok[i];
    if (t < 0 || t >= V) {  // no out-of-range read: the row is NaN (loss NaN, step skipped)
      __stcs(out + q, make_uint4(0x7fff7fffu, 0x7fff7fffu, 0x7fff7fffu, 0x7fff7fffu));
      continue;
    }
    const uint4 a = __ldg(wte + t * hv + c);
    const uint4 b = __ldg(wpe + (i % S) * hv + c);
    // one fp32 add per element (no 0 + x first: keeps the sign of -0 + -0)
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a);
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b);
    float f[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      f[2 * k] = __fadd_rn(to_f<DT>(ua[k] & 0xffff), to_f<DT>(ub[k] & 0xffff));
      f[2 * k + 1] = __fadd_rn(to_f<DT>(ua[k] >> 16), to_f<DT>(ub[k] >> 16));
    }
    __stcs(out + q, pack8<DT>(f));
  }
}

// K4 semantics fused in (accumulate): slot = round(float(slot) + float(round(sum)))
template <int DT>
__device__ __forceinline__ uint4 add_rounded(const uint4& old, const float* a) {
  const uint4 r = pack8<DT>(a);
  const uint32_t* uo = reinterpret_cast<const uint32_t*>(&old);
  const uint32_t* ur = reinterpret_cast<const uint32_t*>(&r);
  float f[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    f[2 * k] = __fadd_rn(to_f<DT>(uo[k] & 0xffff), to_f<DT>(ur[k] & 0xffff));
    f[2 * k + 1] = __fadd_rn(to_f<DT>(uo[k] >> 16), to_f<DT>(ur[k] >> 16));
  }
  return pack8<DT>(f);
}

template <int DT>
__global__ void embed_bwd_kernel(const int64_t* __restrict__ order,
                                 const int64_t* __restrict__ row_start, int64_t n, int S,
                                 int64_t V, int H, const uint4* __restrict__ dout,
                                 uint4* __restrict__ gwte, uint4* __restrict__ gwpe,
                                 int accumulate) {
  const int hv = H / 8;
  const int c = threadIdx.x;
  if (c >= hv) return;
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  const int64_t r = blockIdx.x;
  if (r < V) {
    const int64_t k0 = row_start[r], k1 = row_start[r + 1];
    for (int64_t k = k0; k < k1; ++k) acc8<DT>(a, __ldcs(dout + order[k] * hv + c));
    uint4* dst = gwte + r * hv + c;
    *dst = accumulate ? add_rounded<DT>(*dst, a) : pack8<DT>(a);
  } else {
    const int64_t s = r - V;
    for (int64_t i = s; i < n; i += S) acc8<DT>(a, __ldcs(dout + i * hv + c));
    gwpe[s * hv + c] = pack8<DT>(a);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

extern "C" int cs_embed_fwd(const int64_t* tokens, int64_t n_tokens, int seq_len,
                            const void* wte, const void* wpe, int64_t vocab, int hidden,
                            void* out, int dtype, void* stream) {
  if (n_tokens < 0 || seq_len <= 0 || hidden <= 0 || hidden % 8 != 0 || vocab <= 0 ||
      (n_tokens > 0 && (!tokens || !wte || !wpe || !out)) ||
      (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_embed_fwd: invalid argument (hidden must be a multiple of 8)");
    return CS_EINVAL;
  }
  if (!aligned16(wte) || !aligned16(wpe) || !aligned16(out)) {
    cs::set_error("cs_embed_fwd: wte / wpe / out must be 16-byte aligned");
    return CS_EALIGN;
  }
  if (n_tokens == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t vecs = n_tokens * (hidden / 8);
  const int threads = 256;
  int64_t grid = (vecs + threads - 1) / threads;
  const int64_t cap = (int64_t)cs_num_sms() * 8;
  if (grid > cap) grid = cap;
  const auto* a = static_cast<const uint4*>(wte);
  const auto* b = static_cast<const uint4*>(wpe);
  auto* o = static_cast<uint4*>(out);
  if (dtype == CS_FP16)
    embed_fwd_kernel<CS_FP16><<<(unsigned)grid, threads, 0, s>>>(tokens, n_tokens, seq_len,
                                                                  hidden, vocab, a, b, o);
  else
    embed_fwd_kernel<CS_BF16><<<(unsigned)grid, threads, 0, s>>>(tokens, n_tokens, seq_len,
                                                                  hidden, vocab, a, b, o);
  cs::note_launches(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs::set_error("cs_embed_fwd: %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

extern "C" int cs_embed_bwd(const int64_t* order, const int64_t* row_start, int64_t n_tokens,
                            int seq_len, const void* dout, int64_t vocab, int hidden,
                            void* gwte, void* gwpe, int accumulate, int dtype, void* stream) {
  if (n_tokens < 0 || seq_len <= 0 || n_tokens % seq_len != 0 || vocab <= 0 || hidden <= 0 ||
      hidden % 8 != 0 || hidden / 8 > 1024 || !row_start || !gwte || !gwpe ||
      (n_tokens > 0 && (!order || !dout)) || (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_embed_bwd: invalid argument (n_tokens %% seq_len == 0, hidden %% 8 == 0,"
                  " hidden <= 8192)");
    return CS_EINVAL;
  }
  if (!aligned16(dout) || !aligned16(gwte) || !aligned16(gwpe)) {
    cs::set_error("cs_embed_bwd: dout / gwte / gwpe must be 16-byte aligned");
    return CS_EALIGN;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int threads = ((hidden / 8 + 31) / 32) * 32;
  const int64_t grid = vocab + seq_len;
  const auto* d = static_cast<const uint4*>(dout);
  auto* gw = static_cast<uint4*>(gwte);
  auto* gp = static_cast<uint4*>(gwpe);
  if (dtype == CS_FP16)
    embed_bwd_kernel<CS_FP16><<<(unsigned)grid, threads, 0, s>>>(
        order, row_start, n_tokens, seq_len, vocab, hidden, d, gw, gp, accumulate);
  else
    embed_bwd_kernel<CS_BF16><<<(unsigned)grid, threads, 0, s>>>(
        order, row_start, n_tokens, seq_len, vocab, hidden, d, gw, gp, accumulate);
  cs::note_launches(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs::set_error("cs_embed_bwd: %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}
