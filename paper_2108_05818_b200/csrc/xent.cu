// Fused LM-head cross entropy for the GPT step on B200 (sm_100a).
//
// Forward: one CTA per row of the fp16/bf16 logits [rows, vocab]; each thread
// keeps an online (max, sum-of-exp) over 128-bit loads, the CTA reduces the
// pairs, and writes loss_row = logsumexp - logit[target] and the row's
// logsumexp (fp32).  Backward: dlogits = (softmax - onehot(target)) * dloss *
// scale, written over the logits buffer in place (the logits are dead after
// the loss), fp32 math, round-to-nearest narrowing.
//
// Traffic: forward reads the logits once (2 B/elem); backward reads and
// writes them once (4 B/elem) — versus the unfused fp32 upcast + log_softmax
// + nll chain (~24 B/elem).

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <math.h>

#include "cs_internal.h"

namespace {

constexpr int kThreads = 512;
constexpr float kLog2e = 1.4426950408889634f;

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

// 2^x on the MUFU with flush-to-zero: one instruction instead of exp2f's
// range-handling wrapper (compare, two scalings).  Every argument here is
// <= 0, so the only difference is that terms below 2^-126 become 0, which
// cannot change a sum of at least 1 (forward) or an fp16 gradient.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void online(float x, float& m, float& s) {
  if (x > m) {
    s = s * ex2((m - x) * kLog2e) + 1.0f;
    m = x;
  } else {
    s += ex2((x - m) * kLog2e);
  }
}

// eight values at once: one max, at most one rescale, eight exp-adds (no
// per-element divergent branch)
template <int DT>
__device__ __forceinline__ void online8(const uint4& w, float& m, float& s) {
  const uint32_t* u = reinterpret_cast<const uint32_t*>(&w);
  float v[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[2 * k] = to_f<DT>(u[k] & 0xffff);
    v[2 * k + 1] = to_f<DT>(u[k] >> 16);
  }
  float mx = v[0];
#pragma unroll
  for (int k = 1; k < 8; ++k) mx = fmaxf(mx, v[k]);
  if (mx > m) {
    s *= ex2((m - mx) * kLog2e);
    m = mx;
  }
  if (m == -INFINITY) return;
  const float mb = m * kLog2e;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += ex2(fmaf(v[k], kLog2e, -mb));
}

__device__ __forceinline__ void merge(float& m, float& s, float m2, float s2) {
  const float mx = fmaxf(m, m2);
  if (mx == -INFINITY) return;
  s = s * ex2((m - mx) * kLog2e) + s2 * ex2((m2 - mx) * kLog2e);
  m = mx;
}

template <int DT>
__global__ void __launch_bounds__(kThreads)
xent_fwd_kernel(const uint16_t* __restrict__ logits, const int64_t* __restrict__ targets,
                int64_t vocab, float* __restrict__ loss_rows, float* __restrict__ lse_rows) {
  const int64_t row = blockIdx.x;
  const uint16_t* x = logits + row * vocab;
  float m = -INFINITY, s = 0.0f;
  const bool vec = (vocab % 8) == 0;
  if (vec) {
    const uint4* xv = reinterpret_cast<const uint4*>(x);
    const int64_t nv = vocab / 8;
    int64_t i = threadIdx.x;
    for (; i + 3 * kThreads < nv; i += 4 * kThreads) {  // four 128-bit loads in flight
      const uint4 w0 = __ldcs(xv + i);
      const uint4 w1 = __ldcs(xv + i + kThreads);
      const uint4 w2 = __ldcs(xv + i + 2 * kThreads);
      const uint4 w3 = __ldcs(xv + i + 3 * kThreads);
      online8<DT>(w0, m, s);
      online8<DT>(w1, m, s);
      online8<DT>(w2, m, s);
      online8<DT>(w3, m, s);
    }
    for (; i + kThreads < nv; i += 2 * kThreads) {
      const uint4 w0 = __ldcs(xv + i);
      const uint4 w1 = __ldcs(xv + i + kThreads);
      online8<DT>(w0, m, s);
      online8<DT>(w1, m, s);
    }
    if (i < nv) online8<DT>(__ldcs(xv + i), m, s);
  } else {
    for (int64_t i = threadIdx.x; i < vocab; i += kThreads) online(to_f<DT>(x[i]), m, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
    merge(m, s, m2, s2);
  }
  __shared__ float sm[kThreads / 32], ss[kThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sm[warp] = m;
    ss[warp] = s;
  }
  __syncthreads();
  if (warp == 0) {
    m = lane < kThreads / 32 ? sm[lane] : -INFINITY;
    s = lane < kThreads / 32 ? ss[lane] : 0.0f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, s, o);
      merge(m, s, m2, s2);
    }
    if (lane == 0) {
      const float lse = m + logf(s);
      lse_rows[row] = lse;
      const int64_t t = targets[row];  // out of range: no read, NaN loss (step skipped)
      loss_rows[row] = (t >= 0 && t < vocab) ? lse - to_f<DT>(x[t]) : __int_as_float(0x7fc00000);
    }
  }
}

template <int DT>
__global__ void __launch_bounds__(kThreads)
xent_bwd_kernel(uint16_t* __restrict__ logits, const int64_t* __restrict__ targets,
                int64_t vocab, const float* __restrict__ lse_rows,
                const float* __restrict__ dloss, float scale) {
  const int64_t row = blockIdx.x;
  uint16_t* x = logits + row * vocab;
  const float lse = lse_rows[row];
  const int64_t tgt = targets[row];
  // an out-of-range target poisons its row's gradient, so the step's
  // overflow check skips the update instead of training on a wrong target
  const float g = (tgt >= 0 && tgt < vocab) ? *dloss * scale : __int_as_float(0x7fc00000);
  if ((vocab % 8) == 0) {
    uint4* xv = reinterpret_cast<uint4*>(x);
    const int64_t nv = vocab / 8;
    for (int64_t i = threadIdx.x; i < nv; i += kThreads) {
      uint4 w = __ldcs(xv + i);
      uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t c = i * 8 + 2 * k;
        float a = ex2((to_f<DT>(u[k] & 0xffff) - lse) * kLog2e) - (c == tgt ? 1.0f : 0.0f);
        float b = ex2((to_f<DT>(u[k] >> 16) - lse) * kLog2e) - (c + 1 == tgt ? 1.0f : 0.0f);
        u[k] = (uint32_t)from_f<DT>(a * g) | ((uint32_t)from_f<DT>(b * g) << 16);
      }
      __stcs(xv + i, w);
    }
  } else {
    for (int64_t c = threadIdx.x; c < vocab; c += kThreads) {
      const float p = ex2((to_f<DT>(x[c]) - lse) * kLog2e) - (c == tgt ? 1.0f : 0.0f);
      x[c] = from_f<DT>(p * g);
    }
  }
}

int check(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs::set_error("%s: launch failed: %s", what, cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

}  // namespace

extern "C" int cs_xent_fwd(const void* logits, const int64_t* targets, int64_t rows,
                           int64_t vocab, int dtype, float* loss_rows, float* lse_rows,
                           void* stream) {
  if (!logits || !targets || !loss_rows || !lse_rows || rows < 0 || vocab <= 0 ||
      rows > 0x7fffffff || (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_xent_fwd: invalid argument");
    return CS_EINVAL;
  }
  if (rows == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint16_t* x = static_cast<const uint16_t*>(logits);
  if (dtype == CS_FP16)
    xent_fwd_kernel<CS_FP16><<<(unsigned)rows, kThreads, 0, s>>>(x, targets, vocab, loss_rows, lse_rows);
  else
    xent_fwd_kernel<CS_BF16><<<(unsigned)rows, kThreads, 0, s>>>(x, targets, vocab, loss_rows, lse_rows);
  cs::note_launches(1);
  return check("cs_xent_fwd");
}

extern "C" int cs_xent_bwd(void* logits, const int64_t* targets, const float* lse_rows,
                           const float* dloss, float scale, int64_t rows, int64_t vocab,
                           int dtype, void* stream) {
  if (!logits || !targets || !lse_rows || !dloss || rows < 0 || vocab <= 0 ||
      rows > 0x7fffffff || (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_xent_bwd: invalid argument");
    return CS_EINVAL;
  }
  if (rows == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint16_t* x = static_cast<uint16_t*>(logits);
  if (dtype == CS_FP16)
    xent_bwd_kernel<CS_FP16><<<(unsigned)rows, kThreads, 0, s>>>(x, targets, vocab, lse_rows, dloss, scale);
  else
    xent_bwd_kernel<CS_BF16><<<(unsigned)rows, kThreads, 0, s>>>(x, targets, vocab, lse_rows, dloss, scale);
  cs::note_launches(1);
  return check("cs_xent_bwd");
}
