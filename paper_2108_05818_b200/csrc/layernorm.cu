// Non-affine LayerNorm with the residual-stream gradient folded into its
// backward (model side of the GPT step on B200).
//
// In a pre-LN block the residual stream h feeds both the LayerNorm and the
// next residual add, so autograd normally sums two gradients for h with an
// extra elementwise pass.  Here the LN function passes h through as the
// residual and its backward produces dh = LN_bwd(dy) + d_residual in one pass.
//
// One warp per row, 128-bit loads, fp32 statistics (two-pass in registers:
// mean, then centred variance), eps inside the rsqrt like torch.

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "cs_internal.h"

namespace {

constexpr int kWarps = 8;       // rows per CTA

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

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int DT>
__device__ __forceinline__ float lo(uint32_t w) { return to_f<DT>(w & 0xffff); }
template <int DT>
__device__ __forceinline__ float hi(uint32_t w) { return to_f<DT>(w >> 16); }

// rows stay in registers as packed 128-bit words; each pass converts on the fly
template <int DT, int NV>
__global__ void __launch_bounds__(kWarps * 32)
ln_fwd_kernel(const uint16_t* __restrict__ x, uint16_t* __restrict__ y,
              float* __restrict__ mean_out, float* __restrict__ rstd_out, int64_t rows, int H,
              float eps) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * H);
  uint4 w[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    w[i] = __ldcs(xr + i * 32 + lane);
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&w[i]);
#pragma unroll
    for (int k = 0; k < 4; ++k) s += lo<DT>(u[k]) + hi<DT>(u[k]);
  }
  const float mean = warp_sum(s) / H;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&w[i]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float a = lo<DT>(u[k]) - mean, b = hi<DT>(u[k]) - mean;
      q += a * a + b * b;
    }
  }
  const float rstd = rsqrtf(warp_sum(q) / H + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + row * H);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    uint4 o;
    const uint32_t* u = reinterpret_cast<const uint32_t*>(&w[i]);
    uint32_t* ou = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      ou[k] = (uint32_t)from_f<DT>((lo<DT>(u[k]) - mean) * rstd) |
              ((uint32_t)from_f<DT>((hi<DT>(u[k]) - mean) * rstd) << 16);
    yr[i * 32 + lane] = o;
  }
  if (lane == 0) {
    mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

// dx = rstd * (dy - mean(dy) - xhat * mean(dy * xhat)) + dres
template <int DT, int NV>
__global__ void __launch_bounds__(kWarps * 32)
ln_bwd_kernel(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ x,
              const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
              const uint16_t* __restrict__ dres, uint16_t* __restrict__ dx, int64_t rows, int H) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (row >= rows) return;
  const float mean = mean_in[row], rstd = rstd_in[row];
  const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * H);
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * H);
  uint4 a[NV], b[NV];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    a[i] = __ldcs(dyr + i * 32 + lane);
    b[i] = __ldcs(xr + i * 32 + lane);
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a[i]);
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b[i]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float g0 = lo<DT>(ua[k]), g1 = hi<DT>(ua[k]);
      s1 += g0 + g1;
      s2 += g0 * ((lo<DT>(ub[k]) - mean) * rstd) + g1 * ((hi<DT>(ub[k]) - mean) * rstd);
    }
  }
  const float m1 = warp_sum(s1) / H, m2 = warp_sum(s2) / H;
  const uint4* rr = dres ? reinterpret_cast<const uint4*>(dres + row * H) : nullptr;
  uint4* dxr = reinterpret_cast<uint4*>(dx + row * H);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    uint4 r = make_uint4(0u, 0u, 0u, 0u);
    if (rr) r = __ldcs(rr + i * 32 + lane);
    const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a[i]);
    const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b[i]);
    const uint32_t* ur = reinterpret_cast<const uint32_t*>(&r);
    uint4 o;
    uint32_t* ou = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float x0 = (lo<DT>(ub[k]) - mean) * rstd, x1 = (hi<DT>(ub[k]) - mean) * rstd;
      const float d0 = rstd * (lo<DT>(ua[k]) - m1 - x0 * m2) + (rr ? lo<DT>(ur[k]) : 0.f);
      const float d1 = rstd * (hi<DT>(ua[k]) - m1 - x1 * m2) + (rr ? hi<DT>(ur[k]) : 0.f);
      ou[k] = (uint32_t)from_f<DT>(d0) | ((uint32_t)from_f<DT>(d1) << 16);
    }
    dxr[i * 32 + lane] = o;
  }
}

template <int DT, int NV>
void launch_fwd(const void* x, void* y, float* mean, float* rstd, int64_t rows, int H, float eps,
                cudaStream_t s) {
  const unsigned grid = (unsigned)((rows + kWarps - 1) / kWarps);
  ln_fwd_kernel<DT, NV><<<grid, kWarps * 32, 0, s>>>(static_cast<const uint16_t*>(x),
                                                      static_cast<uint16_t*>(y), mean, rstd,
                                                      rows, H, eps);
}

template <int DT, int NV>
void launch_bwd(const void* dy, const void* x, const float* mean, const float* rstd,
                const void* dres, void* dx, int64_t rows, int H, cudaStream_t s) {
  const unsigned grid = (unsigned)((rows + kWarps - 1) / kWarps);
  ln_bwd_kernel<DT, NV><<<grid, kWarps * 32, 0, s>>>(
      static_cast<const uint16_t*>(dy), static_cast<const uint16_t*>(x), mean, rstd,
      static_cast<const uint16_t*>(dres), static_cast<uint16_t*>(dx), rows, H);
}

// dispatch on H / 256 (elements per lane / 8) for the supported widths
template <int DT>
bool dispatch_fwd(const void* x, void* y, float* m, float* r, int64_t rows, int H, float eps,
                  cudaStream_t s) {
  switch (H / 256) {
    case 1: launch_fwd<DT, 1>(x, y, m, r, rows, H, eps, s); return true;
    case 2: launch_fwd<DT, 2>(x, y, m, r, rows, H, eps, s); return true;
    case 4: launch_fwd<DT, 4>(x, y, m, r, rows, H, eps, s); return true;
    case 8: launch_fwd<DT, 8>(x, y, m, r, rows, H, eps, s); return true;
    case 9: launch_fwd<DT, 9>(x, y, m, r, rows, H, eps, s); return true;
    case 12: launch_fwd<DT, 12>(x, y, m, r, rows, H, eps, s); return true;
    case 16: launch_fwd<DT, 16>(x, y, m, r, rows, H, eps, s); return true;
    default: return false;
  }
}

template <int DT>
bool dispatch_bwd(const void* dy, const void* x, const float* m, const float* r,
                  const void* dres, void* dx, int64_t rows, int H, cudaStream_t s) {
  switch (H / 256) {
    case 1: launch_bwd<DT, 1>(dy, x, m, r, dres, dx, rows, H, s); return true;
    case 2: launch_bwd<DT, 2>(dy, x, m, r, dres, dx, rows, H, s); return true;
    case 4: launch_bwd<DT, 4>(dy, x, m, r, dres, dx, rows, H, s); return true;
    case 8: launch_bwd<DT, 8>(dy, x, m, r, dres, dx, rows, H, s); return true;
    case 9: launch_bwd<DT, 9>(dy, x, m, r, dres, dx, rows, H, s); return true;
    case 12: launch_bwd<DT, 12>(dy, x, m, r, dres, dx, rows, H, s); return true;
    case 16: launch_bwd<DT, 16>(dy, x, m, r, dres, dx, rows, H, s); return true;
    default: return false;
  }
}

bool supported(int H) {
  const int v = H / 256;
  return H % 256 == 0 && (v == 1 || v == 2 || v == 4 || v == 8 || v == 9 || v == 12 || v == 16);
}

}  // namespace

extern "C" int cs_layernorm_supported(int H) { return supported(H) ? 1 : 0; }

extern "C" int cs_layernorm_fwd(const void* x, void* y, float* mean, float* rstd, int64_t rows,
                                int H, float eps, int dtype, void* stream) {
  if (!x || !y || !mean || !rstd || rows < 0 || !supported(H) ||
      (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_layernorm_fwd: invalid argument (H must be 256 x {1,2,4,8,9,12,16})");
    return CS_EINVAL;
  }
  if (rows == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == CS_FP16) dispatch_fwd<CS_FP16>(x, y, mean, rstd, rows, H, eps, s);
  else dispatch_fwd<CS_BF16>(x, y, mean, rstd, rows, H, eps, s);
  cs::note_launches(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs::set_error("cs_layernorm_fwd: %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}

extern "C" int cs_layernorm_bwd(const void* dy, const void* x, const float* mean,
                                const float* rstd, const void* dres, void* dx, int64_t rows,
                                int H, int dtype, void* stream) {
  if (!dy || !x || !mean || !rstd || !dx || rows < 0 || !supported(H) ||
      (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_layernorm_bwd: invalid argument");
    return CS_EINVAL;
  }
  if (rows == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == CS_FP16) dispatch_bwd<CS_FP16>(dy, x, mean, rstd, dres, dx, rows, H, s);
  else dispatch_bwd<CS_BF16>(dy, x, mean, rstd, dres, dx, rows, H, s);
  cs::note_launches(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs::set_error("cs_layernorm_bwd: %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}
