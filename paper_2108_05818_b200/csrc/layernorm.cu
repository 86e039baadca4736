// Non-affine LayerNorm with the residual-stream gradient folded into its
// backward (model side of the GPT step on B200).
//
// In a pre-LN block the residual stream h feeds both the LayerNorm and the
// next residual add, so autograd normally sums two gradients for h with an
// extra elementwise pass.  Here the LN function passes h through as the
// residual and its backward produces dh = LN_bwd(dy) + d_residual in one pass.
//
// Forward: one warp per row, 128-bit loads, fp32 statistics (two-pass in registers:
// mean, then centred variance), eps inside the rsqrt like torch.

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "cs_internal.h"

namespace {

constexpr int kWarps = 4;       // rows per CTA (4: 5 CTAs = 20 rows in flight per SM at 90 regs; 8: 16)

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
//
// One row per CTA of H/8 threads: each thread owns one 128-bit vector of dy,
// x and dres, all three loads issued before the reduction (the warp-per-row
// form held 64 elements/lane in 150 registers = 8 warps/SM and exposed the
// dres load after the reduction; this form runs ~40 registers, up to 8 rows
// in flight per SM).  Block reduction: warp shuffles, then one smem pass.
template <int DT>
__global__ void __launch_bounds__(1024)
ln_bwd_row_kernel(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ x,
                  const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
                  const uint16_t* __restrict__ dres, uint16_t* __restrict__ dx, int H) {
  __shared__ float red[2][32];
  const int64_t row = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nwarps = blockDim.x >> 5;
  const float mean = mean_in[row], rstd = rstd_in[row];
  const int64_t base = row * (int64_t)H / 8 + t;
  const uint4 a = __ldcs(reinterpret_cast<const uint4*>(dy) + base);
  const uint4 b = __ldcs(reinterpret_cast<const uint4*>(x) + base);
  uint4 r = make_uint4(0u, 0u, 0u, 0u);
  if (dres) r = __ldcs(reinterpret_cast<const uint4*>(dres) + base);
  const uint32_t* ua = reinterpret_cast<const uint32_t*>(&a);
  const uint32_t* ub = reinterpret_cast<const uint32_t*>(&b);
  const uint32_t* ur = reinterpret_cast<const uint32_t*>(&r);
  float xh[8], g[8];
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    g[2 * k] = lo<DT>(ua[k]);
    g[2 * k + 1] = hi<DT>(ua[k]);
    xh[2 * k] = (lo<DT>(ub[k]) - mean) * rstd;
    xh[2 * k + 1] = (hi<DT>(ub[k]) - mean) * rstd;
    s1 += g[2 * k] + g[2 * k + 1];
    s2 += g[2 * k] * xh[2 * k] + g[2 * k + 1] * xh[2 * k + 1];
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (lane == 0) {
    red[0][warp] = s1;
    red[1][warp] = s2;
  }
  __syncthreads();
  if (warp == 0) {
    float v1 = lane < nwarps ? red[0][lane] : 0.f;
    float v2 = lane < nwarps ? red[1][lane] : 0.f;
    v1 = warp_sum(v1);
    v2 = warp_sum(v2);
    if (lane == 0) {
      red[0][0] = v1;
      red[1][0] = v2;
    }
  }
  __syncthreads();
  const float m1 = red[0][0] / H, m2 = red[1][0] / H;
  uint4 o;
  uint32_t* ou = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float d0 = rstd * (g[2 * k] - m1 - xh[2 * k] * m2) + lo<DT>(ur[k]);
    const float d1 = rstd * (g[2 * k + 1] - m1 - xh[2 * k + 1] * m2) + hi<DT>(ur[k]);
    ou[k] = (uint32_t)from_f<DT>(d0) | ((uint32_t)from_f<DT>(d1) << 16);
  }
  reinterpret_cast<uint4*>(dx)[base] = o;
}

template <int DT, int NV>
void launch_fwd(const void* x, void* y, float* mean, float* rstd, int64_t rows, int H, float eps,
                cudaStream_t s) {
  const unsigned grid = (unsigned)((rows + kWarps - 1) / kWarps);
  ln_fwd_kernel<DT, NV><<<grid, kWarps * 32, 0, s>>>(static_cast<const uint16_t*>(x),
                                                      static_cast<uint16_t*>(y), mean, rstd,
                                                      rows, H, eps);
}

template <int DT>
void launch_bwd(const void* dy, const void* x, const float* mean, const float* rstd,
                const void* dres, void* dx, int64_t rows, int H, cudaStream_t s) {
  ln_bwd_row_kernel<DT><<<(unsigned)rows, H / 8, 0, s>>>(
      static_cast<const uint16_t*>(dy), static_cast<const uint16_t*>(x), mean, rstd,
      static_cast<const uint16_t*>(dres), static_cast<uint16_t*>(dx), H);
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
  if (dtype == CS_FP16) launch_bwd<CS_FP16>(dy, x, mean, rstd, dres, dx, rows, H, s);
  else launch_bwd<CS_BF16>(dy, x, mean, rstd, dres, dx, rows, H, s);
  cs::note_launches(1);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cs::set_error("cs_layernorm_bwd: %s", cudaGetErrorString(e));
    return (int)e;
  }
  return 0;
}
