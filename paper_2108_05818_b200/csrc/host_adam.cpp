// Host fused Adam for optimizer triplets the placement plan keeps in pinned
// host DRAM (PatrickStar's device-aware placement, PAPER §5;
// /root/reference/pkg/src/chunkstar/profiler.py:93-130 decides it and
// engine.py:249-251/265-267 bill the grad D2H and param H2D `adam_copy`).
//
// Same per-element arithmetic and rounding as the CUDA kernel K1
// (cs_adam_chunks): the fmas are explicit _mm256_fmadd_ps, everything else is
// individually rounded (compiled with -ffp-contract=off), IEEE sqrt/div,
// round-to-nearest-even narrowing.  8 lanes per step; OpenMP over 64
// Ki-element ranges of every item.
#include <immintrin.h>
#include <omp.h>

#include <cstring>
#include <vector>

#include "cs_internal.h"

namespace {

struct Consts {
  __m256 gs, nss, sb, b2, c1, c2, eps, wd, decay;
  bool adamw, has_wd;
};

template <int DT>
__attribute__((target("avx2,fma,f16c"))) inline __m256 load16(const uint16_t* p) {
  const __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p));
  if (DT == CS_FP16) return _mm256_cvtph_ps(h);
  return _mm256_castsi256_ps(_mm256_slli_epi32(_mm256_cvtepu16_epi32(h), 16));
}

// Round-to-nearest-even narrowing; NaN lanes become the canonical NaN
// 0x7fff, which is what the device conversions (cvt.rn.f16.f32 /
// cvt.rn.bf16.f32, used by K1) produce -- without the blend a bf16 NaN with
// high mantissa bits would wrap to -0 and fp16 would keep the payload.
template <int DT>
__attribute__((target("avx2,fma,f16c"))) inline void store16(uint16_t* p, __m256 f) {
  const __m256i nan = _mm256_castps_si256(_mm256_cmp_ps(f, f, _CMP_UNORD_Q));
  __m128i h;
  if (DT == CS_FP16) {
    h = _mm256_cvtps_ph(f, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
    const __m128i nan16 =
        _mm_packs_epi32(_mm256_castsi256_si128(nan), _mm256_extracti128_si256(nan, 1));
    h = _mm_blendv_epi8(h, _mm_set1_epi16(0x7fff), nan16);
  } else {  // bf16 round-to-nearest-even: (x + 0x7fff + lsb) >> 16
    const __m256i x = _mm256_castps_si256(f);
    const __m256i lsb = _mm256_and_si256(_mm256_srli_epi32(x, 16), _mm256_set1_epi32(1));
    __m256i r = _mm256_srli_epi32(
        _mm256_add_epi32(_mm256_add_epi32(x, _mm256_set1_epi32(0x7fff)), lsb), 16);
    r = _mm256_blendv_epi8(r, _mm256_set1_epi32(0x7fff), nan);
    h = _mm_packus_epi32(_mm256_castsi256_si128(r), _mm256_extracti128_si256(r, 1));
  }
  _mm_storeu_si128(reinterpret_cast<__m128i*>(p), h);
}

// in: g16 (gradients), p32, m, v; out: o16, o32, om, ov (may alias the inputs
// unless STREAM; STREAM needs 32-byte aligned fp32 and 16-byte aligned fp16 outputs)
template <int DT, bool STREAM = false>
__attribute__((target("avx2,fma,f16c"))) inline void adam8_oop(
    const uint16_t* g16, const float* p32, const float* m, const float* v, uint16_t* o16,
    float* o32, float* om, float* ov, const Consts& c) {
  __m256 g = _mm256_mul_ps(load16<DT>(g16), c.gs);
  __m256 p = _mm256_loadu_ps(p32);
  if (c.has_wd) {
    if (c.adamw) p = _mm256_mul_ps(p, c.decay);
    else g = _mm256_fmadd_ps(c.wd, p, g);
  }
  const __m256 m0 = _mm256_loadu_ps(m);
  const __m256 mm = _mm256_fmadd_ps(c.c1, _mm256_sub_ps(g, m0), m0);
  const __m256 vv = _mm256_fmadd_ps(_mm256_mul_ps(c.c2, g), g,
                                    _mm256_mul_ps(_mm256_loadu_ps(v), c.b2));
  const __m256 denom = _mm256_add_ps(_mm256_div_ps(_mm256_sqrt_ps(vv), c.sb), c.eps);
  p = _mm256_add_ps(p, _mm256_div_ps(_mm256_mul_ps(c.nss, mm), denom));
  if (STREAM) {  // fresh output lines: non-temporal stores skip the read-for-ownership
    _mm256_stream_ps(o32, p);
    _mm256_stream_ps(om, mm);
    _mm256_stream_ps(ov, vv);
    alignas(16) uint16_t h[8];
    store16<DT>(h, p);
    _mm_stream_si128(reinterpret_cast<__m128i*>(o16),
                     _mm_load_si128(reinterpret_cast<const __m128i*>(h)));
  } else {
    _mm256_storeu_ps(o32, p);
    _mm256_storeu_ps(om, mm);
    _mm256_storeu_ps(ov, vv);
    store16<DT>(o16, p);
  }
}

template <int DT>
__attribute__((target("avx2,fma,f16c"))) void adam_range_oop(const CsAdamItem& in,
                                                          const CsAdamItem& out, int64_t lo,
                                                          int64_t hi, const Consts& c) {
  const uint16_t* g16 = static_cast<const uint16_t*>(in.p16);
  uint16_t* o16 = static_cast<uint16_t*>(out.p16);
  int64_t e = lo;
  const bool aligned = ((reinterpret_cast<uintptr_t>(out.p32) | reinterpret_cast<uintptr_t>(out.m) |
                         reinterpret_cast<uintptr_t>(out.v)) & 31) == 0 &&
                       (reinterpret_cast<uintptr_t>(o16) & 15) == 0 && (lo & 7) == 0;
  if (aligned) {
    for (; e + 8 <= hi; e += 8)
      adam8_oop<DT, true>(g16 + e, in.p32 + e, in.m + e, in.v + e, o16 + e, out.p32 + e,
                          out.m + e, out.v + e, c);
  } else {
    for (; e + 8 <= hi; e += 8)
      adam8_oop<DT>(g16 + e, in.p32 + e, in.m + e, in.v + e, o16 + e, out.p32 + e, out.m + e,
                    out.v + e, c);
  }
  if (e < hi) {  // tail: the same 8-lane code on a padded copy
    alignas(32) uint16_t t16[8] = {0};
    alignas(32) float tp[8] = {0}, tm[8] = {0}, tv[8] = {0};
    const int64_t k = hi - e;
    std::memcpy(t16, g16 + e, k * 2);
    std::memcpy(tp, in.p32 + e, k * 4);
    std::memcpy(tm, in.m + e, k * 4);
    std::memcpy(tv, in.v + e, k * 4);
    adam8_oop<DT>(t16, tp, tm, tv, t16, tp, tm, tv, c);
    std::memcpy(o16 + e, t16, k * 2);
    std::memcpy(out.p32 + e, tp, k * 4);
    std::memcpy(out.m + e, tm, k * 4);
    std::memcpy(out.v + e, tv, k * 4);
  }
}

template <int DT>
__attribute__((target("avx2,fma,f16c"))) inline void adam8(uint16_t* p16, float* p32, float* m,
                                                        float* v, const Consts& c) {
  __m256 g = _mm256_mul_ps(load16<DT>(p16), c.gs);
  __m256 p = _mm256_loadu_ps(p32);
  if (c.has_wd) {
    if (c.adamw) p = _mm256_mul_ps(p, c.decay);
    else g = _mm256_fmadd_ps(c.wd, p, g);
  }
  const __m256 m0 = _mm256_loadu_ps(m);
  const __m256 mm = _mm256_fmadd_ps(c.c1, _mm256_sub_ps(g, m0), m0);
  const __m256 vv = _mm256_fmadd_ps(_mm256_mul_ps(c.c2, g), g,
                                    _mm256_mul_ps(_mm256_loadu_ps(v), c.b2));
  const __m256 denom = _mm256_add_ps(_mm256_div_ps(_mm256_sqrt_ps(vv), c.sb), c.eps);
  p = _mm256_add_ps(p, _mm256_div_ps(_mm256_mul_ps(c.nss, mm), denom));
  _mm256_storeu_ps(p32, p);
  _mm256_storeu_ps(m, mm);
  _mm256_storeu_ps(v, vv);
  store16<DT>(p16, p);
}

template <int DT>
__attribute__((target("avx2,fma,f16c"))) void adam_range(const CsAdamItem& it, int64_t lo,
                                                      int64_t hi, const Consts& c) {
  uint16_t* p16 = static_cast<uint16_t*>(it.p16);
  int64_t e = lo;
  for (; e + 8 <= hi; e += 8) adam8<DT>(p16 + e, it.p32 + e, it.m + e, it.v + e, c);
  if (e < hi) {  // tail: run the same 8-lane code on a padded copy
    alignas(32) uint16_t t16[8] = {0};
    alignas(32) float tp[8] = {0}, tm[8] = {0}, tv[8] = {0};
    const int64_t k = hi - e;
    std::memcpy(t16, p16 + e, k * 2);
    std::memcpy(tp, it.p32 + e, k * 4);
    std::memcpy(tm, it.m + e, k * 4);
    std::memcpy(tv, it.v + e, k * 4);
    adam8<DT>(t16, tp, tm, tv, c);
    std::memcpy(p16 + e, t16, k * 2);
    std::memcpy(it.p32 + e, tp, k * 4);
    std::memcpy(it.m + e, tm, k * 4);
    std::memcpy(it.v + e, tv, k * 4);
  }
}

// A skipped step leaves p32 / m / v alone, but the 16-bit chunk holds the
// step's gradients (grad overwrite): put the unchanged parameters back.
template <int DT>
__attribute__((target("avx2,fma,f16c"))) void restore_item(const CsAdamItem& it, int threads) {
  if (it.n <= 0) return;
  uint16_t* q16 = static_cast<uint16_t*>(it.p16);
  const int64_t nv = it.n & ~(int64_t)7;
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t e = 0; e < nv; e += 8) store16<DT>(q16 + e, _mm256_loadu_ps(it.p32 + e));
  for (int64_t e = nv; e < it.n; ++e) {
    alignas(32) float t[8] = {it.p32[e]};
    alignas(16) uint16_t o[8];
    store16<DT>(o, _mm256_load_ps(t));
    q16[e] = o[0];
  }
}

__attribute__((target("avx2,fma,f16c"))) Consts make_consts(const CsAdamHyper& h,
                                                         const CsStepState& s) {
  // scalars formed in double and rounded once, exactly as cs_adam_chunks
  Consts c;
  c.gs = _mm256_set1_ps(s.grad_scale);
  c.nss = _mm256_set1_ps(-s.step_size);
  c.sb = _mm256_set1_ps(s.sqrt_bc2);
  c.b2 = _mm256_set1_ps((float)h.beta2);
  c.c1 = _mm256_set1_ps((float)(1.0 - h.beta1));
  c.c2 = _mm256_set1_ps((float)(1.0 - h.beta2));
  c.eps = _mm256_set1_ps((float)h.eps);
  c.wd = _mm256_set1_ps((float)h.weight_decay);
  c.decay = _mm256_set1_ps((float)(1.0 - h.lr * h.weight_decay));
  c.adamw = h.adamw != 0;
  c.has_wd = h.weight_decay != 0.0f;
  return c;
}

}  // namespace

extern "C" int cs_adam_chunks_host(const CsAdamItem* items, int n_items, int dtype,
                                   const CsAdamHyper* hyper, const CsStepState* state,
                                   int n_threads) {
  if (n_items < 0 || (n_items > 0 && !items) || !hyper || !state ||
      (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_adam_chunks_host: invalid argument");
    return CS_EINVAL;
  }
  if (!__builtin_cpu_supports("avx2") || !__builtin_cpu_supports("fma") ||
      !__builtin_cpu_supports("f16c")) {
    cs::set_error("cs_adam_chunks_host: host CPU lacks AVX2/FMA/F16C");
    return CS_EINVAL;
  }
  if (state->skip) {  // non-finite gradients: no update, p16 = round(p32) restored
    const int threads = cs::host_threads(n_threads);
    for (int i = 0; i < n_items; ++i)
      if (dtype == CS_FP16) restore_item<CS_FP16>(items[i], threads);
      else restore_item<CS_BF16>(items[i], threads);
    return 0;
  }
  const Consts c = make_consts(*hyper, *state);
  constexpr int64_t kRange = 1 << 16;
  std::vector<std::pair<int, int64_t>> ranges;
  for (int i = 0; i < n_items; ++i) {
    if (items[i].n < 0 || (items[i].n > 0 && (!items[i].p16 || !items[i].p32 ||
                                              !items[i].m || !items[i].v))) {
      cs::set_error("cs_adam_chunks_host: item %d invalid", i);
      return CS_EINVAL;
    }
    for (int64_t lo = 0; lo < items[i].n; lo += kRange) ranges.emplace_back(i, lo);
  }
  const int64_t nr = (int64_t)ranges.size();
  const int threads = cs::host_threads(n_threads);
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t r = 0; r < nr; ++r) {
    const CsAdamItem& it = items[ranges[r].first];
    const int64_t lo = ranges[r].second;
    const int64_t hi = lo + kRange < it.n ? lo + kRange : it.n;
    if (dtype == CS_FP16) adam_range<CS_FP16>(it, lo, hi, c);
    else adam_range<CS_BF16>(it, lo, hi, c);
  }
  return 0;
}

extern "C" int cs_adam_chunks_host_oop(const CsAdamItem* in, const CsAdamItem* out,
                                       int n_items, int dtype, const CsAdamHyper* hyper,
                                       const CsStepState* state, int n_threads) {
  if (n_items < 0 || (n_items > 0 && (!in || !out)) || !hyper || !state ||
      (dtype != CS_FP16 && dtype != CS_BF16) || state->skip) {
    cs::set_error("cs_adam_chunks_host_oop: invalid argument (a skipped step has no update)");
    return CS_EINVAL;
  }
  if (!__builtin_cpu_supports("avx2") || !__builtin_cpu_supports("fma") ||
      !__builtin_cpu_supports("f16c")) {
    cs::set_error("cs_adam_chunks_host_oop: host CPU lacks AVX2/FMA/F16C");
    return CS_EINVAL;
  }
  const Consts c = make_consts(*hyper, *state);
  constexpr int64_t kRange = 1 << 16;
  std::vector<std::pair<int, int64_t>> ranges;
  for (int i = 0; i < n_items; ++i) {
    const CsAdamItem& a = in[i];
    const CsAdamItem& b = out[i];
    if (a.n < 0 || a.n != b.n ||
        (a.n > 0 && (!a.p16 || !a.p32 || !a.m || !a.v || !b.p16 || !b.p32 || !b.m || !b.v))) {
      cs::set_error("cs_adam_chunks_host_oop: item %d invalid", i);
      return CS_EINVAL;
    }
    for (int64_t lo = 0; lo < a.n; lo += kRange) ranges.emplace_back(i, lo);
  }
  const int64_t nr = (int64_t)ranges.size();
  const int threads = cs::host_threads(n_threads);
#pragma omp parallel num_threads(threads)
  {
#pragma omp for schedule(static)
    for (int64_t r = 0; r < nr; ++r) {
      const int i = ranges[r].first;
      const int64_t lo = ranges[r].second;
      const int64_t hi = lo + kRange < in[i].n ? lo + kRange : in[i].n;
      if (dtype == CS_FP16) adam_range_oop<CS_FP16>(in[i], out[i], lo, hi, c);
      else adam_range_oop<CS_BF16>(in[i], out[i], lo, hi, c);
    }
    _mm_sfence();  // each thread's non-temporal stores are visible before the join
  }
  return 0;
}

namespace {
// Host twin of K2 (sumsq.cu): the canonical per-item order, fp32 adds and
// multiplies as separate rounded operations (no FMA; -ffp-contract=off).
constexpr int64_t kSqTile = 8192;

template <int DT>
__attribute__((target("avx2,f16c"))) inline __m256 widen8(const uint16_t* p) {
  const __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p));
  if (DT == CS_FP16) return _mm256_cvtph_ps(h);
  return _mm256_castsi256_ps(_mm256_slli_epi32(_mm256_cvtepu16_epi32(h), 16));
}

// the 8 warp partials of one zero-padded tile
template <int DT>
__attribute__((target("avx2,f16c"))) void tile_partials(const uint16_t* tile, float* out8) {
  float lane[256];
  for (int tau = 0; tau < 256; ++tau) {
    __m256 a = _mm256_setzero_ps();
    for (int u = 0; u < 4; ++u) {
      const __m256 x = widen8<DT>(tile + (256 * u + tau) * 8);
      a = _mm256_add_ps(a, _mm256_mul_ps(x, x));
    }
    alignas(32) float aj[8];
    _mm256_store_ps(aj, a);
    lane[tau] = ((aj[0] + aj[1]) + (aj[2] + aj[3])) + ((aj[4] + aj[5]) + (aj[6] + aj[7]));
  }
  for (int w = 0; w < 8; ++w) {
    float v[32];
    std::memcpy(v, lane + 32 * w, sizeof(v));
    for (int o = 16; o > 0; o >>= 1) {
      float nv[32];
      for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ o];
      std::memcpy(v, nv, sizeof(v));
    }
    out8[w] = v[0];
  }
}

template <int DT>
double item_sumsq(const uint16_t* g, int64_t n, int threads) {
  const int64_t tiles = (n + kSqTile - 1) / kSqTile;
  std::vector<float> part((size_t)tiles * 8);
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t t = 0; t < tiles; ++t) {
    const int64_t base = t * kSqTile;
    if (base + kSqTile <= n) {
      tile_partials<DT>(g + base, part.data() + t * 8);
    } else {
      std::vector<uint16_t> pad(kSqTile, 0);
      std::memcpy(pad.data(), g + base, (size_t)(n - base) * 2);
      tile_partials<DT>(pad.data(), part.data() + t * 8);
    }
  }
  // 32 groups of 256 strands (strand s folds q = s, s + 8192, ...), each
  // group a fixed tree, the group values folded in order
  const int64_t q_n = tiles * 8;
  double total = 0.0;
  for (int c = 0; c < 32; ++c) {
    double d[256];
    for (int r = 0; r < 256; ++r) {
      double acc = 0.0;
      for (int64_t q = 256 * c + r; q < q_n; q += 8192) acc += (double)part[q];
      d[r] = acc;
    }
    for (int w = 128; w > 0; w >>= 1)
      for (int r = 0; r < w; ++r) d[r] += d[r + w];
    total += d[0];
  }
  return total;
}
}  // namespace

extern "C" int cs_grad_sumsq_host(const CsGradItem* items, int n_items, int dtype, double* out,
                                  int n_threads) {
  if (n_items < 0 || (n_items > 0 && (!items || !out)) || (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_grad_sumsq_host: invalid argument");
    return CS_EINVAL;
  }
  if (!__builtin_cpu_supports("avx2") || !__builtin_cpu_supports("f16c")) {
    cs::set_error("cs_grad_sumsq_host: host CPU lacks AVX2/F16C");
    return CS_EINVAL;
  }
  const int threads = cs::host_threads(n_threads);
  for (int i = 0; i < n_items; ++i) {
    const uint16_t* g = static_cast<const uint16_t*>(items[i].g16);
    if (items[i].n < 0 || (items[i].n > 0 && !g)) {
      cs::set_error("cs_grad_sumsq_host: item %d invalid", i);
      return CS_EINVAL;
    }
    out[i] = dtype == CS_FP16 ? item_sumsq<CS_FP16>(g, items[i].n, threads)
                              : item_sumsq<CS_BF16>(g, items[i].n, threads);
  }
  return 0;
}
