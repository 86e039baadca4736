// Host embedding operator for a CPU-placed embedding (PatrickStar's
// device-aware operator placement, PAPER §5;
// /root/reference/pkg/src/chunkstar/profiler.py:70-74 decides the device,
// engine.py:202-223 bills the CPU branch: "weights stay put; one activation
// block crosses per pass" — B*S*H fp16 down at FWD, its gradient up at BWD).
//
// The fp16/bf16 weights (wte [V,H], wpe [S,H]) live in pinned host DRAM.
// Forward: out[i,:] = round(float(wte[tok[i],:]) + float(wpe[i % S,:])),
// exactly torch's `F.embedding(tok, wte) + wpe[:S]` (one fp32 add, one
// rounding).  Backward (grad overwrite into the weight buffers, as the chunk
// path does, engine.py:177-190): the rows of wte hit by a token get the fp32
// sum of their dout rows in ascending token order, rounded once; rows no
// token hits get 0; wpe[s,:] gets the fp32 sum over b ascending of
// dout[b*S+s,:].  Deterministic; bit-identical to the numpy oracle
// (oracle/numerics.py embed_*).  Compiled with -ffp-contract=off.
#include <immintrin.h>
#include <omp.h>

#include <cstring>
#include <vector>

#include "cs_internal.h"

namespace {

template <int DT>
__attribute__((target("avx2,f16c"))) inline __m256 load8(const uint16_t* p) {
  const __m128i h = _mm_loadu_si128(reinterpret_cast<const __m128i*>(p));
  if (DT == CS_FP16) return _mm256_cvtph_ps(h);
  return _mm256_castsi256_ps(_mm256_slli_epi32(_mm256_cvtepu16_epi32(h), 16));
}

template <int DT>
__attribute__((target("avx2,f16c"))) inline void store8(uint16_t* p, __m256 f) {
  __m128i h;
  if (DT == CS_FP16) {
    h = _mm256_cvtps_ph(f, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
  } else {  // bf16 round-to-nearest-even
    const __m256i x = _mm256_castps_si256(f);
    const __m256i lsb = _mm256_and_si256(_mm256_srli_epi32(x, 16), _mm256_set1_epi32(1));
    const __m256i r = _mm256_srli_epi32(
        _mm256_add_epi32(_mm256_add_epi32(x, _mm256_set1_epi32(0x7fff)), lsb), 16);
    h = _mm_packus_epi32(_mm256_castsi256_si128(r), _mm256_extracti128_si256(r, 1));
  }
  _mm_storeu_si128(reinterpret_cast<__m128i*>(p), h);
}

template <int DT>
__attribute__((target("avx2,f16c"))) void fwd_rows(const int64_t* tok, int64_t n, int S,
                                                   const uint16_t* wte, const uint16_t* wpe,
                                                   int H, uint16_t* out, int threads) {
#pragma omp parallel for num_threads(threads) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const uint16_t* a = wte + tok[i] * (int64_t)H;
    const uint16_t* b = wpe + (i % S) * (int64_t)H;
    uint16_t* o = out + i * (int64_t)H;
    for (int c = 0; c < H; c += 8) store8<DT>(o + c, _mm256_add_ps(load8<DT>(a + c),
                                                                    load8<DT>(b + c)));
  }
}

// Sum of squares of one stored (rounded) 16-bit row, in double, fixed order.
template <int DT>
__attribute__((target("avx2,f16c"))) double row_sumsq(const uint16_t* g, int H) {
  __m256d acc0 = _mm256_setzero_pd(), acc1 = _mm256_setzero_pd();
  for (int c = 0; c < H; c += 8) {
    const __m256 f = load8<DT>(g + c);
    const __m256d lo = _mm256_cvtps_pd(_mm256_castps256_ps128(f));
    const __m256d hi = _mm256_cvtps_pd(_mm256_extractf128_ps(f, 1));
    acc0 = _mm256_add_pd(acc0, _mm256_mul_pd(lo, lo));
    acc1 = _mm256_add_pd(acc1, _mm256_mul_pd(hi, hi));
  }
  alignas(32) double t[8];
  _mm256_store_pd(t, acc0);
  _mm256_store_pd(t + 4, acc1);
  return ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
}

template <int DT>
__attribute__((target("avx2,f16c"))) void bwd_rows(const int64_t* tok, int64_t n, int S,
                                                   const uint16_t* dout, int64_t V, int H,
                                                   uint16_t* gwte, uint16_t* gwpe,
                                                   int threads, double* sumsq) {
  // per-row squared sums of the stored gradients (only rows a token hit are
  // nonzero), reduced in row order below: deterministic for any thread count
  std::vector<double> row_sq(sumsq ? V + S : 0, 0.0);
  // counting sort of token positions by row (stable: ascending i per row)
  std::vector<int64_t> start(V + 1, 0), order(n);
  for (int64_t i = 0; i < n; ++i) ++start[tok[i] + 1];
  for (int64_t v = 0; v < V; ++v) start[v + 1] += start[v];
  {
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (int64_t i = 0; i < n; ++i) order[fill[tok[i]]++] = i;
  }
#pragma omp parallel num_threads(threads)
  {
    std::vector<float> acc(H);
    float* a = acc.data();
#pragma omp for schedule(dynamic, 64)
    for (int64_t v = 0; v < V; ++v) {
      uint16_t* g = gwte + v * (int64_t)H;
      if (start[v] == start[v + 1]) {
        std::memset(g, 0, (size_t)H * 2);
        continue;
      }
      for (int c = 0; c < H; c += 8) _mm256_storeu_ps(a + c, _mm256_setzero_ps());
      for (int64_t k = start[v]; k < start[v + 1]; ++k) {
        const uint16_t* d = dout + order[k] * (int64_t)H;
        for (int c = 0; c < H; c += 8)
          _mm256_storeu_ps(a + c, _mm256_add_ps(_mm256_loadu_ps(a + c), load8<DT>(d + c)));
      }
      for (int c = 0; c < H; c += 8) store8<DT>(g + c, _mm256_loadu_ps(a + c));
      if (sumsq) row_sq[v] = row_sumsq<DT>(g, H);
    }
    const int64_t B = n / S;
#pragma omp for schedule(static)
    for (int64_t s = 0; s < S; ++s) {
      for (int c = 0; c < H; c += 8) _mm256_storeu_ps(a + c, _mm256_setzero_ps());
      for (int64_t b = 0; b < B; ++b) {
        const uint16_t* d = dout + (b * S + s) * (int64_t)H;
        for (int c = 0; c < H; c += 8)
          _mm256_storeu_ps(a + c, _mm256_add_ps(_mm256_loadu_ps(a + c), load8<DT>(d + c)));
      }
      for (int c = 0; c < H; c += 8) store8<DT>(gwpe + s * (int64_t)H + c, _mm256_loadu_ps(a + c));
      if (sumsq) row_sq[V + s] = row_sumsq<DT>(gwpe + s * (int64_t)H, H);
    }
  }
  if (sumsq) {
    double total = 0.0;
    for (double x : row_sq) total += x;
    *sumsq = total;
  }
}

bool host_ok() {
  return __builtin_cpu_supports("avx2") && __builtin_cpu_supports("f16c");
}

int check_tokens(const int64_t* tok, int64_t n, int64_t V, const char* who) {
  for (int64_t i = 0; i < n; ++i)
    if (tok[i] < 0 || tok[i] >= V) {
      cs::set_error("%s: token %lld at %lld out of [0, %lld)", who, (long long)tok[i],
                    (long long)i, (long long)V);
      return CS_EINVAL;
    }
  return 0;
}

}  // namespace

extern "C" int cs_embed_fwd_host(const int64_t* tokens, int64_t n_tokens, int seq_len,
                                 const void* wte, const void* wpe, int64_t vocab, int hidden,
                                 void* out, int dtype, int n_threads) {
  if (n_tokens < 0 || seq_len <= 0 || vocab <= 0 || hidden <= 0 || hidden % 8 != 0 ||
      (n_tokens > 0 && (!tokens || !wte || !wpe || !out)) ||
      (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_embed_fwd_host: invalid argument (hidden must be a multiple of 8)");
    return CS_EINVAL;
  }
  if (!host_ok()) {
    cs::set_error("cs_embed_fwd_host: host CPU lacks AVX2/F16C");
    return CS_EINVAL;
  }
  if (int rc = check_tokens(tokens, n_tokens, vocab, "cs_embed_fwd_host")) return rc;
  const int threads = cs::host_threads(n_threads);
  const auto* a = static_cast<const uint16_t*>(wte);
  const auto* b = static_cast<const uint16_t*>(wpe);
  auto* o = static_cast<uint16_t*>(out);
  if (dtype == CS_FP16) fwd_rows<CS_FP16>(tokens, n_tokens, seq_len, a, b, hidden, o, threads);
  else fwd_rows<CS_BF16>(tokens, n_tokens, seq_len, a, b, hidden, o, threads);
  return 0;
}

extern "C" int cs_embed_bwd_host(const int64_t* tokens, int64_t n_tokens, int seq_len,
                                 const void* dout, int64_t vocab, int hidden, void* gwte,
                                 void* gwpe, int dtype, int n_threads, double* sumsq) {
  if (n_tokens < 0 || seq_len <= 0 || n_tokens % seq_len != 0 || vocab <= 0 || hidden <= 0 ||
      hidden % 8 != 0 || !gwte || !gwpe || (n_tokens > 0 && (!tokens || !dout)) ||
      (dtype != CS_FP16 && dtype != CS_BF16)) {
    cs::set_error("cs_embed_bwd_host: invalid argument (n_tokens must be a multiple of "
                  "seq_len, hidden of 8)");
    return CS_EINVAL;
  }
  if (!host_ok()) {
    cs::set_error("cs_embed_bwd_host: host CPU lacks AVX2/F16C");
    return CS_EINVAL;
  }
  if (int rc = check_tokens(tokens, n_tokens, vocab, "cs_embed_bwd_host")) return rc;
  const int threads = cs::host_threads(n_threads);
  const auto* d = static_cast<const uint16_t*>(dout);
  auto* gw = static_cast<uint16_t*>(gwte);
  auto* gp = static_cast<uint16_t*>(gwpe);
  if (dtype == CS_FP16)
    bwd_rows<CS_FP16>(tokens, n_tokens, seq_len, d, vocab, hidden, gw, gp, threads, sumsq);
  else
    bwd_rows<CS_BF16>(tokens, n_tokens, seq_len, d, vocab, hidden, gw, gp, threads, sumsq);
  return 0;
}
