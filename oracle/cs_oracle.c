/*
 * cs_oracle.c — CPU ORACLE for the chunk-step numerics.  TEST
 * INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py as the CHECKER.  Never
 * linked into, or called by, the product path.
 *
 * What it restates
 *   The reference (/root/reference) is an accounting simulator with NO
 *   numerics: SPEC.md:15 puts "numerical ADAM math" out of scope and the
 *   only statements of the arithmetic are PAPER.md:136, 166-169, 402-403
 *   ("grad fp16 chunks are converted to fp32 on the fly ... param fp32
 *   chunks are copied into param fp16 chunk").  The Adam itself is the one
 *   PatrickStar upstream runs (its FP16 Adam / torch_adam_update; upstream
 *   repository not vendored under /root/reference), i.e. textbook
 *   Adam/AdamW with bias correction:
 *       m = b1 m + (1-b1) g ;  v = b2 v + (1-b2) g^2
 *       p -= lr/(1-b1^t) * m / (sqrt(v)/sqrt(1-b2^t) + eps)
 *   PARITY STATUS: the numerics are *unpinned by the reference* (it has
 *   none).  This oracle is pinned instead against torch.optim.Adam /
 *   AdamW (PyTorch 2.11, CPU, fp32) by tests/golden/gen_adam_golden.py
 *   (committed fixtures, relative tolerance 1e-6) — the published
 *   implementation of the same algorithm.
 *
 *   Decisions (layout, FSM, schedule, collectives) are pinned bit-exactly
 *   to the reference itself: tests/golden/gen_decision_golden.py imports
 *   /root/reference/pkg/src/chunkstar and freezes its ledgers.
 *
 * Rounding contract shared with the kernels: the association of
 * torch.optim.Adam's CPU single-tensor path (lerp_ / addcmul_ / addcdiv_,
 * which PyTorch's vectorised CPU kernels evaluate with the fmas written
 * below — verified element-exact against torch 2.11 in this container),
 * explicit fmaf() and otherwise individually rounded ops (compiled
 * -ffp-contract=off, no fast-math), IEEE sqrt/div (torch's CPU sqrt is not
 * correctly rounded, the one source of residual ulp differences vs torch),
 * narrowing by round-to-nearest-even implemented here in integer code.
 */
#include <math.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>

/* ---- 16-bit float conversions (independent software implementation) ---- */

static uint32_t bits_of(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float float_of(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

float or_half_to_float(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t exp = (h >> 10) & 0x1fu;
  uint32_t mant = h & 0x3ffu;
  if (exp == 0x1fu) return float_of(sign | 0x7f800000u | (mant << 13));
  if (exp == 0) {
    if (mant == 0) return float_of(sign);
    /* subnormal: mant * 2^-24, exact in float */
    const float mag = (float)mant * 5.9604644775390625e-08f;
    return sign ? -mag : mag;
  }
  return float_of(sign | ((exp + 112u) << 23) | (mant << 13));
}

uint16_t or_float_to_half(float f) {
  const uint32_t x = bits_of(f);
  const uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
  const uint32_t a = x & 0x7fffffffu;
  if (a >= 0x7f800000u) return sign | (a > 0x7f800000u ? 0x7e00u : 0x7c00u);
  if (a >= 0x477ff000u) return sign | 0x7c00u; /* rounds to infinity */
  if (a >= 0x38800000u) {                      /* normal half */
    uint32_t r = a - 0x38000000u;              /* rebias 127 -> 15 */
    r += 0x0fffu + ((r >> 13) & 1u);           /* nearest-even on 13 dropped bits */
    return sign | (uint16_t)(r >> 13);
  }
  /* subnormal half: value = M * 2^(e-150) = m * 2^-24, m = M >> (126 - e) */
  const uint32_t e = a >> 23;
  if (e < 102u) return sign;
  const uint32_t M = (a & 0x7fffffu) | 0x800000u;
  const uint32_t shift = 126u - e;
  uint32_t q = M >> shift;
  const uint32_t rem = M & ((1u << shift) - 1u), halfway = 1u << (shift - 1u);
  if (rem > halfway || (rem == halfway && (q & 1u))) ++q;
  return sign | (uint16_t)q;
}

float or_bf16_to_float(uint16_t h) { return float_of((uint32_t)h << 16); }

uint16_t or_float_to_bf16(float f) {
  const uint32_t x = bits_of(f);
  if ((x & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((x >> 16) | 0x40u);
  return (uint16_t)((x + 0x7fffu + ((x >> 16) & 1u)) >> 16);
}

static float widen(uint16_t h, int dtype) {
  return dtype == 0 ? or_half_to_float(h) : or_bf16_to_float(h);
}
static uint16_t narrow(float f, int dtype) {
  return dtype == 0 ? or_float_to_half(f) : or_float_to_bf16(f);
}

/* ---- step scalars (mirrors the documented CsStepState layout) ----------- */

typedef struct {
  double beta1_pow, beta2_pow;
  int64_t step;
  float loss_scale;
  int32_t good_steps;
  float grad_scale, step_size, sqrt_bc2;
  int32_t skip;
  float grad_norm, sumsq;
} OrStepState;

void or_step_state_init(OrStepState* s, float loss_scale) {
  memset(s, 0, sizeof(*s));
  s->beta1_pow = 1.0;
  s->beta2_pow = 1.0;
  s->loss_scale = loss_scale;
  s->grad_scale = 1.0f / loss_scale;
  s->sqrt_bc2 = 1.0f;
}

/* Skip on non-finite sumsq (backoff), else clip coefficient (torch
 * clip_grad_norm_ convention: max_norm/(norm+1e-6), capped at 1), bias
 * corrections from running beta powers in double, growth every interval. */
void or_adam_prepare(OrStepState* s, double lr, double beta1, double beta2, float max_norm,
                     float growth, float backoff, int32_t interval, int32_t dynamic_scale) {
  const float sumsq = s->sumsq, ls = s->loss_scale;
  if (!isfinite(sumsq)) {
    s->skip = 1;
    s->grad_norm = sumsq;
    if (dynamic_scale) { s->loss_scale = ls * backoff; s->good_steps = 0; }
    return;
  }
  const float norm = sqrtf(sumsq) / ls;
  float clip = 1.0f;
  if (max_norm > 0.0f) {
    const float c = max_norm / (norm + 1e-6f);
    clip = c < 1.0f ? c : 1.0f;
  }
  s->grad_scale = (1.0f / ls) * clip;
  s->grad_norm = norm;
  s->skip = 0;
  s->step += 1;
  s->beta1_pow = s->beta1_pow * beta1;
  s->beta2_pow = s->beta2_pow * beta2;
  s->step_size = (float)(lr / (1.0 - s->beta1_pow));
  s->sqrt_bc2 = (float)sqrt(1.0 - s->beta2_pow);
  if (dynamic_scale) {
    s->good_steps += 1;
    if (s->good_steps >= interval) { s->loss_scale = ls * growth; s->good_steps = 0; }
  }
}

/* ---- Adam over one chunk prefix ---------------------------------------- */

void or_adam(uint16_t* p16, float* p32, float* m, float* v, int64_t n, int dtype,
             double lr, double beta1, double beta2, double eps, double wd, int adamw,
             const OrStepState* s, int n_threads) {
  if (s->skip) {
    /* skipped step (non-finite gradients): p32 / m / v stay, but the 16-bit
     * chunk holds this step's gradients (grad overwrite) — put the unchanged
     * parameters back over them */
    for (int64_t i = 0; i < n; ++i) p16[i] = narrow(p32[i], dtype);
    return;
  }
  /* scalars formed in double, rounded once (torch.optim.Adam passes python
   * floats to its float kernels the same way) */
  const float b2 = (float)beta2, omb1 = (float)(1.0 - beta1), omb2 = (float)(1.0 - beta2);
  const float decay = (float)(1.0 - lr * wd), wdf = (float)wd, epsf = (float)eps;
  const float gs = s->grad_scale, ss = s->step_size, sb = s->sqrt_bc2;
#pragma omp parallel for num_threads(n_threads > 0 ? n_threads : 1) schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    float g = widen(p16[i], dtype) * gs;
    float p = p32[i];
    if (wd != 0.0) {
      if (adamw) p = p * decay;
      else g = fmaf(wdf, p, g);                        /* g.add(p, alpha=wd) */
    }
    const float mi = fmaf(omb1, g - m[i], m[i]);        /* m.lerp_(g, 1-b1) */
    const float vi = fmaf(omb2 * g, g, v[i] * b2);     /* v.mul_(b2).addcmul_(g, g, 1-b2) */
    const float denom = sqrtf(vi) / sb + epsf;         /* (v.sqrt() / sqrt(bc2)).add_(eps) */
    p = p + (-ss * mi) / denom;                        /* p.addcdiv_(m, denom, -step_size) */
    m[i] = mi;
    v[i] = vi;
    p32[i] = p;
    p16[i] = narrow(p, dtype);
  }
}

/* ---- gradient sum of squares (double accumulation) ---------------------- */

double or_grad_sumsq(const uint16_t* g, int64_t n, int dtype) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double f = widen(g[i], dtype);
    acc += f * f;
  }
  return acc;
}

/* ---- K2's canonical order (paper_2108_05818_b200/csrc/sumsq.cu) ----------
 * S(item): zero-padded 8192-element tiles; lane tau, group u, j: element
 * 8192 t + (256 u + tau) 8 + j; a_j folds x*x over u (fp32); the lane value
 * is the fixed fp32 tree over a_0..a_7; each warp of 32 lanes is an
 * xor-butterfly (o = 16..1) of fp32 adds; the (tile, warp) partials are
 * summed in double by 8192 strided folds, 32 fixed trees of 256 and an
 * ordered fold of the 32 group values.  Scalar C, every
 * fp32 operation rounded on its own (-ffp-contract=off). */

double or_grad_sumsq_item(const uint16_t* g, int64_t n, int dtype) {
  const int64_t tiles = (n + 8191) / 8192;
  const int64_t q_n = tiles * 8;
  float* part = (float*)malloc((size_t)(q_n > 0 ? q_n : 1) * sizeof(float));
  for (int64_t t = 0; t < tiles; ++t) {
    float lane[256];
    for (int tau = 0; tau < 256; ++tau) {
      float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int u = 0; u < 4; ++u)
        for (int j = 0; j < 8; ++j) {
          const int64_t e = 8192 * t + (256 * (int64_t)u + tau) * 8 + j;
          const float x = e < n ? (float)widen(g[e], dtype) : 0.0f;
          const float sq = x * x;
          a[j] = a[j] + sq;
        }
      const float l01 = a[0] + a[1], l23 = a[2] + a[3], l45 = a[4] + a[5], l67 = a[6] + a[7];
      const float lo = l01 + l23, hi = l45 + l67;
      lane[tau] = lo + hi;
    }
    for (int w = 0; w < 8; ++w) {
      float v[32], nv[32];
      for (int l = 0; l < 32; ++l) v[l] = lane[32 * w + l];
      for (int o = 16; o > 0; o >>= 1) {
        for (int l = 0; l < 32; ++l) nv[l] = v[l] + v[l ^ o];
        for (int l = 0; l < 32; ++l) v[l] = nv[l];
      }
      part[8 * t + w] = v[0];
    }
  }
  double total = 0.0;
  for (int c = 0; c < 32; ++c) {      /* 32 groups of 256 strands, stride 8192 */
    double d[256];
    for (int r = 0; r < 256; ++r) {
      double acc = 0.0;
      for (int64_t q = 256 * c + r; q < q_n; q += 8192) acc = acc + (double)part[q];
      d[r] = acc;
    }
    for (int w = 128; w > 0; w >>= 1)
      for (int r = 0; r < w; ++r) d[r] = d[r] + d[r + w];
    total = total + d[0];
  }
  free(part);
  return total;
}

/* the global value: the item sums folded in slot order, rounded to fp32 */
float or_sumsq_total(const double* item_sums, int n) {
  double t = 0.0;
  for (int i = 0; i < n; ++i) t = t + item_sums[i];
  return (float)t;
}

/* ---- pack / accumulate / cast / optimizer-state birth ------------------- */

void or_pack(uint16_t* chunk, int64_t offset, const uint16_t* src, int64_t n, int dtype,
             int accumulate) {
  uint16_t* d = chunk + offset;
  for (int64_t i = 0; i < n; ++i)
    d[i] = accumulate ? narrow(widen(d[i], dtype) + widen(src[i], dtype), dtype) : src[i];
}

void or_cast_pack(uint16_t* chunk, int64_t offset, const float* src, int64_t n, int dtype) {
  for (int64_t i = 0; i < n; ++i) chunk[offset + i] = narrow(src[i], dtype);
}

void or_master_init(float* p32, float* m, float* v, const void* src, int src_dtype, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    p32[i] = src_dtype == 2 ? ((const float*)src)[i]
                            : widen(((const uint16_t*)src)[i], src_dtype);
    m[i] = 0.0f;
    v[i] = 0.0f;
  }
}
