/* TEST INFRASTRUCTURE ONLY — multi-threaded CPU restatement of the expert FFN and LM head for
 * full-size oracle decodes (32-layer Phi / Mixtral / 48-layer Qwen3 widths), where the numpy
 * oracle's cached fp32 expert matrices (oracle/model.py Model.expert_f32) would need tens of GB.
 *
 * Same definitions as oracle/model.py, restated for speed:
 *   weights    bf16(val(idx) * scale) from the counter hash (model.py uniform/gen; model_ref.c
 *              orc_gen_bf16), generated row by row on the fly and never stored
 *   INT4 draft per row, per 128-column group: s = bf16(amax / 7.5), q = clamp(rint(w/s)+8, 0, 15),
 *              w' = (q-8)*s (model.py quantize/dequantize: RTN on GPTQ's symmetric g128 grid,
 *              PAPER.md:564)
 *   FFN        g = G x, u = U x (double accumulation, rounded to fp32), a = bf16(silu(g)*u) with
 *              the deterministic exp (model_ref.c orc_act), y = D a (double -> fp32)
 *   LM head    model_ref.c orc_lm_head (fixed-order warp dot), rows split over threads
 *
 * The device's tensor-core FFN differs from this in accumulation order only; tests compare it
 * within |dy| <= 2e-3 max|y| + 1e-5.  Routing and argmax, computed from the
 * resulting hidden states with model_ref.c, are compared bit-exactly.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void orc_act(const float* g, const float* u, int f, uint16_t* a);
float orc_warp_dot(const uint16_t* x, const uint16_t* w, int n);

static inline float bf2f(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }
static inline uint16_t f2bf(float f) {
  uint32_t u; memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
/* model.py tensor_key(seed, tensor) */
uint64_t orc_tensor_key(uint64_t seed, uint64_t tensor) { return mix64(seed ^ mix64(tensor)); }

/* one weight row (cols values starting at flat index start), widened to fp32; with q4 the
 * row is replaced by its INT4 dequantisation */
static void gen_row(uint64_t key, uint64_t start, int cols, float scale, int q4, float* w) {
  for (int i = 0; i < cols; ++i) {
    const uint64_t z = mix64(key + (start + (uint64_t)i) * 0xD1B54A32D192ED03ull);
    const int32_t hi = (int32_t)(z >> 40) - (1 << 23);
    const float v = ((float)hi + 0.5f) * (1.0f / 8388608.0f);
    w[i] = bf2f(f2bf(v * scale));
  }
  if (!q4) return;
  for (int g0 = 0; g0 < cols; g0 += 128) {
    float amax = 0.0f;
    for (int i = g0; i < g0 + 128; ++i) amax = fmaxf(amax, fabsf(w[i]));
    const float s = bf2f(f2bf(amax / 7.5f));
    const float sd = s == 0.0f ? 1.0f : s;      /* model.py: sf_safe */
    const float ss = s == 0.0f ? 1.0f : s;      /* stored scale: bf16(1.0) when amax == 0 */
    for (int i = g0; i < g0 + 128; ++i) {
      float q = rintf(w[i] / sd) + 8.0f;
      q = q < 0.0f ? 0.0f : (q > 15.0f ? 15.0f : q);
      w[i] = (q - 8.0f) * ss;
    }
  }
}

#define T_EXPERT(l, e, m) (0x1000000ull + ((uint64_t)(l) * 1024 + (uint64_t)(e)) * 4 + (uint64_t)(m))

/* Expert (l, e) FFN for M tokens: xn [M][d] bf16 -> y [M][d] fp32 (and act [M][f] bf16 if
 * non-NULL).  draft != 0 runs the INT4 draft of the expert. */
int orc_expert_ffn(uint64_t seed, int l, int e, int d, int f, float a_up, float a_down, int draft,
                   int M, const uint16_t* xn, float* y, uint16_t* act_out) {
  const uint64_t kg = orc_tensor_key(seed, T_EXPERT(l, e, 0)), ku = orc_tensor_key(seed, T_EXPERT(l, e, 1)),
                 kd = orc_tensor_key(seed, T_EXPERT(l, e, 2));
  float* x = (float*)malloc(sizeof(float) * (size_t)M * d);
  float* gv = (float*)malloc(sizeof(float) * (size_t)M * f);
  float* uv = (float*)malloc(sizeof(float) * (size_t)M * f);
  float* af = (float*)malloc(sizeof(float) * (size_t)M * f);
  uint16_t* a = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)M * f);
  if (!x || !gv || !uv || !af || !a) return 1;
  for (size_t i = 0; i < (size_t)M * d; ++i) x[i] = bf2f(xn[i]);
#pragma omp parallel
  {
    float* wg = (float*)malloc(sizeof(float) * (size_t)d);
    float* wu = (float*)malloc(sizeof(float) * (size_t)d);
#pragma omp for schedule(static)
    for (int r = 0; r < f; ++r) {
      gen_row(kg, (uint64_t)r * d, d, a_up, draft, wg);
      gen_row(ku, (uint64_t)r * d, d, a_up, draft, wu);
      for (int m = 0; m < M; ++m) {
        const float* xm = x + (size_t)m * d;
        double sg = 0.0, su = 0.0;
        for (int c = 0; c < d; ++c) {
          sg += (double)wg[c] * (double)xm[c];
          su += (double)wu[c] * (double)xm[c];
        }
        gv[(size_t)m * f + r] = (float)sg;
        uv[(size_t)m * f + r] = (float)su;
      }
    }
    free(wg);
    free(wu);
  }
  for (int m = 0; m < M; ++m) orc_act(gv + (size_t)m * f, uv + (size_t)m * f, f, a + (size_t)m * f);
  for (size_t i = 0; i < (size_t)M * f; ++i) af[i] = bf2f(a[i]);
#pragma omp parallel
  {
    float* wd = (float*)malloc(sizeof(float) * (size_t)f);
#pragma omp for schedule(static)
    for (int r = 0; r < d; ++r) {
      gen_row(kd, (uint64_t)r * f, f, a_down, draft, wd);
      for (int m = 0; m < M; ++m) {
        const float* am = af + (size_t)m * f;
        double s = 0.0;
        for (int c = 0; c < f; ++c) s += (double)wd[c] * (double)am[c];
        y[(size_t)m * d + r] = (float)s;
      }
    }
    free(wd);
  }
  if (act_out) memcpy(act_out, a, sizeof(uint16_t) * (size_t)M * f);
  free(x);
  free(gv);
  free(uv);
  free(af);
  free(a);
  return 0;
}

/* orc_lm_head (model_ref.c) with the vocabulary rows split over threads; argmax tie -> lower id */
void orc_lm_head_mt(const uint16_t* xn, const uint16_t* lm, int T, int V, int d, float* logits,
                    int32_t* argmax) {
#pragma omp parallel for schedule(static)
  for (int v = 0; v < V; ++v)
    for (int t = 0; t < T; ++t) logits[(size_t)t * V + v] = orc_warp_dot(xn + (size_t)t * d, lm + (size_t)v * d, d);
  for (int t = 0; t < T; ++t) {
    int best = 0;
    for (int v = 1; v < V; ++v)
      if (logits[(size_t)t * V + v] > logits[(size_t)t * V + best]) best = v;
    argmax[t] = best;
  }
}

/* bf16 tensor rows [r0, r1) of a (rows x cols) generated tensor, multi-threaded */
void orc_gen_rows_mt(uint64_t key, int64_t r0, int64_t r1, int cols, float scale, uint16_t* out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = r0; r < r1; ++r)
    for (int c = 0; c < cols; ++c) {
      const uint64_t z = mix64(key + ((uint64_t)r * cols + (uint64_t)c) * 0xD1B54A32D192ED03ull);
      const int32_t hi = (int32_t)(z >> 40) - (1 << 23);
      const float v = ((float)hi + 0.5f) * (1.0f / 8388608.0f);
      out[(size_t)(r - r0) * cols + c] = f2bf(v * scale);
    }
}

/* exported for the CPU tests: one generated (and optionally INT4 round-tripped) weight row */
void orc_weight_row(uint64_t key, uint64_t start, int cols, float scale, int q4, float* w) {
  gen_row(key, start, cols, scale, q4, w);
}
