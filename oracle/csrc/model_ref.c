/* TEST INFRASTRUCTURE ONLY — CPU restatement of the order-sensitive fp32 arithmetic of the
 * decode path (DESIGN.md §3 "numerics contract").  No reference implementation of the MoE
 * math exists in /root/reference (SPEC.md:17 puts kernels out of scope); the semantics come
 * from PAPER.md:466-474 (bf16 routers/norms), 489-496 (fused INT4 draft, grouped verify),
 * 564 (symmetric INT4, group 128).  Compiled with -ffp-contract=off so every a*b+c below is
 * two roundings unless written as fmaf().
 *
 *   orc_warp_dot     fixed-order dot: lane t owns 8-element chunks t, t+32, ... (fmaf in
 *                    order), then an xor-butterfly over 32 lanes (16,8,4,2,1)
 *   orc_sumsq_cta    fixed-order sum of squares: thread t of 256 owns float4 chunks t, t+256..,
 *                    xor-butterfly per warp, then warp partials summed 0..7
 *   orc_rmsnorm      r = 1/sqrtf(sumsq/d + eps); xn = bf16((h*r)*gamma)
 *   orc_det_exp      range-reduced degree-7 polynomial exp (same ops as the device)
 *   orc_router_topk  logits -> top-k (desc, tie -> lower id) -> softmax over the selection
 *   orc_gen_bf16     the counter-hash weight generator (oracle/model.py uniform/gen, restated
 *                    in C only for speed; pinned to the numpy version by test_oracle_cpu)
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline float bf2f(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }
static inline uint16_t f2bf(float f) {
  uint32_t u; memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

float orc_warp_dot(const uint16_t* x, const uint16_t* w, int n) {
  float lane[32];
  int nchunks = n / 8;
  for (int t = 0; t < 32; ++t) {
    float acc = 0.0f;
    for (int c = t; c < nchunks; c += 32)
      for (int e = 0; e < 8; ++e) acc = fmaf(bf2f(x[8 * c + e]), bf2f(w[8 * c + e]), acc);
    lane[t] = acc;
  }
  for (int off = 16; off >= 1; off >>= 1) {
    float nv[32];
    for (int t = 0; t < 32; ++t) nv[t] = lane[t] + lane[t ^ off];
    memcpy(lane, nv, sizeof(nv));
  }
  return lane[0];
}

float orc_sumsq_cta(const float* h, int d) {
  float thr[256];
  int nchunks = d / 4;
  for (int t = 0; t < 256; ++t) {
    float acc = 0.0f;
    for (int c = t; c < nchunks; c += 256)
      for (int e = 0; e < 4; ++e) acc = fmaf(h[4 * c + e], h[4 * c + e], acc);
    thr[t] = acc;
  }
  float part[8];
  for (int wp = 0; wp < 8; ++wp) {
    float lane[32];
    for (int t = 0; t < 32; ++t) lane[t] = thr[wp * 32 + t];
    for (int off = 16; off >= 1; off >>= 1) {
      float nv[32];
      for (int t = 0; t < 32; ++t) nv[t] = lane[t] + lane[t ^ off];
      memcpy(lane, nv, sizeof(nv));
    }
    part[wp] = lane[0];
  }
  float tot = part[0];
  for (int wp = 1; wp < 8; ++wp) tot = tot + part[wp];
  return tot;
}

void orc_rmsnorm(const float* h, const uint16_t* gamma, int d, float eps, uint16_t* out) {
  float ss = orc_sumsq_cta(h, d);
  float ms = ss / (float)d;
  float r = 1.0f / sqrtf(ms + eps);
  for (int i = 0; i < d; ++i) out[i] = f2bf((h[i] * r) * bf2f(gamma[i]));
}

float orc_det_exp(float x) {
  x = fminf(fmaxf(x, -87.0f), 88.0f);
  float t = x * 1.44269504088896341f;
  float n = rintf(t);
  float r = fmaf(n, -0.693145751953125f, x);
  r = fmaf(n, -1.428606820309417232e-6f, r);
  float p = 1.9841270e-4f;
  p = fmaf(p, r, 1.3888889e-3f);
  p = fmaf(p, r, 8.3333333e-3f);
  p = fmaf(p, r, 4.1666667e-2f);
  p = fmaf(p, r, 1.6666667e-1f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  int ni = (int)n;
  uint32_t sb = (uint32_t)(ni + 127) << 23;
  float s; memcpy(&s, &sb, 4);
  return p * s;
}

/* logits[e] for e < E, then top-k + renormalised softmax.  ids/wts have K entries. */
void orc_router_topk(const uint16_t* xn, const uint16_t* wr, int E, int d, int K,
                     float* logits, int32_t* ids, float* wts) {
  for (int e = 0; e < E; ++e) logits[e] = orc_warp_dot(xn, wr + (size_t)e * d, d);
  unsigned char used[1024];
  memset(used, 0, sizeof(used));
  for (int j = 0; j < K; ++j) {
    int best = -1;
    for (int e = 0; e < E; ++e) {
      if (used[e]) continue;
      if (best < 0 || logits[e] > logits[best]) best = e;  /* strict: tie keeps lower id */
    }
    used[best] = 1;
    ids[j] = best;
  }
  float m = logits[ids[0]];
  float ex[64], s = 0.0f;
  for (int j = 0; j < K; ++j) { ex[j] = orc_det_exp(logits[ids[j]] - m); s = s + ex[j]; }
  for (int j = 0; j < K; ++j) wts[j] = ex[j] / s;
}

/* LM head: logits[t][v] = warp_dot(xn[t], lm[v]); argmax tie -> lower id. */
void orc_lm_head(const uint16_t* xn, const uint16_t* lm, int T, int V, int d, float* logits,
                 int32_t* argmax) {
  for (int t = 0; t < T; ++t) {
    int best = 0;
    for (int v = 0; v < V; ++v) {
      float z = orc_warp_dot(xn + (size_t)t * d, lm + (size_t)v * d, d);
      logits[(size_t)t * V + v] = z;
      if (z > logits[(size_t)t * V + best]) best = v;
    }
    argmax[t] = best;
  }
}

/* silu-gated activation for one token: a[i] = bf16(silu(g_i) * u_i) with g,u fp32 inputs. */
void orc_act(const float* g, const float* u, int f, uint16_t* a) {
  for (int i = 0; i < f; ++i) {
    float s = g[i] / (1.0f + orc_det_exp(-g[i]));
    a[i] = f2bf(s * u[i]);
  }
}

/* w[i] = bf16(val(start + i) * scale), val(idx) = ((mix(key + idx*STEP) >> 40) - 2^23 + 0.5) * 2^-23 */
static inline uint64_t orc_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
void orc_gen_bf16(uint64_t key, uint64_t start, int64_t n, float scale, uint16_t* out) {
  for (int64_t i = 0; i < n; ++i) {
    const uint64_t z = orc_mix(key + (start + (uint64_t)i) * 0xD1B54A32D192ED03ull);
    const int32_t hi = (int32_t)(z >> 40) - (1 << 23);
    const float v = ((float)hi + 0.5f) * (1.0f / 8388608.0f);
    out[i] = f2bf(v * scale);
  }
}
