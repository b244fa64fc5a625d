// Shared-KV decode attention for the draft step and the verify window (the
// draft and the target share the bf16 attention weights and ONE KV cache; a rejected draft is
// rolled back by resetting the committed length -- the next cycle's writes overwrite the stale
// rows).
//
// Per layer (live.cpp):  K1 (combine + attention RMSNorm) -> QKV projection (dense tcgen05 GEMM,
// k_umma_grouped with one group of T tokens) -> k_attn_window -> O projection (dense tcgen05
// GEMM) -> K1 (dense combine h += o, MoE RMSNorm, router).
//
// k_attn_partial + k_attn_combine: split-K over the context per (window token t, KV head g).  The window's own keys/values come
// straight from the QKV GEMM's fp32 split planes (summed in split order, rounded to bf16 -- the
// same bf16 values the cache stores), so tokens of one window never wait on each other's cache
// writes; positions before the window are read from the cache.  The CTA writes its token's K/V
// row into the cache for later steps.  Scores for the G = H/Hkv query heads that share the KV
// head are kept in shared memory (context <= P positions), softmax in fp32, output bf16.
// Latency-bound: the context is a few hundred positions x 4 KB of K/V per layer (Phi).
#include "common.cuh"
#include "kernels.h"

namespace mspq {
namespace {

constexpr int AT_THREADS = 256, AT_WARPS = AT_THREADS / 32, AT_MAXG = 8;
constexpr int AT_SPLITS = 16, AT_MAXPOS = 4096, AT_MAXCHUNK = AT_MAXPOS / AT_SPLITS;
constexpr int AT_MAXSPLIT = 8;  // QKV projection K-split planes (the engine's kMaxSplit)
constexpr int AT_PRE = 2;       // keys per warp whose K and V rows are loaded before the score loop (<= 2)

MSPQ_D float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Split-K (flash-decoding) over the context: CTA (t, g, s) takes key positions
// [s*chunk, (s+1)*chunk) of token t's causal range (chunk = ceil(n / AT_SPLITS)), so a T = 1 draft
// step still spreads over Hkv x AT_SPLITS CTAs.  Lane l owns head dims [VEC*l, VEC*l + VEC)
// (Dh = 32 VEC): q in registers, one vector load per key row; warps stride over the chunk's keys.
// Each CTA leaves (max, sum of exp, unnormalised V sum) per head; k_attn_combine merges the
// AT_SPLITS partials in split order (deterministic) and writes bf16.
MSPQ_D int attn_chunk(int n) { return (n + AT_SPLITS - 1) / AT_SPLITS; }

// merge the AT_SPLITS partials of (t, g) in split order: o = sum_s e^(m_s - M) acc_s / sum_s e^(m_s - M) l_s
// (run by the last of the (t, g) CTAs to finish; the partials are read from L2)
MSPQ_D void attn_merge(const AttnArgs& a, int t, int g) {
  const int G = a.H / a.Hkv, Dh = a.Dh, Nq = a.H * Dh;
  const float* part = a.part + ((size_t)t * a.Hkv + g) * AT_SPLITS * (size_t)G * (Dh + 2);
  const size_t ps = (size_t)G * (Dh + 2);
  for (int o = threadIdx.x; o < G * Dh; o += AT_THREADS) {
    const int i = o / Dh;
    float ms[AT_SPLITS];
#pragma unroll
    for (int s = 0; s < AT_SPLITS; ++s) ms[s] = __ldcg(part + s * ps + i);
    float M = -INFINITY;
#pragma unroll
    for (int s = 0; s < AT_SPLITS; ++s) M = fmaxf(M, ms[s]);
    float den = 0.0f, num = 0.0f;
#pragma unroll
    for (int s = 0; s < AT_SPLITS; ++s) {
      if (ms[s] == -INFINITY) continue;
      const float w = __expf(__fsub_rn(ms[s], M));
      den = fmaf(w, __ldcg(part + s * ps + G + i), den);
      num = fmaf(w, __ldcg(part + s * ps + 2 * G + o), num);
    }
    const uint16_t ob = f2bf(__fdiv_rn(num, den));
    const int col = g * G * Dh + o;
    if (a.out) a.out[(int64_t)t * Nq + col] = ob;
    if (a.oimg) *reinterpret_cast<uint16_t*>(a.oimg + (int64_t)(col >> 6) * (a.o_bn * 128) + sw128_off(t, col & 63)) = ob;
  }
}

template <int VEC, int MG>  // MG: register arrays sized for G = H / Hkv <= MG (4 or AT_MAXG)
__global__ void __launch_bounds__(AT_THREADS, 2) k_attn_partial(AttnArgs a) {
  pdl_enter();  // launched with launch_pdl (kernels.h)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = blockIdx.x, g = blockIdx.y, sp = blockIdx.z;
  const int G = a.H / a.Hkv, Dh = a.Dh;
  const int Nq = a.H * Dh, Nkv = a.Hkv * Dh, Nqkv = Nq + 2 * Nkv;
  // token t of the batch: its window starts at batch row wb, it belongs to request stream s_id
  // (own KV cache) and sits at position pt; one stream: wb = 0, s_id = 0, pt = *pos0 + t
  int wb = 0, s_id = 0, pt;
  if (a.meta) {
    wb = a.meta[3 * t];
    s_id = a.meta[3 * t + 1];
    pt = a.meta[3 * t + 2];
  } else {
    pt = *a.pos0 + t;
  }
  const int tl = t - wb, p0 = pt - tl, n = pt + 1;
  uint16_t* const kc = a.kc + (int64_t)s_id * a.kv_stream_stride;
  uint16_t* const vc = a.vc + (int64_t)s_id * a.kv_stream_stride;
  const int chunk = attn_chunk(n), j0 = sp * chunk, j1 = min(n, j0 + chunk);
  uint16_t* wk = reinterpret_cast<uint16_t*>(smem_raw);     // [T][Dh] in-window keys, bf16
  uint16_t* wv = wk + a.T * Dh;                             // [T][Dh] in-window values
  float* sc = reinterpret_cast<float*>(wv + a.T * Dh);     // [G][chunk] scores -> exp
  float* red = sc + (size_t)G * AT_MAXCHUNK;                // [AT_WARPS][G][Dh] value partials
  __shared__ float hmax[AT_MAXG], hsum[AT_MAXG];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* part = a.part + (((size_t)t * a.Hkv + g) * AT_SPLITS + sp) * (size_t)G * (Dh + 2);
  // (1) the window rows inside this chunk (split planes summed in order, rounded to bf16 like the
  // cache): window tokens tt with p0 + tt in [j0, j1); most chunks hold none
  const int w0 = max(j0, p0) - p0, w1 = j1 - p0;
  for (int i = tid; i < (w1 - w0) * Dh; i += AT_THREADS) {
    const int tt = w0 + i / Dh, dd = i % Dh;
    const float* src = a.qkv + (int64_t)(wb + tt) * Nqkv + Nq + g * Dh + dd;
    // every split's K and V value in flight at once, then summed in split order
    float kr[AT_MAXSPLIT], vr[AT_MAXSPLIT];
#pragma unroll
    for (int s = 0; s < AT_MAXSPLIT; ++s) {
      kr[s] = s < a.splits ? src[s * a.split_stride] : 0.0f;
      vr[s] = s < a.splits ? src[s * a.split_stride + Nkv] : 0.0f;
    }
    float kv = 0.0f, vv = 0.0f;
#pragma unroll
    for (int s = 0; s < AT_MAXSPLIT; ++s)
      if (s < a.splits) {
        kv = __fadd_rn(kv, kr[s]);
        vv = __fadd_rn(vv, vr[s]);
      }
    wk[tt * Dh + dd] = f2bf(kv);
    wv[tt * Dh + dd] = f2bf(vv);
  }
  // q: the lane's VEC dims of the G heads, split planes summed in order; two splits' vector loads
  // (2 G of them) in flight per step
  float q[MG][VEC];
#pragma unroll
  for (int i = 0; i < MG; ++i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) q[i][v] = 0.0f;
  const float* qsrc = a.qkv + (int64_t)t * Nqkv + (g * G) * Dh + lane * VEC;
  for (int s0 = 0; s0 < a.splits; s0 += 2) {
    float qr[2][MG][VEC];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int i = 0; i < MG; ++i) {
        const bool ok = i < G && s0 + u < a.splits;
        const float* src = qsrc + (int64_t)(s0 + u) * a.split_stride + i * Dh;
        if (VEC == 4) {
          const float4 f = ok ? *reinterpret_cast<const float4*>(src) : make_float4(0.f, 0.f, 0.f, 0.f);
          qr[u][i][0] = f.x;
          qr[u][i][1] = f.y;
          qr[u][i][2 % VEC] = f.z;
          qr[u][i][3 % VEC] = f.w;
        } else {
          const float2 f = ok ? *reinterpret_cast<const float2*>(src) : make_float2(0.f, 0.f);
          qr[u][i][0] = f.x;
          qr[u][i][1] = f.y;
        }
      }
#pragma unroll
    for (int u = 0; u < 2; ++u)
      if (s0 + u < a.splits)
#pragma unroll
        for (int i = 0; i < MG; ++i)
#pragma unroll
          for (int v = 0; v < VEC; ++v) q[i][v] = __fadd_rn(q[i][v], qr[u][i][v]);
  }
  __syncthreads();
  if (j0 <= pt && pt < j1)  // the chunk holding the token's own position writes its cache row
    for (int dd = tid; dd < Dh; dd += AT_THREADS) {
      kc[((int64_t)pt * a.Hkv + g) * Dh + dd] = wk[tl * Dh + dd];
      vc[((int64_t)pt * a.Hkv + g) * Dh + dd] = wv[tl * Dh + dd];
    }
  auto row_vec = [&](const uint16_t* cache, const uint16_t* win, int j, float* o) {
    const uint16_t* r = (j < p0 ? cache + ((int64_t)j * a.Hkv + g) * Dh : win + (j - p0) * Dh) + lane * VEC;
    if (VEC == 4) {
      const uint2 u = *reinterpret_cast<const uint2*>(r);
      o[0] = __uint_as_float(u.x << 16);
      o[1] = __uint_as_float(u.x & 0xffff0000u);
      o[2] = __uint_as_float(u.y << 16);
      o[3] = __uint_as_float(u.y & 0xffff0000u);
    } else {
      const uint32_t u = *reinterpret_cast<const uint32_t*>(r);
      o[0] = __uint_as_float(u << 16);
      o[1] = __uint_as_float(u & 0xffff0000u);
    }
  };
  // the warp's first AT_PRE keys: K AND V rows loaded together up front (one memory round trip
  // instead of one per key and per operand; short decode contexts have <= 2 keys per warp)
  float kpre[AT_PRE][VEC], vpre[AT_PRE][VEC];
#pragma unroll
  for (int p = 0; p < AT_PRE; ++p) {
    const int j = j0 + warp + p * AT_WARPS;
    if (j < j1) {
      row_vec(kc, wk, j, kpre[p]);
      row_vec(vc, wv, j, vpre[p]);
    }
  }
  // (2) scores of this chunk
  for (int j = j0 + warp, p = 0; j < j1; j += AT_WARPS, ++p) {
    float kk[VEC];
    if (p < AT_PRE) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) kk[v] = p == 0 ? kpre[0][v] : kpre[AT_PRE - 1][v];  // static indices
    } else {
      row_vec(kc, wk, j, kk);
    }
#pragma unroll
    for (int i = 0; i < MG; ++i)
      if (i < G) {
        float pp = 0.0f;
#pragma unroll
        for (int v = 0; v < VEC; ++v) pp = fmaf(q[i][v], kk[v], pp);
        pp = warp_butterfly_sum(pp);
        if (lane == 0) sc[i * AT_MAXCHUNK + (j - j0)] = __fmul_rn(pp, a.scale);
      }
  }
  __syncthreads();
  // (3) chunk max and exp sums per head (warp i owns head i)
  if (warp < G) {
    float* sr = sc + warp * AT_MAXCHUNK;
    float m = -INFINITY;
    for (int j = lane; j < j1 - j0; j += 32) m = fmaxf(m, sr[j]);
    m = warp_max(m);
    float s = 0.0f;
    for (int j = lane; j < j1 - j0; j += 32) {
      const float e = __expf(__fsub_rn(sr[j], m));
      sr[j] = e;
      s = __fadd_rn(s, e);
    }
    s = warp_butterfly_sum(s);
    if (lane == 0) {
      hmax[warp] = m;
      hsum[warp] = s;
    }
  }
  __syncthreads();
  // (4) unnormalised value sums, per-warp partials added in warp order
  float acc[MG][VEC];
#pragma unroll
  for (int i = 0; i < MG; ++i)
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[i][v] = 0.0f;
  for (int j = j0 + warp, p = 0; j < j1; j += AT_WARPS, ++p) {
    float vv[VEC];
    if (p < AT_PRE) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) vv[v] = p == 0 ? vpre[0][v] : vpre[AT_PRE - 1][v];
    } else {
      row_vec(vc, wv, j, vv);
    }
#pragma unroll
    for (int i = 0; i < MG; ++i)
      if (i < G) {
        const float pj = sc[i * AT_MAXCHUNK + (j - j0)];
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc[i][v] = fmaf(pj, vv[v], acc[i][v]);
      }
  }
#pragma unroll
  for (int i = 0; i < MG; ++i)
    if (i < G)
#pragma unroll
      for (int v = 0; v < VEC; ++v) red[((size_t)warp * G + i) * Dh + lane * VEC + v] = acc[i][v];
  __syncthreads();
  for (int o = tid; o < G * Dh; o += AT_THREADS) {
    float x = 0.0f;
#pragma unroll
    for (int w = 0; w < AT_WARPS; ++w) x = __fadd_rn(x, red[(size_t)w * G * Dh + o]);
    part[2 * G + o] = x;
  }
  if (tid < G) {
    part[tid] = j1 > j0 ? hmax[tid] : -INFINITY;
    part[G + tid] = j1 > j0 ? hsum[tid] : 0.0f;
  }
  // the last of the AT_SPLITS CTAs of (t, g) merges (threadfence-reduction pattern); it resets
  // the counter, so the workspace stays zeroed between launches
  __shared__ int last;
  __threadfence();
  __syncthreads();
  int* cnt = a.cnt + t * a.Hkv + g;
  if (tid == 0) last = atomicAdd(cnt, 1) == AT_SPLITS - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  attn_merge(a, t, g);
  if (tid == 0) *cnt = 0;
}

}  // namespace

size_t attn_smem_bytes(int T, int H, int Hkv, int Dh, int P) {
  const int G = H / Hkv;
  (void)P;
  return (size_t)2 * T * Dh * 2 + (size_t)G * AT_MAXCHUNK * 4 + (size_t)AT_WARPS * G * Dh * 4;
}
size_t attn_part_floats(int T, int H, int Hkv, int Dh) {  // merge counters + partials, in 4-byte words
  return (size_t)AT_CNT + (size_t)T * Hkv * AT_SPLITS * (size_t)(H / Hkv) * (Dh + 2);
}

cudaError_t launch_attn_window(const AttnArgs& a0, cudaStream_t st) {
  if (a0.P > AT_MAXPOS || a0.T * a0.Hkv > AT_CNT || a0.splits < 1 || a0.splits > AT_MAXSPLIT)
    return cudaErrorInvalidValue;
  AttnArgs a = a0;
  a.cnt = reinterpret_cast<int*>(a0.part);
  a.part = a0.part + AT_CNT;
  const size_t smem = attn_smem_bytes(a.T, a.H, a.Hkv, a.Dh, a.P);
  const dim3 grid(a.T, a.Hkv, AT_SPLITS);
  cudaError_t e;
  auto go = [&](auto kern) {
    cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem);
    return e2 == cudaSuccess ? launch_pdl(kern, grid, dim3(AT_THREADS), smem, st, a) : e2;
  };
  const bool g4 = a.H / a.Hkv <= 4;
  if (a.Dh == 128)
    e = g4 ? go(k_attn_partial<4, 4>) : go(k_attn_partial<4, AT_MAXG>);
  else if (a.Dh == 64)
    e = g4 ? go(k_attn_partial<2, 4>) : go(k_attn_partial<2, AT_MAXG>);
  else
    return cudaErrorInvalidValue;
  return e;
}

}  // namespace mspq
