// Shared-KV decode attention for the draft step and the verify window (the
// draft and the target share the bf16 attention weights and ONE KV cache; a rejected draft is
// rolled back by resetting the committed length -- the next cycle's writes overwrite the stale
// rows).
//
// Per layer (live.cpp):  K1 (combine + attention RMSNorm) -> QKV projection (dense tcgen05 GEMM,
// k_umma_grouped with one group of T tokens) -> k_attn_window -> O projection (dense tcgen05
// GEMM) -> K1 (dense combine h += o, MoE RMSNorm, router).
//
// k_attn_window: one CTA per (window token t, KV head g).  The window's own keys/values come
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

MSPQ_D float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(AT_THREADS) k_attn_window(AttnArgs a) {
  pdl_enter();  // launched with launch_pdl (kernels.h)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int t = blockIdx.x, g = blockIdx.y;
  const int G = a.H / a.Hkv, Dh = a.Dh;
  const int Nq = a.H * Dh, Nkv = a.Hkv * Dh, Nqkv = Nq + 2 * Nkv;
  const int p0 = *a.pos0, pt = p0 + t, n = pt + 1;
  float* qs = reinterpret_cast<float*>(smem_raw);        // [G][Dh] fp32
  uint16_t* wk = reinterpret_cast<uint16_t*>(qs + G * Dh);  // [T][Dh] in-window keys, bf16
  uint16_t* wv = wk + a.T * Dh;                              // [T][Dh] in-window values
  float* sc = reinterpret_cast<float*>(wv + a.T * Dh);      // [G][P] scores -> probabilities
  __shared__ float hsum[AT_MAXG];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // (1) q of the G heads (their columns are contiguous), in-window k/v of tokens 0..t
  for (int i = tid; i < G * Dh; i += AT_THREADS) {
    const float* src = a.qkv + (int64_t)t * Nqkv + g * G * Dh + i;
    float v = 0.0f;
    for (int s = 0; s < a.splits; ++s) v = __fadd_rn(v, src[s * a.split_stride]);
    qs[i] = v;
  }
  for (int i = tid; i < (t + 1) * Dh; i += AT_THREADS) {
    const int tt = i / Dh, dd = i - tt * Dh;
    const float* src = a.qkv + (int64_t)tt * Nqkv + Nq + g * Dh + dd;
    float kv = 0.0f, vv = 0.0f;
    for (int s = 0; s < a.splits; ++s) {
      kv = __fadd_rn(kv, src[s * a.split_stride]);
      vv = __fadd_rn(vv, src[s * a.split_stride + Nkv]);
    }
    wk[i] = f2bf(kv);
    wv[i] = f2bf(vv);
  }
  __syncthreads();
  for (int dd = tid; dd < Dh; dd += AT_THREADS) {  // this token's row of the shared cache
    a.kc[((int64_t)pt * a.Hkv + g) * Dh + dd] = wk[t * Dh + dd];
    a.vc[((int64_t)pt * a.Hkv + g) * Dh + dd] = wv[t * Dh + dd];
  }
  // (2) scores, one warp per key position
  for (int j = warp; j < n; j += AT_WARPS) {
    const uint16_t* kr = j < p0 ? a.kc + ((int64_t)j * a.Hkv + g) * Dh : wk + (j - p0) * Dh;
    float part[AT_MAXG];
#pragma unroll
    for (int i = 0; i < AT_MAXG; ++i) part[i] = 0.0f;
    for (int dd = lane; dd < Dh; dd += 32) {
      const float kk = bf2f(kr[dd]);
#pragma unroll
      for (int i = 0; i < AT_MAXG; ++i)
        if (i < G) part[i] = fmaf(qs[i * Dh + dd], kk, part[i]);
    }
#pragma unroll
    for (int i = 0; i < AT_MAXG; ++i)
      if (i < G) {
        const float z = warp_butterfly_sum(part[i]);
        if (lane == 0) sc[i * a.P + j] = __fmul_rn(z, a.scale);
      }
  }
  __syncthreads();
  // (3) softmax numerators per head (warp i owns head i)
  if (warp < G) {
    float* sr = sc + warp * a.P;
    float m = -INFINITY;
    for (int j = lane; j < n; j += 32) m = fmaxf(m, sr[j]);
    m = warp_max(m);
    float s = 0.0f;
    for (int j = lane; j < n; j += 32) {
      const float e = __expf(__fsub_rn(sr[j], m));
      sr[j] = e;
      s = __fadd_rn(s, e);
    }
    s = warp_butterfly_sum(s);
    if (lane == 0) hsum[warp] = s;
  }
  __syncthreads();
  // (4) o = sum_j p_j v_j / sum_j p_j
  for (int o = tid; o < G * Dh; o += AT_THREADS) {
    const int i = o / Dh, dd = o - i * Dh;
    const float* pr = sc + i * a.P;
    float acc = 0.0f;
    for (int j = 0; j < n; ++j) {
      const uint16_t* vr = j < p0 ? a.vc + ((int64_t)j * a.Hkv + g) * Dh : wv + (j - p0) * Dh;
      acc = fmaf(pr[j], bf2f(vr[dd]), acc);
    }
    a.out[(int64_t)t * Nq + g * G * Dh + o] = f2bf(__fdiv_rn(acc, hsum[i]));
  }
}

}  // namespace

size_t attn_smem_bytes(int T, int H, int Hkv, int Dh, int P) {
  const int G = H / Hkv;
  return (size_t)G * Dh * 4 + (size_t)2 * T * Dh * 2 + (size_t)G * P * 4;
}

cudaError_t launch_attn_window(const AttnArgs& a, cudaStream_t st) {
  const size_t smem = attn_smem_bytes(a.T, a.H, a.Hkv, a.Dh, a.P);
  cudaError_t e = cudaFuncSetAttribute(k_attn_window, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(k_attn_window, dim3(a.T, a.Hkv), dim3(AT_THREADS), smem, st, a);
}

}  // namespace mspq
