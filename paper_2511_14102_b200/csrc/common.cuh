// Shared device helpers for the MoE-SpeQ B200 decode path (sm_100a).
//
// Numerics contract: every order-sensitive fp32 reduction whose result feeds
// an integer decision (router logits -> expert ids, LM logits -> token ids) uses a FIXED
// reduction order that oracle/csrc/model_ref.c restates exactly.  Explicit __f*_rn / fmaf
// intrinsics are used wherever nvcc would otherwise contract a*b+c into an FMA.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define MSPQ_HD __host__ __device__ __forceinline__
#define MSPQ_D __device__ __forceinline__
// Dynamic shared-memory limit for kernels whose size varies per launch (K1 staging <= ~205 KB,
// attention): set as a constant, so a captured graph node and a later direct launch of another size
// never race on the function attribute; static smem + this stays under sm_100's 227 KB opt-in.
constexpr int kMaxDynSmem = 210 * 1024;

namespace mspq {

// ------------------------------------------------------------------ bf16 bit helpers
MSPQ_HD float bf2f(uint16_t b) {
#ifdef __CUDA_ARCH__
  return __uint_as_float(((uint32_t)b) << 16);
#else
  uint32_t u = ((uint32_t)b) << 16;
  float f;
  __builtin_memcpy(&f, &u, 4);
  return f;
#endif
}
MSPQ_HD uint16_t f2bf(float f) {  // round to nearest even (finite inputs)
#ifdef __CUDA_ARCH__
  uint32_t u = __float_as_uint(f);
#else
  uint32_t u;
  __builtin_memcpy(&u, &f, 4);
#endif
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

// ------------------------------------------------------------------ counter-based RNG
// splitmix64 finaliser; weight(seed, tensor, idx) is position-independent so any tensor can
// be regenerated anywhere (host oracle, device init) bit-identically.
MSPQ_HD uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
MSPQ_HD uint64_t tensor_key(uint64_t seed, uint64_t tensor) { return mix64(seed ^ mix64(tensor)); }
MSPQ_HD float unit_val(uint64_t key, uint64_t idx) {
  uint64_t z = mix64(key + idx * 0xD1B54A32D192ED03ull);
  int32_t hi = (int32_t)(z >> 40) - (1 << 23);
  return ((float)hi + 0.5f) * (1.0f / 8388608.0f);
}

// tensor ids (oracle/model.py)
enum : uint64_t { T_EMBED = 1, T_POS = 2, T_LM = 3, T_FINAL_GAMMA = 4 };
MSPQ_HD uint64_t t_gamma(int l) { return 0x100ull + (uint64_t)l * 16; }
MSPQ_HD uint64_t t_router(int l) { return 0x100ull + (uint64_t)l * 16 + 1; }
MSPQ_HD uint64_t t_expert(int l, int e, int m) {
  return 0x1000000ull + (((uint64_t)l * 1024 + (uint64_t)e) * 4 + (uint64_t)m);
}

// ------------------------------------------------------------------ deterministic exp
// Range reduction by ln2 (hi/lo split) + degree-7 Horner polynomial, all with fmaf; the
// final 2^n scale is an exact power-of-two multiply.  Same op sequence as orc_det_exp.
MSPQ_D float det_exp(float x) {
  x = fminf(fmaxf(x, -87.0f), 88.0f);
  float t = __fmul_rn(x, 1.44269504088896341f);
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
  float s = __uint_as_float((uint32_t)((int)n + 127) << 23);
  return __fmul_rn(p, s);
}

MSPQ_D float silu_det(float g) { return __fdiv_rn(g, __fadd_rn(1.0f, det_exp(-g))); }

// ------------------------------------------------------------------ warp helpers
// byte offset of bf16 element (row, col) inside one UMMA K-major SWIZZLE_128B image of 64 columns
MSPQ_HD int sw128_off(int row, int col) {
  return (row >> 3) * 1024 + (row & 7) * 128 + ((((col >> 3) ^ (row & 7)) & 7) << 4) + (col & 7) * 2;
}

MSPQ_D float warp_butterfly_sum(float v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
  return v;
}

// 8 bf16 packed in a uint4 -> 8 floats
MSPQ_D void bf16x8_to_f32(const uint4& v, float* o) {
  o[0] = __uint_as_float(v.x << 16);
  o[1] = __uint_as_float(v.x & 0xffff0000u);
  o[2] = __uint_as_float(v.y << 16);
  o[3] = __uint_as_float(v.y & 0xffff0000u);
  o[4] = __uint_as_float(v.z << 16);
  o[5] = __uint_as_float(v.z & 0xffff0000u);
  o[6] = __uint_as_float(v.w << 16);
  o[7] = __uint_as_float(v.w & 0xffff0000u);
}

MSPQ_D uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Fixed-order warp dot over n bf16 (n % 256 == 0): lane owns 8-element chunks lane, lane+32,
// ... accumulated with fmaf in order, then an xor butterfly.  == orc_warp_dot.
// Loads are issued 4 chunks ahead of the (unchanged) accumulation order for memory-level
// parallelism.
MSPQ_D float warp_dot_bf16(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, int n,
                           int lane) {
  float acc = 0.0f;
  const int nchunks = n >> 3;
  int c = lane;
  for (; c + 96 < nchunks; c += 128) {
    uint4 wv[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      wv[u] = ldg_nc_v4(w + 8 * (c + 32 * u));
      xv[u] = *reinterpret_cast<const uint4*>(x + 8 * (c + 32 * u));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float xf[8], wf[8];
      bf16x8_to_f32(xv[u], xf);
      bf16x8_to_f32(wv[u], wf);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc = fmaf(xf[e], wf[e], acc);
    }
  }
  for (; c < nchunks; c += 32) {
    uint4 xv = *reinterpret_cast<const uint4*>(x + 8 * c);
    uint4 wv = ldg_nc_v4(w + 8 * c);
    float xf[8], wf[8];
    bf16x8_to_f32(xv, xf);
    bf16x8_to_f32(wv, wf);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc = fmaf(xf[e], wf[e], acc);
  }
  return warp_butterfly_sum(acc);
}

// Two fixed-order warp dots sharing x (each identical to warp_dot_bf16), loads interleaved.
MSPQ_D void warp_dot2_bf16(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w0,
                           const uint16_t* __restrict__ w1, int n, int lane, float& z0, float& z1) {
  float a0 = 0.0f, a1 = 0.0f;
  const int nchunks = n >> 3;
  int c = lane;
  // 8 chunks of each row in flight per step (16 weight loads per lane); x comes from shared memory
  for (; c + 224 < nchunks; c += 256) {
    uint4 v0[8], v1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      v0[u] = ldg_nc_v4(w0 + 8 * (c + 32 * u));
      v1[u] = ldg_nc_v4(w1 + 8 * (c + 32 * u));
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint4 xv = *reinterpret_cast<const uint4*>(x + 8 * (c + 32 * u));
      float xf[8], f0[8], f1[8];
      bf16x8_to_f32(xv, xf);
      bf16x8_to_f32(v0[u], f0);
      bf16x8_to_f32(v1[u], f1);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        a0 = fmaf(xf[e], f0[e], a0);
        a1 = fmaf(xf[e], f1[e], a1);
      }
    }
  }
  for (; c + 96 < nchunks; c += 128) {
    uint4 v0[4], v1[4], xv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v0[u] = ldg_nc_v4(w0 + 8 * (c + 32 * u));
      v1[u] = ldg_nc_v4(w1 + 8 * (c + 32 * u));
      xv[u] = *reinterpret_cast<const uint4*>(x + 8 * (c + 32 * u));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      float xf[8], f0[8], f1[8];
      bf16x8_to_f32(xv[u], xf);
      bf16x8_to_f32(v0[u], f0);
      bf16x8_to_f32(v1[u], f1);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        a0 = fmaf(xf[e], f0[e], a0);
        a1 = fmaf(xf[e], f1[e], a1);
      }
    }
  }
  for (; c < nchunks; c += 32) {
    const uint4 xv = *reinterpret_cast<const uint4*>(x + 8 * c);
    const uint4 v0 = ldg_nc_v4(w0 + 8 * c), v1 = ldg_nc_v4(w1 + 8 * c);
    float xf[8], f0[8], f1[8];
    bf16x8_to_f32(xv, xf);
    bf16x8_to_f32(v0, f0);
    bf16x8_to_f32(v1, f1);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      a0 = fmaf(xf[e], f0[e], a0);
      a1 = fmaf(xf[e], f1[e], a1);
    }
  }
  z0 = warp_butterfly_sum(a0);
  z1 = warp_butterfly_sum(a1);
}


// ---- mbarrier + 1-D bulk copy (cp.async.bulk) helpers, shared by the tcgen05 kernels and K1
MSPQ_D uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

MSPQ_D void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(bar)), "r"(count) : "memory");
}
MSPQ_D void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
MSPQ_D bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// bounded wait: a lost arrival traps (error) instead of hanging the GPU
MSPQ_D void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(bar, parity))
    if (clock64() - t0 > 4000000000LL) __trap();
}
MSPQ_D void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
MSPQ_D void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
MSPQ_D void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
// fire-and-forget L2 prefetch of [src, src + bytes) (bytes a multiple of 16)
MSPQ_D void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

}  // namespace mspq
