// K3 v2: the bf16 verify expert FFN as a tcgen05 grouped GEMM (swap-AB) on sm_100a.
//
//   D[128 weight rows, BN tokens] += W_tile[128 x 64] . X_tile[BN x 64]^T      (kind::f16, fp32 acc)
//
// The weight operand (M = 128) is the expert matrix streamed from the HBM slot pool; the
// tokens of one expert group (<= k+1 of them, reorder_verification) are the N = 16/32 operand.
// Experts are stored TILE-MAJOR: each 128-row x 64-column block is a contiguous 16 KB image of
// the UMMA K-major SWIZZLE_128B canonical layout, so one cp.async.bulk (TMA bulk copy) lands it
// in shared memory ready for the tensor core -- no register staging, no tensor-map per buffer.
//
// CTA = 6 warps: warp 0 = bulk-copy producer, warp 1 = TMEM allocator + single-thread MMA
// issuer, warps 2-5 = epilogue (TMEM lanes 32*(w%4)..+31 -> registers -> fp32 partials).
// One CTA per (group, 128-row tile, K split); K splits write separate partial planes that the
// consumer sums in fixed order (deterministic, no atomics).
#include <cstdlib>
#include "common.cuh"
#include "kernels.h"

namespace mspq {
namespace {

constexpr int BM = 128, BK = 64, TILE_A = BM * BK * 2;

// try_wait with a suspend-time hint: the waiting warp sleeps until the phase completes (or
// ~1 ms passes) instead of spinning and stealing issue slots from the working warps
MSPQ_D bool mbar_try_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(bar)), "r"(parity), "r"(1000000u)
      : "memory");
  return ok != 0;
}
MSPQ_D void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  if (mbar_try_sleep(bar, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try_sleep(bar, parity))
    if (clock64() - t0 > 4000000000LL) __trap();
}
MSPQ_D void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
MSPQ_D void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

MSPQ_D uint64_t sw128_desc(uint32_t saddr) {
  // start>>4 [0,14) | LBO=1 [16,30) | SBO=1024>>4 [32,46) | version 1 [46,48) | SWIZZLE_128B [61,64)
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, M=128, N=n
__host__ __device__ constexpr uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
// kind::f16 instruction descriptor with fp16 A/B (format 0), D f32, both K-major
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
MSPQ_D void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}
MSPQ_D void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
MSPQ_D void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// byte offset of element (row, col) inside one SW128 K-major image with 64 columns per row
MSPQ_D void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}


template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1) k_umma_grouped(UmmaArgs a) {
  // launched with launch_pdl (kernels.h); with a.early_a only the producer's B loads and the
  // global writes wait for the predecessor (UmmaArgs::early_a)
  if (!a.early_a) pdl_enter();
  const int S = a.splits, RT = a.rows / BM;
  const int unit = blockIdx.x;
  const int s = unit % S, rt = (unit / S) % RT, g = unit / (S * RT);
  if (g >= *a.n_groups || !gmask_has(a.gmask, g)) return;
  const int kb_total = a.kdim / BK;
  const int per = (kb_total + S - 1) / S;
  const int kb0 = s * per, nk = max(0, min(kb_total, kb0 + per) - kb0);
  const int e0 = a.group_off[g], m = a.group_off[g + 1] - e0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* outp = a.out + (int64_t)s * a.out_split_stride;
  if (nk == 0) {  // empty split: contribute zeros
    if (a.early_a) pdl_enter();
    for (int i = threadIdx.x; i < m * BM; i += blockDim.x)
      outp[(int64_t)(e0 + i / BM) * a.rows + rt * BM + (i % BM)] = 0.0f;
    return;
  }
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = base;
  unsigned char* sB = base + STAGES * TILE_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * BN * 128);
  uint64_t* empty = full + STAGES;
  uint64_t* accf = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // with early_a every thread but the producer waits here (nothing to do before B lands anyway)
  if (a.early_a && threadIdx.x != 0) pdl_enter();
  if (warp == 0) {
    if (lane == 0) {  // producer
      const unsigned char* wsrc = a.w_base + (int64_t)a.group_buf[g] * a.blob_bytes + a.w_off +
                                  ((int64_t)rt * kb_total + kb0) * TILE_A;
      const unsigned char* bsrc = a.bimg + ((int64_t)g * kb_total + kb0) * (BN * 128);
      int i0 = 0;
      if (a.early_a) {  // the ring's first A tiles before the wait, their B tiles after it
        i0 = min(nk, STAGES);
        for (int i = 0; i < i0; ++i) {
          mbar_expect_tx(&full[i], TILE_A + BN * 128);
          bulk_g2s(sA + i * TILE_A, wsrc + (int64_t)i * TILE_A, TILE_A, &full[i]);
        }
        pdl_enter();
        for (int i = 0; i < i0; ++i) bulk_g2s(sB + i * BN * 128, bsrc + (int64_t)i * BN * 128, BN * 128, &full[i]);
      }
      for (int i = i0; i < nk; ++i) {
        const int st = i % STAGES, r = i / STAGES;
        if (r > 0) mbar_wait(&empty[st], (r - 1) & 1);
        mbar_expect_tx(&full[st], TILE_A + BN * 128);
        bulk_g2s(sA + st * TILE_A, wsrc + (int64_t)i * TILE_A, TILE_A, &full[st]);
        bulk_g2s(sB + st * BN * 128, bsrc + (int64_t)i * BN * 128, BN * 128, &full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = idesc_bf16(BN);
      for (int i = 0; i < nk; ++i) {
        const int st = i % STAGES, r = i / STAGES;
        mbar_wait(&full[st], r & 1);
        tc_fence_after();
        const uint64_t da = sw128_desc(su32(sA + st * TILE_A));
        const uint64_t db = sw128_desc(su32(sB + st * BN * 128));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)  // +32 bytes per K=16 step inside the 128-byte swizzle row
          umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (i | k) != 0);
        umma_commit(&empty[st]);
      }
      umma_commit(accf);
    }
  } else {  // epilogue warps 2..5
    mbar_wait(accf, 0);
    tc_fence_after();
    const int q = warp & 3;
    const int row = rt * BM + q * 32 + lane;
    float v[BN];
    tmem_ld16(tmem + ((uint32_t)(q * 32) << 16), v);
    if (BN == 32) tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + 16, v + 16);
    if (a.act_img) {
      // W13 with one K split: rows 2i / 2i+1 are gate_i / up_i in adjacent lanes; act =
      // bf16(silu(gate) * up) goes straight into the W2 B image (k_finalize_act's arithmetic)
      const int i = row >> 1, kbt2 = (a.rows >> 1) / BK;
      unsigned char* img = a.act_img + ((int64_t)g * kbt2 + i / BK) * (BN * 128);
#pragma unroll
      for (int t = 0; t < BN; ++t) {
        const float up = __shfl_down_sync(0xffffffffu, v[t], 1);
        if (t < m && (lane & 1) == 0)
          *reinterpret_cast<uint16_t*>(img + sw128_off(t, i % BK)) = f2bf(__fmul_rn(silu_det(v[t]), up));
      }
    } else {
#pragma unroll
      for (int t = 0; t < BN; ++t)
        if (t < m) outp[(int64_t)(e0 + t) * a.rows + row] = v[t];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
  }
}

// K2 B operand (F16): the draft GEMM runs kind::f16 on fp16 operands.  A k-block's columns
// 0..31 are "class 1" (A = 1024 + q), columns 32..63 "class 16" (A = 1024 + 16 q), so the token
// image holds b = fp16(x) for class 1 and b = fp16(x / 16) for class 16, and
//   sum_k (q_k - 8) x_k = D - sum_k c_k b_k,   c = 1032 (class 1) | 1152 (class 16)
// (class 1: (1024 + q) b - 1032 b = (q - 8) b; class 16: (1024 + 16q) b - 1152 b = (q - 8) 16 b).
// csum[g][row][kb] = sum over the k-block of c_k b_k in fp32, fixed reduction order.
MSPQ_D uint16_t f2h_bits(float v) {
  const __half h = __float2half_rn(v);
  return *reinterpret_cast<const uint16_t*>(&h);
}
MSPQ_D float h2f_bits(uint16_t b) { return __half2float(*reinterpret_cast<const __half*>(&b)); }

// Gather the tokens of every group into the SW128 B images [G][kdim/64][BN x 64]: bf16 (K3), or
// class-scaled fp16 plus csum (K2, F16).
template <bool F16>
__global__ void k_gather_b(const uint16_t* __restrict__ x, int ld, SchedPtrs s, int kdim, int BN,
                           unsigned char* __restrict__ img, float* __restrict__ csum) {
  pdl_enter();
  const int kb = blockIdx.x, g = blockIdx.y;
  if (g >= *s.n_groups) return;
  const int e0 = s.group_off[g], m = s.group_off[g + 1] - e0;
  const int kbt = kdim / BK;
  unsigned char* dst = img + ((int64_t)g * kbt + kb) * (BN * 128);
  for (int i = threadIdx.x; i < BN * 8; i += blockDim.x) {  // blockDim.x is a multiple of 8
    const int r = i >> 3, c = i & 7;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < m) v = *reinterpret_cast<const uint4*>(x + (int64_t)s.entry_tok[e0 + r] * ld + kb * BK + c * 8);
    if (F16) {
      const float mul = c < 4 ? 1.0f : 0.0625f, cc = c < 4 ? 1032.0f : 1152.0f;
      uint32_t w[4] = {v.x, v.y, v.z, v.w};
      float part = 0.0f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint16_t lo = f2h_bits(bf2f((uint16_t)(w[j] & 0xFFFFu)) * mul);
        const uint16_t hi = f2h_bits(bf2f((uint16_t)(w[j] >> 16)) * mul);
        part = fmaf(cc, h2f_bits(lo), part);
        part = fmaf(cc, h2f_bits(hi), part);
        w[j] = (uint32_t)lo | ((uint32_t)hi << 16);
      }
      v = make_uint4(w[0], w[1], w[2], w[3]);
      part += __shfl_xor_sync(0xffffffffu, part, 1);
      part += __shfl_xor_sync(0xffffffffu, part, 2);
      part += __shfl_xor_sync(0xffffffffu, part, 4);
      if (c == 0) csum[((int64_t)g * BN + r) * kbt + kb] = part;
    }
    *reinterpret_cast<uint4*>(dst + sw128_off(r, c * 8)) = v;
  }
}

// Stage-1 finalize: sum the K-split partials of the interleaved gate/up rows, act = bf16(silu(g)*u),
// written straight into the stage-2 B images (entry -> its group's row); F16: class-scaled fp16
// of the bf16 act plus csum, as in k_gather_b.
template <bool F16>
__global__ void k_finalize_act(const float* __restrict__ p1, int splits, int64_t split_stride, SchedPtrs s,
                               const int32_t* __restrict__ entry_group, int n_entries, int f, int BN,
                               unsigned char* __restrict__ img, float* __restrict__ csum, GMask gm) {
  __shared__ float wpart[8];
  const int e = blockIdx.y;
  if (e >= s.group_off[*s.n_groups]) return;
  const int g = entry_group[e], t = e - s.group_off[g];
  if (!gmask_has(gm, g)) return;  // block-uniform
  const int kbt = f / BK;
  for (int i0 = blockIdx.x * blockDim.x; i0 < f; i0 += gridDim.x * blockDim.x) {  // f % 256 == 0
    const int i = i0 + threadIdx.x;
    float gv = 0.0f, uv = 0.0f;
    for (int sp = 0; sp < splits; ++sp) {
      const float* row = p1 + sp * split_stride + (int64_t)e * 2 * f;
      gv = __fadd_rn(gv, row[2 * i]);
      uv = __fadd_rn(uv, row[2 * i + 1]);
    }
    uint16_t act = f2bf(__fmul_rn(silu_det(gv), uv));
    if (F16) {
      const bool c1 = (i % BK) < 32;
      act = f2h_bits(bf2f(act) * (c1 ? 1.0f : 0.0625f));
      float part = (c1 ? 1032.0f : 1152.0f) * h2f_bits(act);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if ((threadIdx.x & 31) == 0) wpart[threadIdx.x >> 5] = part;
      __syncthreads();
      if ((threadIdx.x & 63) == 0)
        csum[((int64_t)g * BN + t) * kbt + i / BK] = wpart[threadIdx.x >> 5] + wpart[(threadIdx.x >> 5) + 1];
      __syncthreads();
    }
    *reinterpret_cast<uint16_t*>(img + ((int64_t)g * kbt + i / BK) * (BN * 128) + sw128_off(t, i % BK)) = act;
  }
}

// row-major [rows][cols] bf16 -> tile-major SW128 images [rows/128][cols/64][16 KB]
__global__ void k_tile_bf16(const uint16_t* __restrict__ src, int rows, int cols, unsigned char* __restrict__ dst) {
  const int64_t chunks = (int64_t)rows * cols / 8;
  const int kbt = cols / BK;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (cols / 8);
    const int c8 = (int)(i - r * (cols / 8)) * 8;
    const int rt = (int)(r / BM), rr = (int)(r % BM), kb = c8 / BK, cc = c8 % BK;
    const uint4 v = *reinterpret_cast<const uint4*>(src + r * cols + c8);
    *reinterpret_cast<uint4*>(dst + ((int64_t)rt * kbt + kb) * TILE_A + sw128_off(rr, cc)) = v;
  }
}

// ============================================================================ K2 v6 (INT4)
// The draft's INT4 (RTN on the GPTQ sym g128 grid) expert GEMM on tcgen05 with the EXPANDED WEIGHTS IN TMEM.
// Per 128-column scale group the producer bulk-copies the two 4 KB packed tiles (weight ring)
// and the two token tiles (token ring); eight dequant warps expand each packed word with ONE
// LOP3 per two weights into exact fp16 pairs -- (1024 + q) for a k-block's columns 0..31, (1024 +
// 16 q) for columns 32..63 (the 0x6400 fp16 magic; the old bf16 path needed a shift + two LOPs +
// an HFMA2 per pair and was the kernel's bound, profiles/r01/k2_ablation_w13.txt) -- and
// tcgen05.st them straight into a TMEM A-slot (lane = weight row, column c = K elements 2c, 2c+1).
// The MMA warps run kind::f16 (fp16 A from TMEM, fp16 token tile B from smem: x for class-1
// columns, x/16 for class-16 columns, so one accumulator serves both), one accumulator per group;
// four epilogue warps remove the bias with the per-token k-block sums csum and apply the group's
// per-row scale in fp32 while the next groups run:
//   y[row] = sum_g s[row][g] * (D_g[row] - C_g),  D_g - C_g = sum_{k in g} (q[row][k] - 8) x[k]
// Every product in D is exact (11-bit fp16 A x 11-bit fp16 B in the fp32 accumulator); the
// accumulation carries the 1024 offset, ~1e-4 relative to the group sum (tolerance 2e-3).
// Tile-major INT4 layout: packed [rows/128][cols/64][128 rows x 8 words]; word W of a row holds
// the k-block's columns 4W @0, 4W+1 @16, 4W+2 @8, 4W+3 @24, 32+4W @4, 33+4W @20, 34+4W @12,
// 35+4W @28 (bit offsets).  Scales [rows/128][cols/128][128] bf16.
MSPQ_D void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// non-blocking probe of a phase
MSPQ_D bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// (w & mask) | 0x64006400 in ONE LOP3: fp16x2 (1024 + q) for mask 0x000F000F, (1024 + 16 q) for
// 0x00F000F0 -- exact; the 1024 / 16 / -8 terms are removed in the epilogue (csum)
MSPQ_D uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

MSPQ_D uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// 32 consecutive TMEM columns of this warp's 32 lanes <- 32 registers per thread
MSPQ_D void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// kind::f16, A from TMEM: D[128 x N] (+)= A_tmem[128 x 16] . B_smem[N x 16]^T
MSPQ_D void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(accum)
      : "memory");
}

// Per-role cycle stamps of the first CTA of the first K2 launch after mspq_debug_timeline(_, -1)
// armed it (diagnostics).
__device__ long long g_int4_tl[2048];
__device__ int g_int4_tl_arm;
__device__ int g_k2_ablate;  // diagnostics: 1 = skip MMAs, 2 = skip TMEM stores, 4 = skip dequant math
MSPQ_D void tl_mark(bool on, int slot) {
  if (on && slot < 2048) g_int4_tl[slot] = clock64();
}

// pure polling wait (mbarrier.test_wait never suspends the thread)
MSPQ_D void mbar_spin(uint64_t* bar, uint32_t parity) {
  const long long t0 = clock64();
  while (!mbar_test(bar, parity))
    if (clock64() - t0 > 4000000000LL) __trap();
}
#ifndef K2_WAIT
#define K2_WAIT mbar_wait
#endif
// warps: 0 producer, 1..NI MMA issuers (warp 1 also allocates TMEM; issuer i takes the groups
// gi = i mod NI: an N=16 MMA costs its issuing THREAD ~56 cycles, but two issuers on one SM
// overlap (tools/micro/mma_rate.cu), so the per-group issue cost is split), then 8 dequant warps
// (lane quarter warp & 3, k-block half of the group), then 4 epilogue warps.
// A bulk copy costs its issuing thread ~0.3 us however small it is (tools/micro/bulk_rate.cu:
// 14 / 29 / 48 GB/s per thread at 4 / 8 / 16 KB), so every copy moves TWO 128-column groups:
// PW weight stages of 16 KB (4 packed tiles) recycle when the dequant warps have read them, PT
// token stages (4 token tiles) when the stage's last MMA completes.  With BROWS = 8 (<= 8
// tokens, N = 16) a token tile holds 8 rows (1 KB) and the descriptor's 8-row-group stride is 0:
// the MMA's rows 8..15 alias rows 0..7, whose results the epilogue never stores.  NA TMEM
// A-slots (64 columns = one group each), NACC TMEM accumulators.
template <int BN, int BROWS, int PW, int PT, int NA, int NACC, int NI, int GS>
__global__ void __launch_bounds__(32 * (14 + NI), 2) k_umma_int4(UmmaArgs a) {
  constexpr int W_DQ = 1 + NI, W_EP = W_DQ + 8, W_TK = W_EP + 4;  // first dequant / epilogue warp, token warp
  constexpr int TILE_Q = BM * BK / 2;             // 4 KB packed per 128x64 tile
  constexpr int TB = BROWS * 128;                 // token tile bytes per k-block
  constexpr int WST = GS * 2 * TILE_Q, TST = GS * 2 * TB;
  constexpr uint32_t ACOL = NI * NACC * BN;       // first A-slot column (issuer i: acc cols i*NACC*BN..)
  constexpr uint32_t TCOLS = (ACOL + NA * 64) <= 128 ? 128 : ((ACOL + NA * 64) <= 256 ? 256 : 512);
  const int S = a.splits, RT = a.rows / BM;
  const int unit = blockIdx.x;
  const int s = unit % S, rt = (unit / S) % RT, g = unit / (S * RT);
  if (g >= *a.n_groups) return;
  const int kb_total = a.kdim / BK;
  int per = (kb_total + S - 1) / S;
  per = (per + 1) & ~1;  // splits align to 128-column scale groups
  const int kb0 = s * per, nk = max(0, min(kb_total, kb0 + per) - kb0);
  const int e0 = a.group_off[g], m = a.group_off[g + 1] - e0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* outp = a.out + (int64_t)s * a.out_split_stride;
  if (nk == 0) {
    for (int i = threadIdx.x; i < m * BM; i += blockDim.x)
      outp[(int64_t)(e0 + i / BM) * a.rows + rt * BM + (i % BM)] = 0.0f;
    return;
  }
  const bool tl = blockIdx.x == 0 && g_int4_tl_arm != 0;
  const int abl = g_k2_ablate;
  const bool tla = g_int4_tl_arm != 0 && blockIdx.x < 256;  // per-CTA start/end (globaltimer ns)
  if (tla && threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_int4_tl[1536 + 2 * blockIdx.x] = t;
  }
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sT = base;             // PT x TST (SW128 token tiles: 1024-aligned)
  unsigned char* sW = sT + PT * TST;    // PW x WST
  // ONE tcgen05.commit per group (a commit costs ~190 cycles of the issuing thread, 4x an
  // N=16 MMA): done[gi % ND] frees the token stage (producer), the A-slot (dequant) and
  // publishes the accumulator (epilogue).  ND >= GS*PT, NA, NI*NACC keeps every waiter in one
  // phase.
  constexpr int ND0 = GS * PT > NA ? GS * PT : NA;
  constexpr int ND = ND0 > NI * NACC ? ND0 : NI * NACC;
  uint64_t* full_w = reinterpret_cast<uint64_t*>(sW + PW * WST);
  uint64_t* empty_w = full_w + PW;
  uint64_t* full_t = empty_w + PW;
  uint64_t* full_a = full_t + PT;
  uint64_t* done = full_a + NA;   // [ND]
  uint64_t* acce = done + ND;     // [NI][NACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + NI * NACC);

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < PW; ++i) {
      mbar_init(&full_w[i], 1);
      mbar_init(&empty_w[i], 8);  // one arrival per dequant warp (256 thread arrivals cost ~1k cycles)
    }
    for (int i = 0; i < PT; ++i) mbar_init(&full_t[i], 1);
    for (int i = 0; i < NA; ++i) mbar_init(&full_a[i], 8);
    for (int i = 0; i < ND; ++i) mbar_init(&done[i], 1);
    for (int i = 0; i < NI * NACC; ++i) mbar_init(&acce[i], 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int ngr = nk / 2;
  const int nst = (ngr + GS - 1) / GS;
  constexpr int NJ = BROWS < BN ? BROWS : BN;  // distinct token columns (8-row mode: 0..7)
  float epi_acc[NJ];  // epilogue warps: per-token row results
#pragma unroll
  for (int j = 0; j < NJ; ++j) epi_acc[j] = 0.0f;
#define epi_acc0 epi_acc[0]

  // self-gather (a.xsrc, one token per group): warp 0 builds the fp16 class-scaled token tiles
  // from the bf16 row itself (no gather kernel, no image in HBM) and keeps each group's
  // correction sum in smem (csm); otherwise token tiles are bulk-copied from a.bimg
  const bool selfg = a.xsrc != nullptr;
  __shared__ float csm[256];
  __shared__ float ksm[2 * GS];
  if (warp == 0) {  // weight producer: one bulk copy per stage, nothing else on this warp
    if (lane == 0) {
      const unsigned char* wsrc = a.w_base + ((int64_t)a.expert_base + a.group_buf[g]) * a.blob_bytes + a.w_off +
                                  ((int64_t)rt * kb_total + kb0) * TILE_Q;
      tl_mark(tl, 0);
      for (int jw = 0; jw < nst; ++jw) {
        if (jw >= PW) K2_WAIT(&empty_w[jw % PW], ((jw / PW) - 1) & 1);
        tl_mark(tl, 1 + jw);
        const int cnt = min(GS, ngr - jw * GS);
        mbar_expect_tx(&full_w[jw % PW], cnt * 2 * TILE_Q);
        bulk_g2s(sW + (jw % PW) * WST, wsrc + (int64_t)jw * WST, cnt * 2 * TILE_Q, &full_w[jw % PW]);
      }
    }
  } else if (warp == W_TK) {  // token producer: bulk copies of the B images, or self-gather
    const unsigned char* bsrc = selfg ? nullptr : a.bimg + ((int64_t)g * kb_total + kb0) * TB;
    const uint16_t* xr = selfg ? a.xsrc + (int64_t)(a.xsrc_by_entry ? e0 : a.entry_tok[e0]) * a.kdim + kb0 * BK
                               : nullptr;
    constexpr int XP = (GS * 2 * 8 + 31) / 32;  // 16-byte x chunks per lane per token stage
    uint4 xq[XP];
    auto load_x = [&](int js) {  // x chunks of token stage js into registers
#pragma unroll
      for (int p2 = 0; p2 < XP; ++p2) {
        const int task = p2 * 32 + lane, kbl = task >> 3, c = task & 7;
        xq[p2] = make_uint4(0, 0, 0, 0);
        if (selfg && js < nst && kbl < 2 * min(GS, ngr - js * GS))
          xq[p2] = *reinterpret_cast<const uint4*>(xr + (int64_t)(js * GS * 2 + kbl) * BK + c * 8);
      }
    };
    if (selfg) load_x(0);
    for (int jt = 0; jt < nst; ++jt) {
      if (jt >= PT) {  // every group of stage jt - PT (the MMA issuers complete out of order)
        const int gl = min(GS * (jt - PT) + GS - 1, ngr - 1);
        for (int gw = GS * (jt - PT); gw <= gl; ++gw) K2_WAIT(&done[gw % ND], (gw / ND) & 1);
      }
      const int cnt = min(GS, ngr - jt * GS);
      unsigned char* tdst = sT + (jt % PT) * TST;
      if (selfg) {
        // task = (k-block kbl of the stage, chunk c of 8 columns); row 0 only (rows 1..7 of the
        // 8-row tile are never stored by the epilogue); x loaded one stage ahead
#pragma unroll
        for (int p2 = 0; p2 < XP; ++p2) {
          const int task = p2 * 32 + lane, kbl = task >> 3, c = task & 7;
          float part = 0.0f;
          if (kbl < 2 * cnt) {
            const float mul = c < 4 ? 1.0f : 0.0625f, cc = c < 4 ? 1032.0f : 1152.0f;
            uint32_t w[4] = {xq[p2].x, xq[p2].y, xq[p2].z, xq[p2].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint16_t lo = f2h_bits(bf2f((uint16_t)(w[j] & 0xFFFFu)) * mul);
              const uint16_t hi = f2h_bits(bf2f((uint16_t)(w[j] >> 16)) * mul);
              part = fmaf(cc, h2f_bits(lo), part);
              part = fmaf(cc, h2f_bits(hi), part);
              w[j] = (uint32_t)lo | ((uint32_t)hi << 16);
            }
            *reinterpret_cast<uint4*>(tdst + kbl * TB + sw128_off(0, c * 8)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
          part += __shfl_xor_sync(0xffffffffu, part, 1);
          part += __shfl_xor_sync(0xffffffffu, part, 2);
          part += __shfl_xor_sync(0xffffffffu, part, 4);
          if (c == 0 && kbl < 2 * GS) ksm[kbl] = part;
        }
        __syncwarp();
        if (lane < cnt) csm[jt * GS + lane] = ksm[2 * lane] + ksm[2 * lane + 1];
        fence_proxy_async_smem();  // generic-proxy tile writes -> the MMA's async-proxy reads
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_t[jt % PT]);
        load_x(jt + 1);
      } else if (lane == 0) {
        mbar_expect_tx(&full_t[jt % PT], cnt * 2 * TB);
        bulk_g2s(tdst, bsrc + (int64_t)jt * TST, cnt * 2 * TB, &full_t[jt % PT]);
      }
    }
  } else if (warp < W_DQ) {
    if (lane == 0) {  // MMA issuer warp - 1: A from the TMEM slot, B from the token stage
      const int is = warp - 1;
      constexpr uint32_t idesc = idesc_f16(BN);
      // SW128 K-major B descriptor; 8-row-group stride 0 in BROWS = 8 mode (rows 8..15 alias 0..7)
      constexpr uint64_t sbo_fix = BROWS == 8 ? ~((uint64_t)0x3FFF << 32) : ~(uint64_t)0;
      for (int gi = is, u = 0; gi < ngr; gi += NI, ++u) {
        const int js = gi / GS, st = js % PT, sl = gi % NA, b = u % NACC;
        if (u >= NACC) K2_WAIT(&acce[is * NACC + b], ((u / NACC) - 1) & 1);
        K2_WAIT(&full_t[st], (js / PT) & 1);
        K2_WAIT(&full_a[sl], (gi / NA) & 1);
        tl_mark(tl, 768 + gi);
        tc_fence_after();
        const uint32_t sb = su32(sT + st * TST + (gi % GS) * 2 * TB);
        if (!(abl & 1))
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_ts(tmem + (is * NACC + b) * BN, tmem + ACOL + sl * 64 + kk * 8,
                  (sw128_desc(sb + (kk >> 2) * TB) & sbo_fix) + 2 * (kk & 3), idesc, kk != 0);
        umma_commit(&done[gi % ND]);
      }
    }
  } else if (warp < W_EP) {  // dequant warps: row q*32 + lane, k-block half h of each group
    const int q = warp & 3, h = (warp - W_DQ) >> 2;

    const int r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    for (int gi = 0; gi < ngr; ++gi) {
      const int js = gi / GS, st = js % PW, sl = gi % NA;
      K2_WAIT(&full_w[st], (js / PW) & 1);
      if (threadIdx.x == 32 * W_DQ) tl_mark(tl, 256 + gi);
      const uint32_t src = su32(sW + st * WST + ((gi % GS) * 2 + h) * TILE_Q + r * 32);
      const uint4 w0 = lds128(src), w1 = lds128(src + 16);
      const uint32_t ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
      // word w -> TMEM columns 2w, 2w+1 (class 1: local K 4w..4w+3) and 16+2w, 17+2w (class 16)
      uint32_t v[32];
      if (abl & 4) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = ws[i & 7];
      } else {
        const uint32_t m_lo = 0x000F000Fu, m_hi = 0x00F000F0u, magic = 0x64006400u;
#pragma unroll
        for (int wi = 0; wi < 8; ++wi) {
          const uint32_t w8 = ws[wi] >> 8;
          v[2 * wi] = lop3_and_or(ws[wi], m_lo, magic);
          v[2 * wi + 1] = lop3_and_or(w8, m_lo, magic);
          v[16 + 2 * wi] = lop3_and_or(ws[wi], m_hi, magic);
          v[17 + 2 * wi] = lop3_and_or(w8, m_hi, magic);
        }
      }
      __syncwarp();
      if (lane == 0 && (gi % GS == GS - 1 || gi == ngr - 1)) mbar_arrive(&empty_w[st]);  // stage consumed
      if (gi >= NA) K2_WAIT(&done[(gi - NA) % ND], ((gi - NA) / ND) & 1);
      tc_fence_after();
      if (!(abl & 2)) tmem_st32(tmem + lane_base + ACOL + sl * 64 + h * 32, v);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_a[sl]);
      if (threadIdx.x == 32 * W_DQ) tl_mark(tl, 512 + gi);
    }
  } else if (warp < W_TK) {  // epilogue warps 10..13: per-group scale, fp32 accumulation in registers
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint16_t* sc = reinterpret_cast<const uint16_t*>(a.w_base + ((int64_t)a.expert_base + a.group_buf[g]) * a.blob_bytes +
                                                           a.s_off) +
                         ((int64_t)rt * (a.kdim / 128) + kb0 / 2) * BM + row;
    float* acc = epi_acc;
    // per-token corrections of each k-block (k_gather_b / k_finalize_act, F16)
    const float* cs = a.csum + (int64_t)g * BROWS * kb_total + kb0;
    // the per-row scales and token 0's corrections of the next SW groups are fetched one batch
    // ahead, so the drain of a group never waits on a global-memory round trip (that latency,
    // paid per group, throttled the MMA issuers through acce).  Self-gather: the corrections
    // live in csm and are applied after the final __syncthreads (sum_g s_g * C_g).
    constexpr int SW = 4;
    float scw[SW], csw[SW], scn[SW], csn[SW];
    auto fetch = [&](int g0, float* sv, float* cv) {
#pragma unroll
      for (int u = 0; u < SW; ++u) {
        const bool ok = g0 + u < ngr;
        sv[u] = ok ? bf2f(sc[(int64_t)(g0 + u) * BM]) : 0.0f;
        cv[u] = ok && !selfg ? cs[2 * (g0 + u)] + cs[2 * (g0 + u) + 1] : 0.0f;
      }
    };
    fetch(0, scn, csn);
    for (int gi = 0; gi < ngr; ++gi) {
      if (gi % SW == 0) {
#pragma unroll
        for (int u = 0; u < SW; ++u) {
          scw[u] = scn[u];
          csw[u] = csn[u];
        }
        if (gi + SW < ngr) fetch(gi + SW, scn, csn);
      }
      const int ab = (gi % NI) * NACC + (gi / NI) % NACC;  // issuer gi % NI, its buffer
      float scale = scw[0], c0 = csw[0];
#pragma unroll
      for (int u = 1; u < SW; ++u)
        if (gi % SW == u) {
          scale = scw[u];
          c0 = csw[u];
        }
      K2_WAIT(&done[gi % ND], (gi / ND) & 1);
      if (threadIdx.x == 32 * W_EP) tl_mark(tl, 1280 + gi);
      tc_fence_after();
      float v[NJ];
      if constexpr (NJ == 8) {
        tmem_ld8(tmem + ((uint32_t)(q * 32) << 16) + ab * BN, v);
      } else {
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + ab * BN, v);
        if constexpr (NJ == 32) tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + ab * BN + 16, v + 16);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[ab]);
      acc[0] = fmaf(scale, v[0] - c0, acc[0]);
#pragma unroll
      for (int j = 1; j < NJ; ++j)
        if (j < m) {
          const float c = cs[(int64_t)j * kb_total + 2 * gi] + cs[(int64_t)j * kb_total + 2 * gi + 1];
          acc[j] = fmaf(scale, v[j] - c, acc[j]);
        }
    }
    if (tla && threadIdx.x == 32 * W_EP) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_int4_tl[1537 + 2 * blockIdx.x] = t;
    }
    if (tl && threadIdx.x == 32 * W_EP) g_int4_tl_arm = 0;  // record one launch only
  }
  tc_fence_before();
  __syncthreads();
  if (warp >= W_EP && warp < W_TK) {  // output: self-gather corrections, then y planes or fused SiLU*up
    const int q = warp & 3;
    const int row = q * 32 + lane;
    if (selfg) {
      const uint16_t* sc = reinterpret_cast<const uint16_t*>(a.w_base + ((int64_t)a.expert_base + a.group_buf[g]) * a.blob_bytes +
                                                             a.s_off) +
                           ((int64_t)rt * (a.kdim / 128) + kb0 / 2) * BM + row;
      float corr = 0.0f;
      for (int gi = 0; gi < ngr; ++gi) corr = fmaf(bf2f(sc[(int64_t)gi * BM]), csm[gi], corr);
      epi_acc0 -= corr;
    }
    if (a.act_out) {
      // interleaved W13 rows: row 2i = gate_i, 2i+1 = up_i; act = bf16(silu(gate) * up), exactly
      // k_finalize_act's arithmetic on a single split
      const float up = __shfl_down_sync(0xffffffffu, epi_acc0, 1);
      if ((lane & 1) == 0 && m > 0)
        a.act_out[(int64_t)e0 * (a.rows / 2) + (rt * BM + row) / 2] = f2bf(__fmul_rn(silu_det(epi_acc0), up));
    } else {
      if (m > 0) outp[(int64_t)e0 * a.rows + rt * BM + row] = epi_acc0;
#pragma unroll
      for (int j = 1; j < NJ; ++j)
        if (j < m) outp[(int64_t)(e0 + j) * a.rows + rt * BM + row] = epi_acc[j];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
#undef epi_acc0
}

// ------------------------------------------------------------------ K2 persistent (draft, T = 1)
// One CTA per SM (all 512 TMEM columns: 7 A-slots + 2 issuers x 2 accumulators) walks units
// u = blockIdx.x, + gridDim.x, ... of (group g, 128-row tile rt, K split s).  The per-CTA rate was
// bounded by the A-slot round trip (dequant -> MMA -> commit -> done -> dequant), ~1 us for 3
// slots; 7 slots in flight and one CTA per SM keep the weight stream going.  Every role walks the
// same unit list; a global group counter gi drives all rings and barrier phases, so a unit's
// pipeline runs straight into the next unit's.  Self-gather only (token rows from a.xsrc): the
// token warp builds the 8-row fp16 tiles, the epilogue computes the unit's bias corrections from
// x at the unit's end (4 epilogue warps, named barrier 1) and writes y / the fused SiLU*up.
template <int PW, int PT, int NA, int NACC, int NI, int GS>
__global__ void __launch_bounds__(32 * (22 + NI), 1) k_umma_int4p(UmmaArgs a, int n_units) {
  constexpr int BN = 16, BROWS = 8;
  // two sets of 8 dequant warps take alternate groups, so one set's TMEM-store round trip
  // overlaps the other's expansion
  constexpr int W_DQ = 1 + NI, W_EP = W_DQ + 16, W_TK = W_EP + 4;
  constexpr int TILE_Q = BM * BK / 2, TB = BROWS * 128;
  constexpr int WST = GS * 2 * TILE_Q, TST = GS * 2 * TB;
  constexpr uint32_t ACOL = NI * NACC * BN, TCOLS = 512;
  static_assert(ACOL + NA * 64 <= 512, "TMEM budget");
  constexpr int ND0 = GS * PT > NA ? GS * PT : NA;
  constexpr int ND = ND0 > NI * NACC ? ND0 : NI * NACC;
  const int S = a.splits, RT = a.rows / BM, kb_total = a.kdim / BK;
  const int ng_live = *a.n_groups;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int abl = g_k2_ablate;
  const bool tl = blockIdx.x == 0 && g_int4_tl_arm != 0;
  const bool tla = g_int4_tl_arm != 0 && blockIdx.x < 256;
  if (tla && threadIdx.x == 0) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_int4_tl[1536 + 2 * blockIdx.x] = t;
  }
  // unit u -> (g, rt, s, kb0, ngr); identical in every role
  struct Unit { int g, rt, s, kb0, ngr, e0, m; };
  auto unit = [&](int u) {
    Unit x;
    x.s = u % S;
    x.rt = (u / S) % RT;
    x.g = u / (S * RT);
    int per = (kb_total + S - 1) / S;
    per = (per + 1) & ~1;
    x.kb0 = x.s * per;
    const int nk = max(0, min(kb_total, x.kb0 + per) - x.kb0);
    x.ngr = x.g < ng_live ? nk / 2 : 0;
    x.e0 = x.g < ng_live ? a.group_off[x.g] : 0;
    x.m = x.g < ng_live ? a.group_off[x.g + 1] - x.e0 : 0;
    return x;
  };
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sT = base;           // PT x TST
  unsigned char* sW = sT + PT * TST;  // PW x WST
  uint64_t* full_w = reinterpret_cast<uint64_t*>(sW + PW * WST);
  uint64_t* empty_w = full_w + PW;
  uint64_t* full_t = empty_w + PW;
  uint64_t* full_a = full_t + PT;
  uint64_t* done = full_a + NA;
  uint64_t* acce = done + ND;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + NI * NACC);
  __shared__ float csu[256];        // epilogue: per-group corrections of the current unit
  __shared__ int stage_last[PT];    // token warp: global index of each token stage's last group
  __shared__ int stage_first[PT];   //              ... and first group
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < PW; ++i) {
      mbar_init(&full_w[i], 1);
      mbar_init(&empty_w[i], 8 * GS);  // 8 dequant warps per group of the stage
    }
    for (int i = 0; i < PT; ++i) mbar_init(&full_t[i], 1);
    for (int i = 0; i < NA; ++i) mbar_init(&full_a[i], 8);
    for (int i = 0; i < ND; ++i) mbar_init(&done[i], 1);
    for (int i = 0; i < NI * NACC; ++i) mbar_init(&acce[i], 4);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {  // weight producer: one bulk copy per stage of GS groups (within a unit)
    if (lane == 0) {
      int jw = 0;  // global stage counter
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit x = unit(u);
        if (x.ngr == 0) continue;
        const unsigned char* wsrc = a.w_base + ((int64_t)a.expert_base + a.group_buf[x.g]) * a.blob_bytes + a.w_off +
                                    ((int64_t)x.rt * kb_total + x.kb0) * TILE_Q;
        const int nst = (x.ngr + GS - 1) / GS;
        for (int j = 0; j < nst; ++j, ++jw) {
          if (jw >= PW) K2_WAIT(&empty_w[jw % PW], ((jw / PW) - 1) & 1);
          tl_mark(tl, 1 + jw);
          const int cnt = min(GS, x.ngr - j * GS);
          mbar_expect_tx(&full_w[jw % PW], cnt * 2 * TILE_Q);
          bulk_g2s(sW + (jw % PW) * WST, wsrc + (int64_t)j * WST, cnt * 2 * TILE_Q, &full_w[jw % PW]);
        }
      }
    }
  } else if (warp == W_TK) {  // token producer: 8-row fp16 class-scaled tiles from the bf16 row
    int jt = 0, gdone = 0;  // global token stage / global group index at the stage start
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const Unit x = unit(u);
      if (x.ngr == 0) continue;
      const uint16_t* xr = a.xsrc + (int64_t)(a.xsrc_by_entry ? x.e0 : a.entry_tok[x.e0]) * a.kdim + x.kb0 * BK;
      const int nst = (x.ngr + GS - 1) / GS;
      for (int j = 0; j < nst; ++j, ++jt) {
        const int cnt = min(GS, x.ngr - j * GS);
        if (jt >= PT) {  // the slot was last read by every group of global stage jt - PT; with
                         // several MMA issuers their completions are not ordered, so wait on each
          const int glast = stage_last[(jt - PT) % PT], gfirst = stage_first[(jt - PT) % PT];
          for (int gw = gfirst; gw <= glast; ++gw) K2_WAIT(&done[gw % ND], (gw / ND) & 1);
        }
        unsigned char* tdst = sT + (jt % PT) * TST;
#pragma unroll
        for (int p2 = 0; p2 < (GS * 16 + 31) / 32; ++p2) {
          const int task = p2 * 32 + lane, kbl = task >> 3, c = task & 7;
          if (kbl < 2 * cnt) {
            const uint4 v = *reinterpret_cast<const uint4*>(xr + (int64_t)(j * GS * 2 + kbl) * BK + c * 8);
            const float mul = c < 4 ? 1.0f : 0.0625f;
            uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint16_t lo = f2h_bits(bf2f((uint16_t)(w[q] & 0xFFFFu)) * mul);
              const uint16_t hi = f2h_bits(bf2f((uint16_t)(w[q] >> 16)) * mul);
              w[q] = (uint32_t)lo | ((uint32_t)hi << 16);
            }
            *reinterpret_cast<uint4*>(tdst + kbl * TB + sw128_off(0, c * 8)) = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          stage_first[jt % PT] = gdone;
          stage_last[jt % PT] = gdone + cnt - 1;
          mbar_arrive(&full_t[jt % PT]);
        }
        gdone += cnt;
      }
    }
  } else if (warp < W_DQ) {  // MMA issuers
    if (lane == 0) {
      const int is = warp - 1;
      constexpr uint32_t idesc = idesc_f16(BN);
      constexpr uint64_t sbo_fix = ~((uint64_t)0x3FFF << 32);  // 8-row tiles: rows 8..15 alias 0..7
      int gi = 0, js = 0;  // global group, global token stage
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const Unit x = unit(u);
        for (int gl = 0; gl < x.ngr; ++gl, ++gi) {
          const int jsg = js + gl / GS;
          if (gi % NI == is) {
            const int uu = gi / NI, sl = gi % NA, b = uu % NACC;
            if (uu >= NACC) K2_WAIT(&acce[is * NACC + b], ((uu / NACC) - 1) & 1);
            K2_WAIT(&full_t[jsg % PT], (jsg / PT) & 1);
            K2_WAIT(&full_a[sl], (gi / NA) & 1);
            tl_mark(tl, 768 + gi);
            tc_fence_after();
            const uint32_t sb = su32(sT + (jsg % PT) * TST + (gl % GS) * 2 * TB);
            if (!(abl & 1))
#pragma unroll
              for (int kk = 0; kk < 8; ++kk)
                umma_ts(tmem + (is * NACC + b) * BN, tmem + ACOL + sl * 64 + kk * 8,
                        (sw128_desc(sb + (kk >> 2) * TB) & sbo_fix) + 2 * (kk & 3), idesc, kk != 0);
            umma_commit(&done[gi % ND]);
          }
        }
        js += (x.ngr + GS - 1) / GS;
      }
    }
  } else if (warp < W_EP) {  // dequant warps: set ds takes groups gi % 2 == ds; row q*32 + lane, half h
    const int ds = (warp - W_DQ) >> 3;
    const int q = warp & 3, h = ((warp - W_DQ) >> 2) & 1;
    const int r = q * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    int gi = 0, jw = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const Unit x = unit(u);
      for (int gl = 0; gl < x.ngr; ++gl, ++gi) {
        if ((gi & 1) != ds) continue;
        const int jsw = jw + gl / GS, st = jsw % PW, sl = gi % NA;
        K2_WAIT(&full_w[st], (jsw / PW) & 1);
        if (threadIdx.x == 32 * W_DQ || threadIdx.x == 32 * (W_DQ + 8)) tl_mark(tl, 256 + gi);
        const uint32_t src = su32(sW + st * WST + ((gl % GS) * 2 + h) * TILE_Q + r * 32);
        const uint4 w0 = lds128(src), w1 = lds128(src + 16);
        const uint32_t ws[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        uint32_t v[32];
        const uint32_t m_lo = 0x000F000Fu, m_hi = 0x00F000F0u, magic = 0x64006400u;
#pragma unroll
        for (int wi = 0; wi < 8; ++wi) {
          const uint32_t w8 = ws[wi] >> 8;
          v[2 * wi] = lop3_and_or(ws[wi], m_lo, magic);
          v[2 * wi + 1] = lop3_and_or(w8, m_lo, magic);
          v[16 + 2 * wi] = lop3_and_or(ws[wi], m_hi, magic);
          v[17 + 2 * wi] = lop3_and_or(w8, m_hi, magic);
        }
        __syncwarp();
        if (lane == 0) {  // one arrival per group; the unit's last (short) stage makes up the rest
          const int cnt = min(GS, x.ngr - (gl / GS) * GS);
          const uint32_t mult = gl == x.ngr - 1 ? (uint32_t)(GS - cnt + 1) : 1u;
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&empty_w[st])), "r"(mult)
                       : "memory");
        }
        if (gi >= NA) K2_WAIT(&done[(gi - NA) % ND], ((gi - NA) / ND) & 1);
        tc_fence_after();
        if (!(abl & 2)) tmem_st32(tmem + lane_base + ACOL + sl * 64 + h * 32, v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_a[sl]);
        if (threadIdx.x == 32 * W_DQ || threadIdx.x == 32 * (W_DQ + 8)) tl_mark(tl, 512 + gi);
      }
      jw += (x.ngr + GS - 1) / GS;
    }
  } else if (warp < W_TK) {  // epilogue: per-group scale, per-unit corrections and output
    const int q = warp & 3, row = q * 32 + lane, et = threadIdx.x - 32 * W_EP;  // et: 0..127
    int gi = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const Unit x = unit(u);
      if (x.g >= ng_live) continue;
      const uint16_t* sc = reinterpret_cast<const uint16_t*>(a.w_base + ((int64_t)a.expert_base + a.group_buf[x.g]) *
                                                                            a.blob_bytes + a.s_off) +
                           ((int64_t)x.rt * (a.kdim / 128) + x.kb0 / 2) * BM + row;
      // the unit's corrections C_g = sum_k c_k b_k (fp16 b as the token warp builds it), one group
      // per thread, fixed order; they only need x, so they are ready before the first drain
      const uint16_t* xr = a.xsrc + (int64_t)(a.xsrc_by_entry ? x.e0 : a.entry_tok[x.e0]) * a.kdim + x.kb0 * BK;
      {  // thread et: chunk c16 = et % 16 (8 columns) of groups et / 16, + 8, ...; the 16 chunks of a
         // group are reduced over 16 consecutive lanes in a fixed xor order
        const int c16 = et & 15, c = c16 & 7;
        const float mul = c < 4 ? 1.0f : 0.0625f, cc = c < 4 ? 1032.0f : 1152.0f;
        for (int g0 = 0; g0 < x.ngr; g0 += 8) {
          const int gg = g0 + (et >> 4);
          float part = 0.0f;
          if (gg < x.ngr) {
            const uint4 v = *reinterpret_cast<const uint4*>(xr + (int64_t)gg * 128 + c16 * 8);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
              part = fmaf(cc, h2f_bits(f2h_bits(bf2f((uint16_t)(w[q2] & 0xFFFFu)) * mul)), part);
              part = fmaf(cc, h2f_bits(f2h_bits(bf2f((uint16_t)(w[q2] >> 16)) * mul)), part);
            }
          }
#pragma unroll
          for (int o = 1; o < 16; o <<= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
          if (c16 == 0 && gg < x.ngr) csu[gg] = part;
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      float acc = 0.0f;
      // the row's scales, SW groups at a time, loaded one batch ahead (a scale load per group on
      // the drain path held the MMA issuers back through acce)
      constexpr int SW = 8;
      float scw[SW], scn[SW];
#pragma unroll
      for (int u2 = 0; u2 < SW; ++u2) scn[u2] = u2 < x.ngr ? bf2f(sc[(int64_t)u2 * BM]) : 0.0f;
      for (int gl = 0; gl < x.ngr; ++gl, ++gi) {
        const int ab = (gi % NI) * NACC + (gi / NI) % NACC;
        if (gl % SW == 0) {
#pragma unroll
          for (int u2 = 0; u2 < SW; ++u2) {
            scw[u2] = scn[u2];
            scn[u2] = gl + SW + u2 < x.ngr ? bf2f(sc[(int64_t)(gl + SW + u2) * BM]) : 0.0f;
          }
        }
        float scale = scw[0];
#pragma unroll
        for (int u2 = 1; u2 < SW; ++u2)
          if (gl % SW == u2) scale = scw[u2];
        K2_WAIT(&done[gi % ND], (gi / ND) & 1);
        if (threadIdx.x == 32 * W_EP) tl_mark(tl, 1280 + gi);
        tc_fence_after();
        float v[8];
        tmem_ld8(tmem + ((uint32_t)(q * 32) << 16) + ab * BN, v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acce[ab]);
        acc = fmaf(scale, v[0] - csu[gl], acc);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // csu is rewritten by the next unit
      if (x.m > 0) {
        if (a.act_out) {
          const float up = __shfl_down_sync(0xffffffffu, acc, 1);
          if ((lane & 1) == 0)
            a.act_out[(int64_t)x.e0 * (a.rows / 2) + (x.rt * BM + row) / 2] = f2bf(__fmul_rn(silu_det(acc), up));
        } else {
          a.out[(int64_t)x.s * a.out_split_stride + (int64_t)x.e0 * a.rows + x.rt * BM + row] = acc;
        }
      }
    }
    if (tla && threadIdx.x == 32 * W_EP) {
      long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      g_int4_tl[1537 + 2 * blockIdx.x] = t;
    }
    if (tl && threadIdx.x == 32 * W_EP) g_int4_tl_arm = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
  }
}

// row-major quantised (standard nibble order, scales [rows][cols/128]) -> tile-major INT4 layout
__global__ void k_tile_int4(const uint32_t* __restrict__ q, const uint16_t* __restrict__ sc, int rows, int cols,
                            uint32_t* __restrict__ tq, uint16_t* __restrict__ ts) {
  const int wpr = cols / 8;  // words per row
  const int kbt = cols / BK, ngr = cols / 128;
  const int64_t nw = (int64_t)rows * wpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / wpr;
    const int w = (int)(i - r * wpr);
    // output word W = w % 8 of k-block kb = w / 8 holds the block's local columns
    //   4W @0, 4W+1 @16, 4W+2 @8, 4W+3 @24 (class 1) and 32+4W @4, 33+4W @20, 34+4W @12, 35+4W @28
    // (class 16): one LOP3 per two fp16 weights (K2 dequant), no shifts for the low byte pair
    const int kb = w / 8, W = w % 8;
    const uint32_t* src = q + r * wpr + kb * 8;
    auto nib = [&](int c) { return (src[c >> 3] >> (4 * (c & 7))) & 0xFu; };
    const uint32_t o = nib(4 * W) | (nib(4 * W + 1) << 16) | (nib(4 * W + 2) << 8) | (nib(4 * W + 3) << 24) |
                       (nib(32 + 4 * W) << 4) | (nib(33 + 4 * W) << 20) | (nib(34 + 4 * W) << 12) |
                       (nib(35 + 4 * W) << 28);
    const int rt = (int)(r / BM), rr = (int)(r % BM);
    tq[(((int64_t)rt * kbt + kb) * BM + rr) * 8 + W] = o;
  }
  const int64_t ns = (int64_t)rows * ngr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ngr;
    const int gg = (int)(i - r * ngr);
    ts[(((int64_t)(r / BM) * ngr) + gg) * BM + (r % BM)] = sc[i];
  }
}

}  // namespace


template <int BN, int STAGES>
static cudaError_t launch_grouped_v(const UmmaArgs& a, int units, cudaStream_t st) {
  const size_t smem = 1024 + STAGES * (TILE_A + BN * 128) + (2 * STAGES + 2) * 8 + 16;
  cudaFuncSetAttribute(k_umma_grouped<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_umma_grouped<BN, STAGES>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  return launch_pdl(k_umma_grouped<BN, STAGES>, dim3(units), dim3(192), smem, st, a);
}

// 3 stages (57 KB smem at BN = 16, 63 KB at BN = 32) fit 3 CTAs per SM with room left for an XC
// decode CTA (25 KB) on the same SM, so a verify layer's W13 (<= 4 experts x 100 row tiles at
// k = 1) stays one wave of 444 while the codec runs beside it (with 4 stages a resident decode CTA
// cut the SM to 2 GEMM CTAs: K3 0.66 of HBM in the cap-4 bench); 3 x 3 x 16 KB in flight per SM
// is still ~2x what the HBM latency needs.
cudaError_t launch_umma_grouped(const UmmaArgs& a, int max_groups, int BN, cudaStream_t st) {
  const int units = max_groups * (a.rows / BM) * a.splits;
  if (units == 0) return cudaSuccess;
  if (BN == 16) return launch_grouped_v<16, 3>(a, units, st);
  return launch_grouped_v<32, 3>(a, units, st);
}

cudaError_t launch_umma_int4(const UmmaArgs& a, int max_groups, int BN, cudaStream_t st) {
  // A bulk copy costs its issuing thread ~0.3 us, so the draft variant (8-row tiles) moves THREE
  // groups (24 KB) per weight copy: 3 x 24 KB in flight, 2 token stages, 3 TMEM A-slots, 2 MMA
  // issuers x 2 accumulators in 256 TMEM columns, ~86 KB smem -> 2 CTAs/SM.  The wider-token
  // variants (tests, T > 8) keep two groups per copy.
  constexpr int NA = 3, NI = 2, THREADS = 32 * (14 + NI);
  const int units = max_groups * (a.rows / BM) * a.splits;
  if (units == 0) return cudaSuccess;
  auto smem = [&](int brows, int pw, int pt, int gs) {
    return (size_t)1024 + pt * gs * 2 * brows * 128 + pw * gs * 2 * (BM * BK / 2) + 64 * 8 + 16;
  };
  if (BN == 16 && a.brows == 8) {
    auto k = k_umma_int4<16, 8, 3, 2, NA, 2, NI, 3>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(8, 3, 2, 3));
    k<<<units, THREADS, smem(8, 3, 2, 3), st>>>(a);
  } else if (BN == 16) {
    auto k = k_umma_int4<16, 16, 5, 2, NA, 2, NI, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(16, 5, 2, 2));
    k<<<units, THREADS, smem(16, 5, 2, 2), st>>>(a);
  } else {
    auto k = k_umma_int4<32, 32, 4, 2, NA, 1, NI, 2>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(32, 4, 2, 2));
    k<<<units, THREADS, smem(32, 4, 2, 2), st>>>(a);
  }
  return cudaGetLastError();
}

// Persistent draft-shape K2 (one token per group, 8-row tiles): one CTA per SM.
cudaError_t launch_umma_int4p(const UmmaArgs& a, int max_groups, cudaStream_t st) {
  constexpr int PW = 6, PT = 4, NA = 6, NACC = 2, NI = 4, GS = 3, THREADS = 32 * (22 + NI);
  const int units = max_groups * (a.rows / BM) * a.splits;
  if (units == 0) return cudaSuccess;
  static int sms = 0;
  if (!sms) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = 1024 + (size_t)PT * GS * 2 * 8 * 128 + (size_t)PW * GS * 2 * (BM * BK / 2) + 64 * 8 + 16;
  auto k = k_umma_int4p<PW, PT, NA, NACC, NI, GS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<std::min(units, std::max(sms, 1)), THREADS, smem, st>>>(a, units);
  return cudaGetLastError();
}

// n < 0 arms the recorder for the next K2 launch; n > 0 copies the stamps out
cudaError_t debug_int4_timeline(long long* dst, int n) {
  if (n <= -100) {  // -100 - mode: K2 ablation mode (diagnostics only; 0 = normal)
    const int mode = -100 - n;
    return cudaMemcpyToSymbol(g_k2_ablate, &mode, sizeof(int));
  }
  if (n < 0) {
    const int one = 1;
    return cudaMemcpyToSymbol(g_int4_tl_arm, &one, sizeof(int));
  }
  const int zero = 0;
  cudaError_t e = cudaMemcpyToSymbol(g_int4_tl_arm, &zero, sizeof(int));
  if (e != cudaSuccess) return e;
  return cudaMemcpyFromSymbol(dst, g_int4_tl, sizeof(long long) * std::min(n, 2048));
}

cudaError_t launch_tile_int4(const uint32_t* q, const uint16_t* s, int rows, int cols, uint32_t* tq, uint16_t* ts,
                             cudaStream_t st) {
  k_tile_int4<<<148 * 4, 256, 0, st>>>(q, s, rows, cols, tq, ts);
  return cudaGetLastError();
}

cudaError_t launch_gather_b(const uint16_t* x, int ld, SchedPtrs s, int max_groups, int kdim, int BN,
                            unsigned char* img, cudaStream_t st, float* csum) {
  if (csum)
    return launch_pdl(k_gather_b<true>, dim3(kdim / BK, max_groups), dim3(128), 0, st, x, ld, s, kdim, BN, img, csum);
  else
    return launch_pdl(k_gather_b<false>, dim3(kdim / BK, max_groups), dim3(128), 0, st, x, ld, s, kdim, BN, img,
                      (float*)nullptr);
  return cudaGetLastError();
}

cudaError_t launch_finalize_act(const float* p1, int splits, int64_t split_stride, SchedPtrs s,
                                const int32_t* entry_group, int n_entries, int f, int BN, unsigned char* img,
                                cudaStream_t st, float* csum, GMask gm) {
  if (csum)
    k_finalize_act<true><<<dim3(f / 256, n_entries), 256, 0, st>>>(p1, splits, split_stride, s, entry_group,
                                                                  n_entries, f, BN, img, csum, gm);
  else
    k_finalize_act<false><<<dim3(f / 256, n_entries), 256, 0, st>>>(p1, splits, split_stride, s, entry_group,
                                                                   n_entries, f, BN, img, nullptr, gm);
  return cudaGetLastError();
}

cudaError_t launch_tile_bf16(const uint16_t* src, int rows, int cols, unsigned char* dst, cudaStream_t st) {
  k_tile_bf16<<<148 * 8, 256, 0, st>>>(src, rows, cols, dst);
  return cudaGetLastError();
}

}  // namespace mspq
