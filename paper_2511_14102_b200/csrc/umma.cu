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
#include "common.cuh"
#include "kernels.h"

namespace mspq {
namespace {

constexpr int BM = 128, BK = 64, TILE_A = BM * BK * 2;

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
MSPQ_HD int sw128_off(int row, int col) {
  return (row >> 3) * 1024 + (row & 7) * 128 + ((((col >> 3) ^ (row & 7)) & 7) << 4) + (col & 7) * 2;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1) k_umma_grouped(UmmaArgs a) {
  const int S = a.splits, RT = a.rows / BM;
  const int unit = blockIdx.x;
  const int s = unit % S, rt = (unit / S) % RT, g = unit / (S * RT);
  if (g >= *a.n_groups) return;
  const int kb_total = a.kdim / BK;
  const int per = (kb_total + S - 1) / S;
  const int kb0 = s * per, nk = max(0, min(kb_total, kb0 + per) - kb0);
  const int e0 = a.group_off[g], m = a.group_off[g + 1] - e0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* outp = a.out + (int64_t)s * a.out_split_stride;
  if (nk == 0) {  // empty split: contribute zeros
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

  if (warp == 0) {
    if (lane == 0) {  // producer
      const unsigned char* wsrc = a.w_base + (int64_t)a.group_buf[g] * a.blob_bytes + a.w_off +
                                  ((int64_t)rt * kb_total + kb0) * TILE_A;
      const unsigned char* bsrc = a.bimg + ((int64_t)g * kb_total + kb0) * (BN * 128);
      for (int i = 0; i < nk; ++i) {
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
    for (int t = 0; t < m && t < BN; ++t) outp[(int64_t)(e0 + t) * a.rows + row] = v[t];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
  }
}

// Gather the tokens of every group into the SW128 B images [G][kdim/64][BN x 64] bf16.
__global__ void k_gather_b(const uint16_t* __restrict__ x, int ld, SchedPtrs s, int kdim, int BN,
                           unsigned char* __restrict__ img) {
  const int kb = blockIdx.x, g = blockIdx.y;
  if (g >= *s.n_groups) return;
  const int e0 = s.group_off[g], m = s.group_off[g + 1] - e0;
  const int kbt = kdim / BK;
  unsigned char* dst = img + ((int64_t)g * kbt + kb) * (BN * 128);
  for (int i = threadIdx.x; i < BN * 8; i += blockDim.x) {
    const int r = i >> 3, c = i & 7;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < m) v = *reinterpret_cast<const uint4*>(x + (int64_t)s.entry_tok[e0 + r] * ld + kb * BK + c * 8);
    *reinterpret_cast<uint4*>(dst + sw128_off(r, c * 8)) = v;
  }
}

// Stage-1 finalize: sum the K-split partials of the interleaved gate/up rows, act = bf16(silu(g)*u),
// written straight into the stage-2 B images (entry -> its group's row).
__global__ void k_finalize_act(const float* __restrict__ p1, int splits, int64_t split_stride, SchedPtrs s,
                               const int32_t* __restrict__ entry_group, int n_entries, int f, int BN,
                               unsigned char* __restrict__ img) {
  const int e = blockIdx.y;
  if (e >= s.group_off[*s.n_groups]) return;
  const int g = entry_group[e], t = e - s.group_off[g];
  const int kbt = f / BK;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < f; i += gridDim.x * blockDim.x) {
    float gv = 0.0f, uv = 0.0f;
    for (int sp = 0; sp < splits; ++sp) {
      const float* row = p1 + sp * split_stride + (int64_t)e * 2 * f;
      gv = __fadd_rn(gv, row[2 * i]);
      uv = __fadd_rn(uv, row[2 * i + 1]);
    }
    const uint16_t act = f2bf(__fmul_rn(silu_det(gv), uv));
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

// ============================================================================ K2 v2 (INT4)
// The draft's GPTQ-sym INT4 expert GEMM on tcgen05.  Per 128x64 tile the producer bulk-copies
// the 4 KB packed tile (+ the token tile); four dequant warps expand it to the exact bf16
// (q - 8) values of the SW128 image (one LOP3 + one HSUB2 per two weights via the 128.0 bf16
// magic), the MMA warp accumulates each 128-column scale group into one of two TMEM buffers, and
// four epilogue warps apply that group's per-row scale in fp32 while the next group runs:
//   y[row] = sum_g s[row][g] * sum_{k in g} (q[row][k] - 8) * x[k]      (exact GPTQ-sym dequant)
// Tile-major INT4 layout: packed [rows/128][cols/64][128 rows x 8 words]; word w of a row holds
// columns 8w..8w+7 with column 8w+2i at bits 4i and 8w+2i+1 at bits 16+4i.  Scales
// [rows/128][cols/128][128] bf16.
MSPQ_D void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
MSPQ_D void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

MSPQ_D uint4 dequant8(uint32_t w) {
  // (w >> 4i) & 0x000F000F | 0x43004300 = bf16x2(128 + q_lo, 128 + q_hi); minus 136 -> exact q - 8
  const __nv_bfloat162 off = __floats2bfloat162_rn(136.0f, 136.0f);
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t t = ((w >> (4 * i)) & 0x000F000Fu) | 0x43004300u;
    __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&t);
    v = __hsub2(v, off);
    o[i] = *reinterpret_cast<uint32_t*>(&v);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

MSPQ_D void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
MSPQ_D uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

// Per-role cycle stamps of the first CTA (diagnostics, read with mspq_debug_timeline).
__device__ long long g_int4_tl[2048];
MSPQ_D void tl_mark(int slot) {
  if (blockIdx.x == 0 && slot < 2048) g_int4_tl[slot] = clock64();
}

// warps: 0 producer, 1 MMA, 2..9 dequant (256 threads, two per tile row), 10..13 epilogue
template <int BN, int KBS, int PS, int DS, int NACC>
__global__ void __launch_bounds__(448, 2) k_umma_int4(UmmaArgs a) {
  constexpr int TILE_Q = BM * BK / 2;  // 4 KB packed per 128x64 tile
  constexpr int TB = BN * 128;         // token tile bytes per k-block
  constexpr int STAGE = KBS * (TILE_Q + TB);  // one bulk-copy stage = KBS consecutive k-blocks
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
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sD = base;                   // DS x (16 KB A + TB)    dequantised k-blocks
  unsigned char* sP = sD + DS * (TILE_A + TB);  // PS x STAGE             packed stages
  uint64_t* full_p = reinterpret_cast<uint64_t*>(sP + PS * STAGE);
  uint64_t* empty_p = full_p + PS;
  uint64_t* full_d = empty_p + PS;
  uint64_t* empty_d = full_d + DS;
  uint64_t* accf = empty_d + DS;  // [NACC]
  uint64_t* acce = accf + NACC;   // [NACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + NACC);
  constexpr uint32_t TCOLS = BN * NACC <= 32 ? 32 : (BN * NACC <= 64 ? 64 : (BN * NACC <= 128 ? 128 : 256));

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < PS; ++i) {
      mbar_init(&full_p[i], 1);
      mbar_init(&empty_p[i], 256);
    }
    for (int i = 0; i < DS; ++i) {
      mbar_init(&full_d[i], 256);
      mbar_init(&empty_d[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], 128);
    }
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
  const int nst = (nk + KBS - 1) / KBS;

  if (warp == 0) {
    if (lane == 0) {  // producer: KBS packed weight tiles + KBS token tiles per bulk stage
      const unsigned char* wsrc = a.w_base + ((int64_t)a.expert_base + a.group_buf[g]) * a.blob_bytes + a.w_off +
                                  ((int64_t)rt * kb_total + kb0) * TILE_Q;
      const unsigned char* bsrc = a.bimg + ((int64_t)g * kb_total + kb0) * TB;
      tl_mark(0);
      for (int j = 0; j < nst; ++j) {
        const int st = j % PS, r = j / PS;
        const int cnt = min(KBS, nk - j * KBS);
        if (r > 0) mbar_wait(&empty_p[st], (r - 1) & 1);
        tl_mark(1 + j);
        mbar_expect_tx(&full_p[st], cnt * (TILE_Q + TB));
        unsigned char* dst = sP + st * STAGE;
        bulk_g2s(dst, wsrc + (int64_t)j * KBS * TILE_Q, cnt * TILE_Q, &full_p[st]);
        bulk_g2s(dst + KBS * TILE_Q, bsrc + (int64_t)j * KBS * TB, cnt * TB, &full_p[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer: one TMEM accumulator per 128-column scale group (NACC buffers)
      constexpr uint32_t idesc = idesc_bf16(BN);
      for (int i = 0; i < nk; ++i) {
        const int st = i % DS, r = i / DS;
        const int gi = i >> 1, b = gi % NACC;
        const bool first = (i & 1) == 0;
        if (first && gi >= NACC) mbar_wait(&acce[b], ((gi / NACC) - 1) & 1);
        mbar_wait(&full_d[st], r & 1);
        tl_mark(768 + i);
        tc_fence_after();
        const uint64_t da = sw128_desc(su32(sD + st * (TILE_A + TB)));
        const uint64_t db = sw128_desc(su32(sD + st * (TILE_A + TB) + TILE_A));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          umma_bf16(tmem + b * BN, da + 2 * k, db + 2 * k, idesc, !(first && k == 0));
        umma_commit(&empty_d[st]);
        if (!first) umma_commit(&accf[b]);
      }
    }
  } else if (warp < 10) {  // dequant warps: threads 2r, 2r+1 own the two halves of tile row r
    const int t = threadIdx.x - 64;
    const int r = t >> 1, hf = t & 1;
    for (int i = 0; i < nk; ++i) {
      const int j = i / KBS, w = i - j * KBS;
      const int ps = j % PS, pr = j / PS, ds = i % DS, dr = i / DS;
      const int cnt = min(KBS, nk - j * KBS);
      mbar_wait_sleep(&full_p[ps], pr & 1);
      if (t == 0) tl_mark(256 + i);
      if (dr > 0) mbar_wait_sleep(&empty_d[ds], (dr - 1) & 1);
      if (t == 0) tl_mark(1024 + i);
      const uint32_t src = su32(sP + ps * STAGE);
      const uint32_t dst = su32(sD + ds * (TILE_A + TB));
      const uint4 w0 = lds128(src + w * TILE_Q + r * 32 + hf * 16);
      const uint32_t ws[4] = {w0.x, w0.y, w0.z, w0.w};
#pragma unroll
      for (int wi = 0; wi < 4; ++wi) sts128(dst + sw128_off(r, 8 * (4 * hf + wi)), dequant8(ws[wi]));
      for (int c = t; c < TB / 16; c += 256) sts128(dst + TILE_A + 16 * c, lds128(src + KBS * TILE_Q + w * TB + 16 * c));
      fence_proxy_async_smem();
      mbar_arrive(&full_d[ds]);
      if (t == 0) tl_mark(512 + i);
      if (w == cnt - 1) mbar_arrive(&empty_p[ps]);
    }
  } else {  // epilogue warps 10..13: per-group scale, fp32 accumulation in registers
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint16_t* sc = reinterpret_cast<const uint16_t*>(a.w_base + ((int64_t)a.expert_base + a.group_buf[g]) * a.blob_bytes +
                                                           a.s_off) +
                         ((int64_t)rt * (a.kdim / 128) + kb0 / 2) * BM + row;
    float acc[BN];
#pragma unroll
    for (int j = 0; j < BN; ++j) acc[j] = 0.0f;
    // the per-row scales of 8 groups are fetched together, ahead of their accumulators, so the
    // drain of one group never waits on a global-memory round trip
    constexpr int SW = 8;
    float scw[SW];
    for (int gi = 0; gi < ngr; ++gi) {
      if (gi % SW == 0) {
#pragma unroll
        for (int u = 0; u < SW; ++u) scw[u] = gi + u < ngr ? bf2f(sc[(int64_t)(gi + u) * BM]) : 0.0f;
      }
      const int b = gi % NACC;
      const float scale = scw[gi % SW];
      mbar_wait_sleep(&accf[b], (gi / NACC) & 1);
      if (threadIdx.x == 320) tl_mark(1280 + gi);
      tc_fence_after();
      float v[BN];
      tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + b * BN, v);
      if (BN == 32) tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + b * BN + 16, v + 16);
      tc_fence_before();
      mbar_arrive(&acce[b]);
#pragma unroll
      for (int j = 0; j < BN; ++j) acc[j] = fmaf(scale, v[j], acc[j]);
    }
    for (int j = 0; j < m && j < BN; ++j) outp[(int64_t)(e0 + j) * a.rows + rt * BM + row] = acc[j];
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
    const uint32_t v = q[i];
    uint32_t o = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t nib = (v >> (4 * j)) & 0xFu;
      o |= nib << ((j & 1) ? 16 + 4 * (j >> 1) : 4 * (j >> 1));
    }
    const int rt = (int)(r / BM), rr = (int)(r % BM), kb = w / 8, ww = w % 8;
    tq[(((int64_t)rt * kbt + kb) * BM + rr) * 8 + ww] = o;
  }
  const int64_t ns = (int64_t)rows * ngr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ngr;
    const int gg = (int)(i - r * ngr);
    ts[(((int64_t)(r / BM) * ngr) + gg) * BM + (r % BM)] = sc[i];
  }
}

}  // namespace

cudaError_t launch_umma_grouped(const UmmaArgs& a, int max_groups, int BN, cudaStream_t st) {
  constexpr int STAGES = 6;
  const int units = max_groups * (a.rows / BM) * a.splits;
  if (units == 0) return cudaSuccess;
  if (BN == 16) {
    const size_t smem = 1024 + STAGES * (TILE_A + 16 * 128) + (2 * STAGES + 2) * 8 + 16;
    cudaFuncSetAttribute(k_umma_grouped<16, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_umma_grouped<16, STAGES><<<units, 192, smem, st>>>(a);
  } else {
    const size_t smem = 1024 + STAGES * (TILE_A + 32 * 128) + (2 * STAGES + 2) * 8 + 16;
    cudaFuncSetAttribute(k_umma_grouped<32, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_umma_grouped<32, STAGES><<<units, 192, smem, st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t launch_umma_int4(const UmmaArgs& a, int max_groups, int BN, cudaStream_t st) {
  // 2 k-blocks per bulk stage x 6 stages (72 KB of packed weights in flight per CTA), 2
  // dequantised slots, 4 TMEM accumulators (one per in-flight 128-column scale group), 8
  // dequant warps: ~108 KB smem and <= 72 registers -> 2 CTAs/SM
  constexpr int KBS = 2, PS = 6, DS = 2, NACC = 4;
  const int units = max_groups * (a.rows / BM) * a.splits;
  if (units == 0) return cudaSuccess;
  auto smem = [&](int bn) {
    return (size_t)1024 + DS * (TILE_A + bn * 128) + PS * KBS * (BM * BK / 2 + bn * 128) +
           (2 * PS + 2 * DS + 2 * NACC) * 8 + 16;
  };
  if (BN == 16) {
    cudaFuncSetAttribute(k_umma_int4<16, KBS, PS, DS, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(16));
    k_umma_int4<16, KBS, PS, DS, NACC><<<units, 448, smem(16), st>>>(a);
  } else {
    cudaFuncSetAttribute(k_umma_int4<32, KBS, PS, DS, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem(32));
    k_umma_int4<32, KBS, PS, DS, NACC><<<units, 448, smem(32), st>>>(a);
  }
  return cudaGetLastError();
}

cudaError_t debug_int4_timeline(long long* dst, int n) {
  return cudaMemcpyFromSymbol(dst, g_int4_tl, sizeof(long long) * std::min(n, 2048));
}

cudaError_t launch_tile_int4(const uint32_t* q, const uint16_t* s, int rows, int cols, uint32_t* tq, uint16_t* ts,
                             cudaStream_t st) {
  k_tile_int4<<<148 * 4, 256, 0, st>>>(q, s, rows, cols, tq, ts);
  return cudaGetLastError();
}

cudaError_t launch_gather_b(const uint16_t* x, int ld, SchedPtrs s, int max_groups, int kdim, int BN,
                            unsigned char* img, cudaStream_t st) {
  k_gather_b<<<dim3(kdim / BK, max_groups), 128, 0, st>>>(x, ld, s, kdim, BN, img);
  return cudaGetLastError();
}

cudaError_t launch_finalize_act(const float* p1, int splits, int64_t split_stride, SchedPtrs s,
                                const int32_t* entry_group, int n_entries, int f, int BN, unsigned char* img,
                                cudaStream_t st) {
  k_finalize_act<<<dim3((f + 255) / 256, n_entries), 256, 0, st>>>(p1, splits, split_stride, s, entry_group,
                                                                    n_entries, f, BN, img);
  return cudaGetLastError();
}

cudaError_t launch_tile_bf16(const uint16_t* src, int rows, int cols, unsigned char* dst, cudaStream_t st) {
  k_tile_bf16<<<148 * 8, 256, 0, st>>>(src, rows, cols, dst);
  return cudaGetLastError();
}

}  // namespace mspq
