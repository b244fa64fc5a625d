// K2 for the draft step (T = 1): INT4 expert GEMV on warp-level MMA (mma.sync m16n8k16, f16 in,
// f32 accumulate) with the weights in FRAGMENT-MAJOR order, so one 16-byte load per lane is four
// ready-made A fragments after one LOP3 per two weights.
//
// Why not tcgen05 here: a single token is an N = 1 GEMM; the UMMA path (k_umma_int4p) pads it to
// N = 16 and moves every 8 KB weight group through smem -> TMEM A-slot -> MMA -> commit hand-offs,
// which capped it at ~1.4 TB/s (~0.2 of HBM, profiles/r01).  Here the weight bytes go straight
// from global memory into registers; the warp MMA does the dot products (its throughput is ~5x
// what one token needs) and the kernel is bound by the bytes in flight.
//
// Layout (mspq_fragtile_int4): W [R][C] -> q[R/16][C/64][32 lanes][4 words].  Word v of lane l
// covers k16-block kb = 4 * chunk + v, rows r0 = 16 rt + l/4, r1 = r0 + 8, columns c = 16 kb +
// 2 (l%4) + {0, 1} ("class 1") and c + 8 + {0, 1} ("class 16"):
//   bits  0 / 16: W[r0][c], W[r0][c+1]      bits  8 / 24: W[r1][c], W[r1][c+1]
//   bits  4 / 20: W[r0][c+8], W[r0][c+9]    bits 12 / 28: W[r1][c+8], W[r1][c+9]
// so (w & 0x000F000F) | 0x64006400 is the fp16 pair (1024 + q) for (a0, a1) and
// (w & 0x00F000F0) | 0x64006400 the pair (1024 + 16 q) for (a4, a5); w >> 8 gives rows r1.  The
// B fragment holds x for class-1 columns and x / 16 for class-16 ones, so D = sum_k (q_k - 8) x_k
// + C, C = sum_k c_k b_k (c = 1032 | 1152), the same exact-product scheme as the tcgen05 K2
// (DESIGN.md §5); the per-128-column bf16 scale is applied in fp32 per group.  Scales stay
// row-major [R][C/128].
#include "common.cuh"
#include "kernels.h"

namespace mspq {
namespace {

constexpr int GV_WARPS = 8, GV_THREADS = 32 * GV_WARPS;

MSPQ_D void mma16816(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
MSPQ_D uint32_t lop_magic(uint32_t w, uint32_t mask) {
  uint32_t o;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(o) : "r"(w), "r"(mask), "r"(0x64006400u));  // (w & mask) | magic
  return o;
}
template <bool H256>
MSPQ_D uint4 ldg_stream(const void* p) {
  uint4 v;
  if (H256)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
  return v;
}

// grid (R / 32, groups, ksplit): CTA = 32 rows of one group's expert matrix over the scale groups
// of its K split; the 8 warps take groups w, w + 8, ... of the split, partial rows reduced in warp
// order.  The first weight loads are issued before the x prologue (they do not depend on it), and
// each group's bias C_g = sum_k c_k b_k is reduced from the B fragments the lanes already hold
// (quad shuffles, fixed order) instead of a serial prologue.  K splits (W2) write separate planes
// [split][groups][rows] that the next K1 combine sums in order.
template <int GV_TILES, int NB, bool H256>
__global__ void __launch_bounds__(GV_THREADS) k_int4_gemv(GemvArgs a) {
  constexpr int ROWS = 16 * GV_TILES;
  // launched with launch_pdl (kernels.h).  W13 (x = the K1 output, schedule written by K1) waits
  // first.  W2's predecessor is W13, whose own wait ordered it after the K1 that wrote the schedule,
  // so W2 may read the schedule and issue its first weight loads (static data) before its wait --
  // they overlap W13's last wave -- and waits only before it reads W13's act rows.
  const bool early = a.x_per_group != 0;
  if (!early) pdl_enter();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int g = blockIdx.y, sp = blockIdx.z, S = gridDim.z;
  if (g >= *a.n_groups) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kdim = a.kdim, ngr = kdim / 128, nchunk = kdim / 64;
  const int gq0 = sp * ngr / S, gq1 = (sp + 1) * ngr / S;
  uint16_t* xh = reinterpret_cast<uint16_t*>(smem_raw);            // [kdim] class-scaled fp16
  float* red = reinterpret_cast<float*>(smem_raw + kdim * 2);       // [GV_WARPS][ROWS] row partials
  const int expert = a.group_expert[g];
  const unsigned char* blob = a.blobs + ((int64_t)a.layer * a.E + expert) * a.blob_bytes;
  const uint4* q = reinterpret_cast<const uint4*>(blob + a.q_off);
  const uint16_t* sc = reinterpret_cast<const uint16_t*>(blob + a.s_off);
  const int rt0 = blockIdx.x * GV_TILES;
  const int gi = lane >> 2, ti = lane & 3;
  // memory-level parallelism: a warp issues the loads of NB scale groups (NB x 2 KB) at once,
  // then multiplies them; the first batch is issued before the x prologue
  uint4 buf[NB][GV_TILES][2];
  auto load_batch = [&](int gfirst) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int gb = gfirst + b * GV_WARPS;
      if (gb < gq1)
#pragma unroll
        for (int i = 0; i < GV_TILES; ++i)
#pragma unroll
          for (int c = 0; c < 2; ++c)
            buf[b][i][c] = ldg_stream<H256>(q + (((int64_t)(rt0 + i) * nchunk + 2 * gb + c) * 32 + lane));
    }
  };
  int gq = gq0 + warp;
  load_batch(gq);
  if (early) pdl_enter();
  const uint16_t* x = a.x + (a.x_per_group ? (int64_t)g * kdim : 0);
  for (int k = 2 * tid; k < kdim; k += 2 * GV_THREADS) {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(x + k);
    const float m = (k & 15) >= 8 ? 0.0625f : 1.0f;
    const __half2 h2 = __floats2half2_rn(__uint_as_float(u << 16) * m, __uint_as_float(u & 0xffff0000u) * m);
    *reinterpret_cast<__half2*>(&xh[k]) = h2;
  }
  __syncthreads();
  float acc[GV_TILES][2];
#pragma unroll
  for (int i = 0; i < GV_TILES; ++i) acc[i][0] = acc[i][1] = 0.0f;
  for (; gq < gq1; gq += NB * GV_WARPS) {
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int gb = gq + b * GV_WARPS;
      if (gb >= gq1) break;
      float d[GV_TILES][4];
#pragma unroll
      for (int i = 0; i < GV_TILES; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.0f;
      float c1 = 0.0f, c16 = 0.0f;  // this lane's share of C_g: sum b over class-1 / class-16 columns
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int kb = 8 * gb + 4 * c + v;  // k16 block
          const uint32_t b0 = *reinterpret_cast<const uint32_t*>(&xh[16 * kb + 2 * ti]);
          const uint32_t b1 = *reinterpret_cast<const uint32_t*>(&xh[16 * kb + 8 + 2 * ti]);
          const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&b0));
          const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&b1));
          c1 = __fadd_rn(__fadd_rn(c1, f0.x), f0.y);
          c16 = __fadd_rn(__fadd_rn(c16, f1.x), f1.y);
#pragma unroll
          for (int i = 0; i < GV_TILES; ++i) {
            const uint4 wv = buf[b][i][c];
            const uint32_t w = v == 0 ? wv.x : v == 1 ? wv.y : v == 2 ? wv.z : wv.w;
            const uint32_t w8 = w >> 8;
            uint32_t af[4];
            af[0] = lop_magic(w, 0x000F000Fu);   // (r0, c..c+1)     1024 + q
            af[1] = lop_magic(w8, 0x000F000Fu);  // (r1, c..c+1)
            af[2] = lop_magic(w, 0x00F000F0u);   // (r0, c+8..c+9)   1024 + 16 q
            af[3] = lop_magic(w8, 0x00F000F0u);  // (r1, c+8..c+9)
            mma16816(d[i], af, b0, b1);
          }
        }
      // C_g over the quad's four column slices (lanes ti = 0..3 of a row group), fixed order
      float cl = fmaf(1152.0f, c16, __fmul_rn(1032.0f, c1));
      cl = __fadd_rn(cl, __shfl_xor_sync(0xffffffffu, cl, 1));
      cl = __fadd_rn(cl, __shfl_xor_sync(0xffffffffu, cl, 2));
#pragma unroll
      for (int i = 0; i < GV_TILES; ++i) {
        const int r0 = 16 * (rt0 + i) + gi;
        const float s0 = bf2f(sc[(int64_t)r0 * ngr + gb]), s1 = bf2f(sc[(int64_t)(r0 + 8) * ngr + gb]);
        acc[i][0] = fmaf(s0, __fsub_rn(d[i][0], cl), acc[i][0]);  // every B column is x: column 2 ti == column 0
        acc[i][1] = fmaf(s1, __fsub_rn(d[i][2], cl), acc[i][1]);
      }
    }
    if (gq + NB * GV_WARPS < gq1) load_batch(gq + NB * GV_WARPS);
  }
  if (ti == 0) {
#pragma unroll
    for (int i = 0; i < GV_TILES; ++i) {
      red[warp * ROWS + 16 * i + gi] = acc[i][0];
      red[warp * ROWS + 16 * i + gi + 8] = acc[i][1];
    }
  }
  __syncthreads();
  if (tid < ((ROWS + 31) & ~31)) {  // whole warps (the shuffle below needs every lane)
    float v = 0.0f;
    if (tid < ROWS)
#pragma unroll
      for (int w = 0; w < GV_WARPS; ++w) v = __fadd_rn(v, red[w * ROWS + tid]);
    const int row = ROWS * blockIdx.x + tid;
    if (a.act) {
      // W13 rows 2i / 2i+1 = gate_i / up_i (adjacent lanes of one warp): act = bf16(silu(gate) * up)
      const float up = __shfl_down_sync(0xffffffffu, v, 1);
      if ((tid & 1) == 0 && tid < ROWS) a.act[(int64_t)g * (a.rows / 2) + row / 2] = f2bf(__fmul_rn(silu_det(v), up));
    } else if (tid < ROWS) {
      a.y[((int64_t)sp * gridDim.y + g) * a.rows + row] = v;
    }
  }
}

// row-major quantised INT4 (standard nibble order) -> fragment-major words (header comment)
__global__ void k_fragtile_int4(const uint32_t* __restrict__ q, int rows, int cols, uint32_t* __restrict__ fq) {
  const int wpr = cols / 8, nchunk = cols / 64;
  const int64_t n = (int64_t)rows * wpr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(i & 3), lane = (int)((i >> 2) & 31);
    const int64_t rest = i >> 7;
    const int chunk = (int)(rest % nchunk);
    const int64_t rt = rest / nchunk;
    const int r0 = (int)(16 * rt + (lane >> 2)), r1 = r0 + 8;
    const int c = 16 * (4 * chunk + v) + 2 * (lane & 3);
    auto nib = [&](int r, int col) { return (q[(int64_t)r * wpr + (col >> 3)] >> (4 * (col & 7))) & 0xFu; };
    fq[i] = nib(r0, c) | (nib(r0, c + 1) << 16) | (nib(r1, c) << 8) | (nib(r1, c + 1) << 24) | (nib(r0, c + 8) << 4) |
            (nib(r0, c + 9) << 20) | (nib(r1, c + 8) << 12) | (nib(r1, c + 9) << 28);
  }
}

}  // namespace

static int g_gemv_variant = 0;  // tools/gemv_bench.py A/B only (mspq_debug_gemv_variant)
void gemv_set_variant(int v) { g_gemv_variant = v; }

template <int TILES, int NB, bool H256>
static cudaError_t launch_gemv_v(const GemvArgs& a, int max_groups, int ksplit, cudaStream_t st) {
  const size_t smem = (size_t)a.kdim * 2 + GV_WARPS * 16 * TILES * 4 + 16;
  if (a.rows % (16 * TILES)) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_int4_gemv<TILES, NB, H256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  return launch_pdl(k_int4_gemv<TILES, NB, H256>, dim3(a.rows / (16 * TILES), max_groups, ksplit), dim3(GV_THREADS),
                    smem, st, a);
}

cudaError_t launch_int4_gemv(const GemvArgs& a, int max_groups, int ksplit, cudaStream_t st) {
  // default: 64 rows per CTA, 2 scale groups (8 KB per warp) per load batch -- best of the A/B at
  // the three BASELINE shapes (profiles/r02/gemv_variants.txt: Phi 2.81, Qwen3 1.67, Mixtral 3.81
  // TB/s in-stream; 32 rows x 4 groups: 2.74 / 1.30 / 3.50; tcgen05 K2: 1.49 / 0.86 / 1.88)
  switch (g_gemv_variant) {
    case 1: return launch_gemv_v<2, 4, true>(a, max_groups, ksplit, st);
    case 3: return launch_gemv_v<1, 4, false>(a, max_groups, ksplit, st);
    case 4: return launch_gemv_v<2, 2, false>(a, max_groups, ksplit, st);
    case 5: return launch_gemv_v<2, 4, false>(a, max_groups, ksplit, st);
    default: return launch_gemv_v<4, 2, false>(a, max_groups, ksplit, st);
  }
}

cudaError_t launch_fragtile_int4(const uint32_t* q, int rows, int cols, uint32_t* fq, cudaStream_t st) {
  k_fragtile_int4<<<148 * 4, 256, 0, st>>>(q, rows, cols, fq);
  return cudaGetLastError();
}

}  // namespace mspq
