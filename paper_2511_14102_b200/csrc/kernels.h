// Internal launcher interface between the C-ABI / host engine and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <utility>

namespace mspq {

// Programmatic dependent launch (PDL) for back-to-back kernels on one stream.  A kernel launched
// with launch_pdl() may be resident before its predecessor finishes, so it must start with
// pdl_enter(): griddepcontrol.wait (the predecessor's writes are complete and visible; nothing may be
// read before it) then launch_dependents (lets the next PDL kernel get scheduled).
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}
#endif
template <typename... P, typename... A>
inline cudaError_t launch_pdl(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

// Expert-grouped schedule (K3's reorder_verification output); device pointers.
struct SchedPtrs {
  int32_t* n_groups;      // [1]
  int32_t* group_expert;  // [G]
  int32_t* group_buf;     // [G]   HBM slot-pool buffer (verify) / expert id (draft)
  int32_t* group_off;     // [G+1] entry offsets
  int32_t* entry_tok;     // [N]   window token of each entry
  int32_t* entry_of;      // [T*K] entry index of (token, k-slot)
  int32_t* entry_group;   // [N]   group of each entry (nullable)
};

// Group subset of a grouped GEMM launch (groups < 256): the verify runs the groups whose experts
// are already resident while the missing ones are still on the link, then the rest.
struct GMask {
  uint32_t w[8];
  int on;
};
__host__ __device__ inline bool gmask_has(const GMask& m, int g) {
  return !m.on || (g < 256 && ((m.w[g >> 5] >> (g & 31)) & 1u));
}

// tcgen05 grouped GEMM (umma.cu): one matrix (W13 or W2) of every group's expert
struct UmmaArgs {
  const unsigned char* w_base;  // slot pool of tile-major bf16 expert blobs
  int64_t blob_bytes;
  int64_t w_off;                // byte offset of the matrix inside a blob
  int rows, kdim;               // rows (2f | d), K (d | f)
  const int32_t* n_groups;
  const int32_t* group_buf;
  const int32_t* group_off;
  const unsigned char* bimg;    // [G][kdim/64][BN*128] swizzled B images
  float* out;                   // [splits][N][rows] fp32 partial planes
  int64_t out_split_stride;
  int splits;
  int64_t s_off;                // INT4: byte offset of the matrix's scales inside a blob
  int expert_base;              // INT4: blob index = expert_base + group_buf[g]
  int brows = 0;                // rows per B image (8 = aliased 8-row tiles, else BN)
  const float* csum = nullptr;  // INT4: [G][brows][kdim/64] epilogue corrections (see k_gather_b)
  const uint16_t* xsrc = nullptr;  // INT4 self-gather: bf16 token rows [.][kdim] (one token per group)
  int xsrc_by_entry = 0;           // row of group g = entry_tok[e0] (0) or the entry e0 (1)
  const int32_t* entry_tok = nullptr;
  uint16_t* act_out = nullptr;     // INT4 W13, split 1: fused act = bf16(silu(gate) * up) [N][rows/2]
  GMask gmask{};                   // K3: only the groups whose bit is set (when gmask.on)
  unsigned char* act_img = nullptr;  // K3 W13, split 1: fused SiLU*up straight into W2's B images
  // K3: the schedule and the A (weight) bytes were complete before the PREDECESSOR kernel's
  // griddepcontrol.wait returned, so the producer may read the schedule and stream its first A
  // tiles before its own wait (overlapping the predecessor's tail); only B waits
  int early_a = 0;
};


// Draft-loop state living on the device so a draft step is a replayable CUDA graph.
struct DraftState {
  int32_t* row;         // ELB row / draft index
  int32_t* draft_toks;  // [kmax]
  int32_t* cur_tok;
  int32_t* cur_pos;
};

struct RouteArgs {
  float* h;                  // [T][d] residual, updated in place by the combine
  const float* y;            // [N][d] expert outputs of the previous layer (nullable)
  const int32_t* entry_of;   // [T][K] entry index of (t, j) in y
  const float* prev_wts;     // [T][K]
  const uint16_t* gamma;     // [d]
  const uint16_t* router;    // [E][d] (nullable -> norm only)
  uint16_t* xn;              // [T][d]
  int32_t* ids;              // [T][K]
  float* wts;                // [T][K]
  float* logits;             // [T][E] (nullable)
  int y_splits;              // K-split partial planes of y, summed in order by the combine
  int64_t y_split_stride;
  int32_t* elb_ids;          // [kmax][L][K] (nullable)
  float* elb_gates;
  const int32_t* elb_row;    // device row counter
  int32_t* sched;            // T == 1: packed draft schedule (nullable), see mspq_gate_topk
  int layer, L, d, E, K;
  float eps;
  unsigned char* bimg = nullptr;  // also write xn as the SW128 B image of a dense GEMM (nullable)
  int bimg_bn = 16;               // rows per B image k-block
  int stage = 0;                  // set by launch_route: h and every y plane of the token land in smem
                                  // by one round of bulk copies instead of one round trip per plane
};

// Shared-KV decode attention over a window of T tokens (attention.cu)
struct AttnArgs {
  const float* qkv;        // [splits][T][(H + 2 Hkv) Dh] fp32 partial planes of the QKV projection
  int splits;
  int64_t split_stride;
  int T, H, Hkv, Dh, P;
  const int32_t* pos0;     // device: position of window token 0
  uint16_t* kc;            // this layer's K cache [P][Hkv][Dh] bf16
  uint16_t* vc;            // V cache
  uint16_t* out;           // [T][H Dh] bf16 attention output (nullable)
  float scale;             // 1/sqrt(Dh)
  unsigned char* oimg = nullptr;  // the output as the O projection's SW128 B image (nullable)
  int o_bn = 16;
  // workspace (attn_part_floats(T, H, Hkv, Dh) words, zeroed once): [AT_CNT merge counters][split-K
  // partials]; the launcher points part / cnt into it
  float* part = nullptr;
  const int32_t* meta = nullptr;  // batched streams: per token (window base row, stream, position)
  int64_t kv_stream_stride = 0;   // elements between two streams' caches (same layer)
  int* cnt = nullptr;             // [T][Hkv] arrivals of the split CTAs (the last one merges, resets to 0)
};
constexpr int AT_CNT = 2048;  // merge counters at the head of the attention workspace: T * Hkv <= AT_CNT
size_t attn_smem_bytes(int T, int H, int Hkv, int Dh, int P);
size_t attn_part_floats(int T, int H, int Hkv, int Dh);
cudaError_t launch_attn_window(const AttnArgs& a, cudaStream_t st);

// K2 for one token: INT4 expert GEMV on warp MMA over fragment-major weights (gemv_int4.cu)
struct GemvArgs {
  const unsigned char* blobs;  // all L*E draft blobs (fragment-major q, row-major scales)
  int64_t blob_bytes;
  int64_t q_off, s_off;        // the matrix's q words and scales inside a blob
  int rows, kdim;
  int layer, E;
  const int32_t* n_groups;     // the draft schedule: group g = expert group_expert[g] = entry g
  const int32_t* group_expert;
  const uint16_t* x;           // bf16 input rows
  int x_per_group;             // 0: one row for every group (W13), 1: row g (W2 on the act rows)
  float* y;                    // W2: [ksplit][groups][rows] fp32 planes
  uint16_t* act;               // W13: [groups][rows/2] bf16 SiLU(gate) * up
};
cudaError_t launch_int4_gemv(const GemvArgs& a, int max_groups, int ksplit, cudaStream_t st);
cudaError_t launch_fragtile_int4(const uint32_t* q, int rows, int cols, uint32_t* fq, cudaStream_t st);
void gemv_set_variant(int v);

cudaError_t launch_umma_grouped(const UmmaArgs& a, int max_groups, int BN, cudaStream_t st);
cudaError_t launch_umma_int4(const UmmaArgs& a, int max_groups, int BN, cudaStream_t st);
cudaError_t launch_umma_int4p(const UmmaArgs& a, int max_groups, cudaStream_t st);
cudaError_t debug_int4_timeline(long long* dst, int n);
cudaError_t launch_tile_int4(const uint32_t* q, const uint16_t* s, int rows, int cols, uint32_t* tq, uint16_t* ts,
                             cudaStream_t st);
cudaError_t launch_gather_b(const uint16_t* x, int ld, SchedPtrs s, int max_groups, int kdim, int BN,
                            unsigned char* img, cudaStream_t st, float* csum = nullptr);
cudaError_t launch_finalize_act(const float* p1, int splits, int64_t split_stride, SchedPtrs s,
                                const int32_t* entry_group, int n_entries, int f, int BN, unsigned char* img,
                                cudaStream_t st, float* csum = nullptr, GMask gm = GMask{});
cudaError_t launch_tile_bf16(const uint16_t* src, int rows, int cols, unsigned char* dst, cudaStream_t st);
cudaError_t launch_fill_bf16(uint64_t seed, uint64_t tensor, float scale, int kind, uint16_t* out,
                             int64_t n, int64_t start, cudaStream_t st);
cudaError_t launch_fill_expert(uint64_t seed, int cl, int ce, int d, int f, float a_up,
                               float a_down, uint16_t* blob, cudaStream_t st);
cudaError_t launch_quantize(const uint16_t* w, int rows, int cols, uint32_t* q, uint16_t* s,
                            cudaStream_t st);
cudaError_t launch_embed(const uint16_t* embed, const uint16_t* pos, const int32_t* tokens,
                         const int32_t* positions, int T, int d, float* h, cudaStream_t st);
cudaError_t launch_route(const RouteArgs& a, int T, cudaStream_t st);
cudaError_t launch_build_schedule(const int32_t* ids, int T, int K, int E, const int32_t* gbuf,
                                  SchedPtrs s, cudaStream_t st);
cudaError_t launch_lm_head(const uint16_t* xn, const uint16_t* lm, int T, int V, int d,
                           float* logits, cudaStream_t st);
cudaError_t launch_argmax(const float* logits, int T, int V, int32_t* out, DraftState ds,
                          cudaStream_t st);
cudaError_t launch_accept(const int32_t* draft, const int32_t* tgt, int k, int32_t* res,
                          int32_t* cur_tok, int32_t* cur_pos, int head_pos, cudaStream_t st);

}  // namespace mspq
