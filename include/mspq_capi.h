/*
 * mspq_capi.h — the C-ABI of the B200-native MoE-SpeQ decode path (libmspq.so).
 *
 * Two layers, both plain C (no torch / C++ types; device pointers are void*, streams are
 * cudaStream_t passed as void*; every call returns an int status and never throws):
 *
 *  (1) Kernel entry points the host engine calls through (SURVEY.md §8b "C-ABI"):
 *        mspq_gate_topk        K1  fused residual-combine + RMSNorm + bf16 router + top-k/softmax
 *                                  (replaces the reference's trace-supplied routing:
 *                                   TokenRecord.target_sets/draft_sets/draft_gates, trace.hpp:43-49,
 *                                   and build_elb's input, scheduler.cpp:41-63)
 *        mspq_build_schedule       expert-grouped entry schedule == reorder_verification
 *                                  (scheduler.cpp:339-357)
 *        mspq_moe_int4_gemv    K2  INT4 (RTN on the GPTQ sym g128 grid) expert FFN of the draft token
 *        mspq_moe_bf16_tc      K3  bf16 grouped expert FFN for the verify (reads the HBM slot pool)
 *        mspq_lm_head / mspq_argmax  logits + greedy token
 *        mspq_accept_scan      K5  accept rule (sim.cpp:352-365) on token ids
 *      plus weight generation / quantisation helpers used by tests.
 *
 *  (2) The engine: the drop-in for the reference's run_simulation (sim.hpp:86) entry point.
 *        mspq_replay           device control plane (K4) over a reference Trace, returning the
 *                              reference's SimReport JSON (sim.cpp:468-510) -- bit-exact.
 *        mspq_engine_create / mspq_engine_configure / mspq_generate
 *                              live speculative decode: INT4 draft -> ELB -> 3-phase prefetch over
 *                              PCIe copy engines into a capped HBM slot pool -> bf16 grouped
 *                              verify -> accept -> Amortization-Roofline governor; returns the
 *                              same SimReport JSON with measured times + per-cycle traces.
 *
 * Status codes: 0 = OK; 1..18 = moespeq::ErrorCode ordinal + 1 (errors.hpp:8-27, same order);
 * 1000 = CUDA error; 1001 = capacity/overflow in the device controller; 2000 = internal.
 */
#ifndef MSPQ_CAPI_H
#define MSPQ_CAPI_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSPQ_OK 0
#define MSPQ_ERR_MALFORMED_RECORD 1
#define MSPQ_ERR_SHAPE_VIOLATION 2
#define MSPQ_ERR_EMPTY_TRACE 3
#define MSPQ_ERR_INVALID_FIDELITY 4
#define MSPQ_ERR_DEGENERATE_SHAPE 5
#define MSPQ_ERR_LAYER_OUT_OF_RANGE 6
#define MSPQ_ERR_SHAPE_MISMATCH 7
#define MSPQ_ERR_RANGE_OUT_OF_BOUNDS 8
#define MSPQ_ERR_EMPTY_CACHE 9
#define MSPQ_ERR_UNKNOWN_POLICY 10
#define MSPQ_ERR_EMPTY_REQUIRED 11
#define MSPQ_ERR_INCOMPLETE_ROUTING 12
#define MSPQ_ERR_K_OUT_OF_RANGE 13
#define MSPQ_ERR_INSUFFICIENT_SAMPLES 14
#define MSPQ_ERR_EMPTY_RANGE 15
#define MSPQ_ERR_INFEASIBLE_BUDGET 16
#define MSPQ_ERR_INVALID_CONFIG 17
#define MSPQ_ERR_IO 18
#define MSPQ_ERR_CUDA 1000
#define MSPQ_ERR_OVERFLOW 1001
#define MSPQ_ERR_INTERNAL 2000

/* Model / draft config (the reference's ModelShape, trace.hpp:29-37, plus the dimensions a
 * real model needs).  Scales are the fp32 values the weight generator multiplies by. */
typedef struct mspq_model_desc {
  int L, E, K;      /* MoE layers, experts per layer, top-k */
  int d, f, V, P;   /* hidden, expert ffn, vocab, positional rows */
  unsigned long long seed;
  float embed_scale, pos_scale, a_router, a_up, a_down, a_lm, eps;
  int unique_experts; /* 0 = every (layer, expert) distinct; else payload = key % unique */
  /* attention (shared by draft and target, bf16): H query heads, Hkv KV heads,
   * head dim Dh; H = 0 = attention-free layers.  a_qkv / a_o scale Wqkv [(H+2Hkv)Dh][d] and
   * Wo [d][H Dh]. */
  int H, Hkv, Dh;
  float a_qkv, a_o;
} mspq_model_desc;

typedef struct mspq_engine_opts {
  int device;
  int kmax;                     /* longest speculation window the buffers are sized for */
  const char* host_store_path;  /* NULL/"" = private cudaHostAlloc; else /dev/shm file shared
                                   by all ranks (rank with host_store_role 0 creates + fills) */
  int host_store_role;
  int slot_extra;               /* extra HBM buffers beyond the cache budget (0 = auto) */
  int log_cap;                  /* per-cycle event log capacity (0 = auto) */
  int trace_level;              /* 0 = counts only, 1 = per-cycle tokens/routing, 2 = + event log */
  int expert_codec;             /* host-store format of the bf16 experts: 0 = raw tile images,
                                   1 = XC lossless blobs (mspq_xc_encode), decoded on the GPU */
  int max_streams;              /* request streams mspq_generate_batch can run together (<= 1 = one) */
} mspq_engine_opts;

typedef struct mspq_engine mspq_engine;

const char* mspq_status_string(int status);
const char* mspq_last_error(void);
void mspq_free(void* p);
int mspq_version(void);

/* ---------------------------------------------------------------- (1) kernel entry points */
int mspq_fill_bf16(unsigned long long seed, unsigned long long tensor, float scale, int kind,
                   void* out_bf16, long long n, long long start, void* stream);
int mspq_fill_expert(unsigned long long seed, int layer, int expert, int d, int f, float a_up,
                     float a_down, void* blob_bf16, void* stream);
int mspq_quantize_int4(const void* w_bf16, int rows, int cols, void* q_u32, void* s_bf16,
                       void* stream);
int mspq_embed(const void* embed, const void* pos, const int32_t* tokens,
               const int32_t* positions, int T, int d, float* h, void* stream);
/* K1.  y/entry_of/prev_wts may be NULL (no combine); entry_of == NULL with y != NULL is the
 * dense combine h[t] += y[t] (the attention output projection); y may hold y_splits partial planes
 * y_split_stride floats apart (summed in order); router NULL = norm only;
 * elb_ids/elb_gates/elb_row NULL = no ELB write.  sched_block (T == 1 only, nullable): also
 * write the token's expert-grouped schedule, packed [n_groups, pad x3, group_expert[K],
 * group_buf[K], group_off[K+1], entry_tok[K], entry_of[K], entry_group[K]]. */
int mspq_gate_topk(float* h, const float* y, const int32_t* entry_of, const float* prev_wts,
                   int y_splits, long long y_split_stride, const void* gamma, const void* router, void* xn, int32_t* ids, float* wts,
                   float* logits, int32_t* elb_ids, float* elb_gates, const int32_t* elb_row,
                   int32_t* sched_block, int layer, int L, int T, int d, int E, int K, float eps,
                   void* stream);
/* K1 that also writes xn as the SW128 B image of a dense tcgen05 GEMM (mspq_dense_bf16_tc with
 * x = NULL reads it from its workspace): bimg = that workspace, T <= 32 */
int mspq_gate_topk_img(float* h, const float* y, const int32_t* entry_of, const float* prev_wts,
                       int y_splits, long long y_split_stride, const void* gamma, const void* router, void* xn,
                       int32_t* ids, float* wts, float* logits, int32_t* elb_ids, float* elb_gates,
                       const int32_t* elb_row, int32_t* sched_block, int layer, int L, int T, int d, int E, int K,
                       float eps, void* bimg, void* stream);
/* schedule arrays: n_groups[1], group_expert[G], group_buf[G], group_off[G+1], entry_tok[T*K],
 * entry_of[T*K]; gbuf[E] (nullable) gives group_buf per expert (else group_buf = expert id) */
int mspq_build_schedule(const int32_t* ids, int T, int K, int E, const int32_t* gbuf, int32_t* n_groups,
                        int32_t* group_expert, int32_t* group_buf, int32_t* group_off,
                        int32_t* entry_tok, int32_t* entry_of, int32_t* entry_group, void* stream);
/* K3 on tcgen05 (umma.cu): the same grouped FFN over TILE-MAJOR bf16 experts (each 128x64
 * block a contiguous SW128 K-major image, see mspq_tile_bf16).  Runs gather -> W13 GEMM ->
 * SiLU*up -> W2 GEMM.  split1/split2 = K splits of the two GEMMs; y = [split2][T*K][d] fp32
 * partial planes (feed mspq_gate_topk with y_splits = split2, stride = T*K*d). */
long long mspq_moe_bf16_tc_ws_bytes(int d, int f, int T, int K, int max_groups, int max_split1);
int mspq_moe_bf16_tc(const int32_t* n_groups, const int32_t* group_expert, const int32_t* group_buf,
                     const int32_t* group_off, const int32_t* entry_tok, const int32_t* entry_group,
                     const void* xn, const void* pool, long long blob_bytes, int d, int f, int T,
                     int K, int max_groups, int split1, int split2, void* ws, float* y,
                     void* stream);
/* K3 on a group subset: only the groups g < 256 whose bit is set in gmask8[8] (NULL = all); the
 * gather of the token images runs when do_gather.  The engine runs the groups whose experts are
 * resident while the missing ones are still being copied, then the rest (same outputs). */
int mspq_moe_bf16_tc_part(const int32_t* n_groups, const int32_t* group_expert, const int32_t* group_buf,
                          const int32_t* group_off, const int32_t* entry_tok, const int32_t* entry_group,
                          const void* xn, const void* pool, long long blob_bytes, int d, int f, int T,
                          int K, int max_groups, int split1, int split2, void* ws, float* y,
                          const uint32_t* gmask8, int do_gather, void* stream);
/* K2 on tcgen05 (umma.cu k_umma_int4): the INT4 draft FFN over TILE-MAJOR INT4 blobs
 * (mspq_tile_int4), blobs indexed by layer*E + group_buf[g] (= expert id for the draft
 * schedule).  Exact dequant (GPTQ sym grid): bf16 (q-8) tiles into smem, per-128-column scales in the
 * fp32 epilogue.  Same workspace size / outputs as mspq_moe_bf16_tc. */
int mspq_moe_int4_tc(const int32_t* n_groups, const int32_t* group_expert, const int32_t* group_buf,
                     const int32_t* group_off, const int32_t* entry_tok, const int32_t* entry_group,
                     const void* xn, const void* blobs, long long blob_bytes, int layer, int E, int d,
                     int f, int T, int K, int max_groups, int split1, int split2, void* ws, float* y,
                     void* stream);
/* Dense bf16 projection on tcgen05 (K3's grouped GEMM with one group of T tokens):
 * out[split][T][rows] fp32 partial planes (out_split_stride floats apart) = x[T][kdim] . W^T,
 * W tile-major SW128 (mspq_tile_bf16).  dsched: device copy of the packed schedule
 * mspq_dense_sched_fill writes (4 + T ints); ws: mspq_dense_ws_bytes(kdim, T) bytes.  x = NULL:
 * ws already holds the B image (written by mspq_gate_topk_img or mspq_attention). */
long long mspq_dense_ws_bytes(int kdim, int T);
int mspq_dense_sched_fill(int32_t* host_packed, int T);
int mspq_dense_bf16_tc(const int32_t* dsched, const void* x, const void* w_tiled, int rows, int kdim, int T,
                       int split, void* ws, float* out, long long out_split_stride, void* stream);
/* Shared-KV decode attention over a window of T tokens at positions *pos0 .. *pos0+T-1 (device
 * pointer): qkv = the QKV projection's split planes [splits][T][(H+2Hkv) Dh]; the window's K/V
 * rows are written into kc/vc ([P][Hkv][Dh] bf16, this layer) and every token attends causally
 * to the cache rows before the window plus the window tokens up to itself; out [T][H Dh] bf16
 * (nullable) and/or oimg = the O projection's B image (a dense GEMM workspace, x = NULL).  Split-K
 * over the context (16 key chunks per token and KV head, merged in order by the last chunk's CTA);
 * ws = mspq_attention_ws_bytes(T, H, Hkv, Dh) bytes, ZERO-FILLED before the first call (its merge
 * counters return to zero after every call); P <= 4096, T * Hkv <= 2048.
 * Draft and target share the cache; rollback = the next window overwrites rows >= its pos0. */
long long mspq_attention_ws_bytes(int T, int H, int Hkv, int Dh);
int mspq_attention(const float* qkv, int splits, long long split_stride, int T, int H, int Hkv, int Dh, int P,
                   const int32_t* pos0, void* kc, void* vc, void* out, void* oimg, void* ws, void* stream);
/* K2 for the draft's single token: INT4 expert GEMV on warp MMA (gemv_int4.cu).  blobs = L*E
 * draft blobs in FRAGMENT-MAJOR order (mspq_fragtile_int4 for q, scales row-major: W13q | W13s |
 * W2q | W2s with the mspq_int4_blob_bytes offsets); groups = the K experts of the token in the
 * draft schedule (n_groups / group_expert, group g = entry g); act [K][f] bf16 scratch (SiLU(gate)
 * * up of W13, fused); y [split2][K][d] fp32 planes (W2 split over its K dimension; the
 * consumer sums them in order). */
int mspq_moe_int4_gemv(const int32_t* n_groups, const int32_t* group_expert, const void* xn, const void* blobs,
                       long long blob_bytes, int layer, int E, int d, int f, int K, int split2, void* act, float* y,
                       void* stream);
/* row-major quantised INT4 q[rows][cols/8] (standard nibble order) -> fragment-major words
 * [rows/16][cols/64][32 lanes][4] for mspq_moe_int4_gemv (layout in gemv_int4.cu) */
int mspq_fragtile_int4(const void* q, int rows, int cols, void* fq, void* stream);
/* diagnostics: tile/batch variant of the draft GEMV (tools/gemv_bench.py A/B; 0 = the default) */
int mspq_debug_gemv_variant(int v);
/* the same over a batch of several request streams' windows: meta[T][3] = per token (batch row of
 * its window's first token, stream index, position); stream s's cache = kc + s * kv_stream_stride */
int mspq_attention_batched(const float* qkv, int splits, long long split_stride, int T, int H, int Hkv, int Dh, int P,
                           const int32_t* meta, long long kv_stream_stride, void* kc, void* vc, void* out, void* oimg,
                           void* ws, void* stream);
/* row-major quantised INT4 (q[rows][cols/8] u32, standard nibble order; s[rows][cols/128] bf16)
 * -> tile-major [rows/128][cols/64][128][8] u32 + [rows/128][cols/128][128] bf16 */
int mspq_tile_int4(const void* q, const void* s, int rows, int cols, void* tq, void* ts, void* stream);
/* diagnostics: per-role clock64 stamps (2048 slots) of the first CTA of the first K2 launch after
 * a call with n < 0 (arms the recorder); n > 0 copies the stamps out */
int mspq_debug_timeline(long long* dst, int n);
/* row-major [rows][cols] bf16 -> tile-major [rows/128][cols/64] SW128 images (16 KB each) */
int mspq_tile_bf16(const void* src, int rows, int cols, void* dst, void* stream);
int mspq_lm_head(const void* xn, const void* lm, int T, int V, int d, float* logits,
                 void* stream);
int mspq_argmax(const float* logits, int T, int V, int32_t* out, void* stream);
/* K5: res[0] = accepted, res[1] = bonus token */
int mspq_accept_scan(const int32_t* draft, const int32_t* target_argmax, int k, int32_t* res,
                     void* stream);
/* draft-loop variants that keep the decode state on the device (graph-replayable):
 * argmax_advance: draft_toks[*row] = tok; *cur_tok = tok; *cur_pos += 1; *row += 1.
 * accept_advance: K5 + next head: *cur_tok = bonus, *cur_pos = head_pos + accepted + 1. */
int mspq_argmax_advance(const float* logits, int V, int32_t* out, int32_t* row,
                        int32_t* draft_toks, int32_t* cur_tok, int32_t* cur_pos, void* stream);
int mspq_accept_advance(const int32_t* draft, const int32_t* target_argmax, int k, int32_t* res,
                        int32_t* cur_tok, int32_t* cur_pos, int head_pos, void* stream);
/* Lossless expert codec (csrc/xcodec.cu): bf16 16 KB tile images <-> one blob of
 * raw sign/mantissa bytes + per-tile Huffman-coded exponents.  The host store keeps experts in
 * this form so the PCIe copy engines move ~2/3 of the bf16 bytes; decode restores the exact
 * images in the HBM slot.  encode blocks on the stream (it builds the code on the host);
 * tiles/scratch/out must be 256-byte aligned device buffers. */
long long mspq_xc_max_blob_bytes(long long n_tiles);
long long mspq_xc_scratch_bytes(long long n_tiles);
int mspq_xc_encode(const void* tiles, long long n_tiles, void* scratch, void* out, long long out_cap,
                   long long* out_bytes, void* stream);
/* decode tiles [tile0, tile1) of a device blob into dst (tile t -> dst + 16 KB * t); n_ctas <= 0
 * picks the default grid (32 CTAs of 8 warps) */
int mspq_xc_decode(const void* blob, int tile0, int tile1, void* dst, int n_ctas, void* stream);
long long mspq_int4_blob_bytes(int d, int f);
long long mspq_bf16_blob_bytes(int d, int f);


/* ---------------------------------------------------------------- K4 expert-cache controller
 * Device-resident cache table (key -> HBM buffer, LRU stamps, per-layer sizes), ELB, planner
 * state and copy-request queue; all decisions are made by kernels (one warp per launch).
 * Restates CacheState / plan_prefetch / select_victim_lookahead / policy_step
 * (scheduler.cpp:76-312) and the cycle's insertion rules (sim.cpp:152-295). */
typedef struct mspq_cache mspq_cache;
typedef struct mspq_cache_view {  /* device pointers owned by the cache */
  int32_t* elb_ids;   /* [kmax][L][K] */
  float* elb_gates;   /* [kmax][L][K] */
  int32_t* scal;      /* scalar slots (see ctl.h CtlScalar) */
  int32_t* req;       /* device alias of host_req */
  int32_t* log;       /* [log_cap][6] (kind, tag, key, hit, victim, buffer) */
  int32_t* plan;      /* [plan_cap][3] (row, key, phase) */
  int32_t* cov;       /* [L][2] */
  int32_t* step;      /* [L][kmax+1][2] */
  int32_t* res;       /* [L*E] key -> buffer */
  int32_t* host_stat; /* HOST pointer: mapped mirror of scal, valid after the launch completes */
  int32_t* host_req;  /* HOST pointer: mapped copy requests of the last launch */
  int32_t* host_sched;/* HOST pointer: [0] n_groups, [1..] group_buf of the last verify step */
  int req_cap, log_cap, plan_cap, nbuf;
} mspq_cache_view;
int mspq_cache_create(int L, int E, int K, int kmax, int nbuf, int log_cap, mspq_cache** out);
int mspq_cache_destroy(mspq_cache* c);
/* mode 0 per-layer / 1 global; policy = moespeq::Policy ordinal; caps[L] (per-layer) */
int mspq_cache_configure(mspq_cache* c, int mode, int policy, const int* caps, int cap_global,
                         int budget, double f1, double f2, void* stream);
int mspq_cache_view_get(mspq_cache* c, mspq_cache_view* v);
/* 1 (default when the state fits) = each launch runs on a shared-memory copy of the table;
 * 0 = operate on global memory directly.  Decisions are identical (tested). */
int mspq_cache_set_staging(mspq_cache* c, int on);
int mspq_cache_begin_cycle(mspq_cache* c, int k, void* stream);
int mspq_cache_plan_row(mspq_cache* c, int row, void* stream);
/* verify step of one layer: policy steps for every (slot, expert) of tgt[nslots][K]; writes
 * gbuf[E] = HBM buffer each required expert is read from (-2 = not required) */
int mspq_cache_verify_layer(mspq_cache* c, int layer, int nslots, const int32_t* tgt,
                            int32_t* gbuf, void* stream);
/* token-major replay of one cycle over device trace arrays (target/draft [n][L][K] int32,
 * gates [n][L][K] double or NULL).  out_*: counts[6], batches[kmax][3], jit_rows[kmax][2],
 * cov[L][2], step[(kmax+1)*L][2], flush_keys[L*E] */
int mspq_cache_replay_cycle(mspq_cache* c, const int32_t* target, const int32_t* draft,
                            const double* gates, int pos, int k_eff, int head_pos,
                            int32_t* out_counts, int32_t* out_batches, int32_t* out_jit_rows,
                            int32_t* out_cov, int32_t* out_step, int32_t* out_flush_keys,
                            void* stream);

/* the whole trace in ONE launch: the Amortization-Roofline governor runs on the device between
 * cycles (same double arithmetic as mspq_governor), cycle ci writes its ReplayOut block to
 * slices + ci * stride at offsets {batches, jit_rows, cov, step} (counts at 0) and k_eff[ci].
 * acc[n] = the trace's acc flags; gov_ints = {use_governor, fixed_k, k_min, k_max, k_slo, kcap};
 * gov_reals = {ema_alpha, initial_accept, pcie_bw, pcie_init, pcie_overhead, expert_bytes,
 * draft_base, draft_per_token}; vs_xy = nvs verify samples (window, seconds). */
int mspq_cache_replay_all(mspq_cache* c, const int32_t* target, const int32_t* draft, const double* gates,
                          const unsigned char* acc, int n, const int32_t* gov_ints, const double* gov_reals,
                          int nvs, const double* vs_xy, int32_t* slices, int stride, const int32_t* offsets,
                          int32_t* k_eff, int32_t* n_cycles, int32_t* flush_keys, void* stream);

/* ---------------------------------------------------------------- (2) engine */
/* run_simulation on the device control plane: trace = reference JSONL (trace.hpp:76-80),
 * config = reference run-config JSON (run_config.hpp:30-50).  *report_json: SimReport JSON;
 * with "log": true in config_json also the per-event hit/miss log. */
int mspq_replay(int device, const char* trace_jsonl, const char* config_json,
                char** report_json);
/* compare_policies / sweep_k (sim.cpp:539-574, sim.hpp:88-109) over mspq_replay:
 * rows [{"policy","capacity","coverage","tpot"}] / [{"k","tpot","mean_accepted","coverage","ttft"}] */
int mspq_compare_policies(int device, const char* trace_jsonl, const char* config_json,
                          const char* policies_json, const char* capacities_json, char** rows_json);
int mspq_sweep_k(int device, const char* trace_jsonl, const char* config_json, const char* ks_json,
                 char** rows_json);
/* Amortization-Roofline governor (perfmodel.cpp:85-217) on a JSON request:
 * {"profile":{...},"p":[...],"alpha":a,"k_min","k_max","k_slo","g","ttft_budget","outcomes"}
 * -> {"select_k","k_slo_ttft","t_cycle":[k=0..],"k_accept":[..],"t_verify":[..],"updated_p"} */
int mspq_governor(const char* request_json, char** out_json);

int mspq_engine_create(const mspq_model_desc* model, const mspq_engine_opts* opts,
                       mspq_engine** out);
int mspq_engine_destroy(mspq_engine* eng);
/* expert-cache budget / policy / governor in the reference run-config schema; resets the cache */
int mspq_engine_configure(mspq_engine* eng, const char* config_json);
/* greedy speculative decode of max_new tokens after the prompt (last prompt token is the
 * first window head).  *report_json: SimReport JSON + measured fields + per-cycle traces. */
int mspq_generate(mspq_engine* eng, const int32_t* prompt, int n_prompt, int max_new,
                  char** report_json);
/* several independent request streams decoded together: each stream has its own prompt, KV cache
 * and draft; every cycle the streams' verify windows go through ONE layer-major verify pass (one
 * grouped GEMM per layer over all streams' tokens, so they share the expert weight reads) over one
 * shared expert cache.  prompts: n_streams prompts back to back, lens[n_streams]; all streams share
 * k (k+1 slots each, n_streams (k+1) <= 32).  Cache policy must be "lru" (the ELB-driven policies
 * are defined for one stream's lookahead).  *report_json: per-stream tokens + per-cycle records. */
int mspq_generate_batch(mspq_engine* eng, const int32_t* prompts, const int32_t* lens, int n_streams,
                        int max_new, char** report_json);
int mspq_engine_info(mspq_engine* eng, char** json);
/* copy a device tensor of the engine out (tests): name in {"embed","pos","lm","router:<l>",
 * "gamma:<l>","gamma:final","draft:<l>:<e>","expert:<l>:<e>" (bf16 tile images, decoded if the
 * store is coded), "expert_blob:<l>:<e>" (the stored bytes as they cross PCIe), "kcache:<l>" /
 * "vcache:<l>" ([P][Hkv][Dh] bf16), "wqkv:<l>" / "wo:<l>" (tile images), "gamma_attn:<l>",
 * trace_level 3 residual captures of the last generate(): "hcap_v:<cycle>" [L+1][T][d],
 * "hcap_d:<cycle>" [k][L+1][d] (entering each layer; index L = final) and, with attention,
 * "hmid_v:<cycle>" [L][T][d] / "hmid_d:<cycle>" [k][L][d] (after the attention residual)} */
int mspq_engine_read(mspq_engine* eng, const char* name, void* host_dst, long long bytes);

/* ---------------------------------------------------------------- (3) peer-expert tier
 * NVLink peer-expert tier (BASELINE.json north_star) with "home"
 * partitioning: in a group of G engines (one per GPU), engine r keeps the bf16 tile images of
 * every expert (l, e) with e % G == r permanently in an HBM home region (filled once from the
 * host store).  A cache miss (demand or prefetch) of an expert homed on an attached peer is
 * copied HBM -> HBM from the peer's home region (copy engine over NVLink / NVSwitch; a local
 * home is a device-to-device copy) instead of over PCIe.  Home regions are immutable after the
 * fill, so peers read them with no coordination.  Cache decisions are unchanged: only the bytes'
 * source moves (the replaced path: the synchronous fetch sim.cpp:338-344, t_pcie_new
 * perfmodel.cpp:104-110).  Experts homed on a peer that is not attached keep the PCIe path.
 *
 * mspq_engine_home_create: allocate + fill this engine's home region; *ipc_handle (64 bytes,
 *   cudaIpcMemHandle_t) lets other processes map it.
 * mspq_engine_peer_attach_ipc: map peer `peer_rank`'s home region from its handle (another
 *   process; same or another GPU, cudaIpcOpenMemHandle with lazy peer access).
 * mspq_engine_peer_attach: the same for a peer engine in this process. */
int mspq_engine_home_create(mspq_engine* eng, int group_size, int rank, void* ipc_handle_out);
int mspq_engine_peer_attach_ipc(mspq_engine* eng, int peer_rank, const void* ipc_handle);
int mspq_engine_peer_attach(mspq_engine* eng, int peer_rank, mspq_engine* peer);

#ifdef __cplusplus
}
#endif
#endif
