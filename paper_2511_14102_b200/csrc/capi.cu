// extern "C" kernel entry points of libmspq.so (include/mspq_capi.h, part 1 + K4).
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/mspq_capi.h"
#include "ctl.h"
#include "kernels.h"
#include "status.h"

static int tc_bn(int T) { return T <= 16 ? 16 : 32; }

using namespace mspq;

namespace mspq {
thread_local std::string g_last_error;
int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return MSPQ_OK;
  return set_error(MSPQ_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
}  // namespace mspq

#define ST(s) reinterpret_cast<cudaStream_t>(s)
#define CK(expr, where) return cuda_status((expr), where)

extern "C" {

const char* mspq_status_string(int s) {
  static const char* names[] = {"OK", "MalformedRecord", "ShapeViolation", "EmptyTrace",
                                "InvalidFidelity", "DegenerateShape", "LayerOutOfRange",
                                "ShapeMismatch", "RangeOutOfBounds", "EmptyCache", "UnknownPolicy",
                                "EmptyRequired", "IncompleteRouting", "KOutOfRange",
                                "InsufficientSamples", "EmptyRange", "InfeasibleBudget",
                                "InvalidConfig", "IoError"};
  if (s >= 0 && s <= 18) return names[s];
  if (s == MSPQ_ERR_CUDA) return "CudaError";
  if (s == MSPQ_ERR_OVERFLOW) return "Overflow";
  return "Internal";
}
const char* mspq_last_error(void) { return g_last_error.c_str(); }
void mspq_free(void* p) { free(p); }
int mspq_version(void) { return 1; }

long long mspq_int4_blob_bytes(int d, int f) {
  return (long long)2 * f * d / 2 + (long long)2 * f * (d / 128) * 2 + (long long)d * f / 2 +
         (long long)d * (f / 128) * 2;
}
long long mspq_bf16_blob_bytes(int d, int f) { return (long long)3 * d * f * 2; }

int mspq_fill_bf16(unsigned long long seed, unsigned long long tensor, float scale, int kind,
                   void* out, long long n, long long start, void* stream) {
  CK(launch_fill_bf16(seed, tensor, scale, kind, (uint16_t*)out, n, start, ST(stream)), "fill_bf16");
}
int mspq_fill_expert(unsigned long long seed, int l, int e, int d, int f, float a_up, float a_down,
                     void* blob, void* stream) {
  CK(launch_fill_expert(seed, l, e, d, f, a_up, a_down, (uint16_t*)blob, ST(stream)), "fill_expert");
}
int mspq_quantize_int4(const void* w, int rows, int cols, void* q, void* s, void* stream) {
  if (cols % 128) return set_error(MSPQ_ERR_SHAPE_MISMATCH, "quantize: cols % 128 != 0");
  CK(launch_quantize((const uint16_t*)w, rows, cols, (uint32_t*)q, (uint16_t*)s, ST(stream)), "quantize");
}
int mspq_embed(const void* embed, const void* pos, const int32_t* tokens, const int32_t* positions,
               int T, int d, float* h, void* stream) {
  CK(launch_embed((const uint16_t*)embed, (const uint16_t*)pos, tokens, positions, T, d, h, ST(stream)),
     "embed");
}
int mspq_gate_topk_img(float* h, const float* y, const int32_t* entry_of, const float* prev_wts,
                       int y_splits, long long y_split_stride, const void* gamma, const void* router, void* xn,
                       int32_t* ids, float* wts, float* logits, int32_t* elb_ids, float* elb_gates,
                       const int32_t* elb_row, int32_t* sched_block, int layer, int L, int T, int d, int E, int K,
                       float eps, void* bimg, void* stream) {
  if (d % 256 || K > 64 || E > 1024 || K > E || (bimg && T > 32))
    return set_error(MSPQ_ERR_SHAPE_MISMATCH, "gate_topk: need d%256==0, K<=min(E,64), E<=1024 (image: T<=32)");
  RouteArgs a{h, y, entry_of, prev_wts, (const uint16_t*)gamma, (const uint16_t*)router,
              (uint16_t*)xn, ids, wts, logits, y_splits < 1 ? 1 : y_splits, y_split_stride,
              elb_ids, elb_gates, elb_row, T == 1 ? sched_block : nullptr, layer, L, d, E, K, eps,
              (unsigned char*)bimg, tc_bn(T)};
  CK(launch_route(a, T, ST(stream)), "gate_topk");
}
int mspq_gate_topk(float* h, const float* y, const int32_t* entry_of, const float* prev_wts,
                   int y_splits, long long y_split_stride, const void* gamma, const void* router, void* xn, int32_t* ids, float* wts,
                   float* logits, int32_t* elb_ids, float* elb_gates, const int32_t* elb_row,
                   int32_t* sched_block, int layer, int L, int T, int d, int E, int K, float eps,
                   void* stream) {
  return mspq_gate_topk_img(h, y, entry_of, prev_wts, y_splits, y_split_stride, gamma, router, xn, ids, wts, logits,
                            elb_ids, elb_gates, elb_row, sched_block, layer, L, T, d, E, K, eps, nullptr, stream);
}
int mspq_build_schedule(const int32_t* ids, int T, int K, int E, const int32_t* gbuf, int32_t* n_groups,
                        int32_t* group_expert, int32_t* group_buf, int32_t* group_off,
                        int32_t* entry_tok, int32_t* entry_of, int32_t* entry_group, void* stream) {
  if (E > 1024 || T * K > 4096) return set_error(MSPQ_ERR_SHAPE_MISMATCH, "build_schedule: E<=1024, T*K<=4096");
  SchedPtrs s{n_groups, group_expert, group_buf, group_off, entry_tok, entry_of, entry_group};
  CK(launch_build_schedule(ids, T, K, E, gbuf, s, ST(stream)), "build_schedule");
}
long long mspq_moe_bf16_tc_ws_bytes(int d, int f, int T, int K, int max_groups, int max_split1) {
  const long long BN = tc_bn(T), N = (long long)T * K;
  auto al = [](long long b) { return (b + 1023) / 1024 * 1024; };
  return al(max_groups * (d / 64) * BN * 128) + al((long long)max_split1 * N * 2 * f * 4) +
         al(max_groups * (f / 64) * BN * 128) + al(max_groups * BN * (d / 64) * 4) +
         al(max_groups * BN * (f / 64) * 4);
}
int mspq_moe_bf16_tc_part(const int32_t* n_groups, const int32_t* group_expert, const int32_t* group_buf,
                          const int32_t* group_off, const int32_t* entry_tok, const int32_t* entry_group,
                          const void* xn, const void* pool, long long blob_bytes, int d, int f, int T, int K,
                          int max_groups, int split1, int split2, void* ws, float* y, const uint32_t* gmask8,
                          int do_gather, void* stream) {
  if (d % 128 || f % 256 || T > 32 || split1 < 1 || split2 < 1)
    return set_error(MSPQ_ERR_SHAPE_MISMATCH, "moe_bf16_tc: d % 128, f % 256, T <= 32, splits >= 1");
  if (gmask8 && max_groups > 256) return set_error(MSPQ_ERR_SHAPE_MISMATCH, "moe_bf16_tc_part: <= 256 groups");
  const int BN = tc_bn(T);
  const long long N = (long long)T * K;
  auto al = [](long long b) { return (b + 1023) / 1024 * 1024; };
  unsigned char* b1 = (unsigned char*)ws;
  float* p1 = (float*)(b1 + al(max_groups * (d / 64) * BN * 128));
  unsigned char* b2 = (unsigned char*)p1 + al((long long)split1 * N * 2 * f * 4);
  SchedPtrs s{(int32_t*)n_groups, (int32_t*)group_expert, (int32_t*)group_buf, (int32_t*)group_off,
              (int32_t*)entry_tok, nullptr, (int32_t*)entry_group};
  GMask gm{};
  if (gmask8) {
    for (int i = 0; i < 8; ++i) gm.w[i] = gmask8[i];
    gm.on = 1;
  }
  cudaStream_t st = ST(stream);
  cudaError_t e = cudaSuccess;
  if (do_gather) {
    e = launch_gather_b((const uint16_t*)xn, d, s, max_groups, d, BN, b1, st);
    if (e != cudaSuccess) return cuda_status(e, "gather_b");
  }
  UmmaArgs u1{(const unsigned char*)pool, blob_bytes, 0, 2 * f, d, n_groups, group_buf, group_off, b1, p1,
              N * 2 * f, split1};
  u1.gmask = gm;
  u1.early_a = do_gather;  // the gather sits between the schedule's writer and W13 (UmmaArgs::early_a)
  if (split1 == 1) u1.act_img = b2;  // SiLU*up in the W13 epilogue, no finalize kernel
  e = launch_umma_grouped(u1, max_groups, BN, st);
  if (e != cudaSuccess) return cuda_status(e, "umma W13");
  if (split1 > 1) {
    e = launch_finalize_act(p1, split1, N * 2 * f, s, entry_group, (int)N, f, BN, b2, st, nullptr, gm);
    if (e != cudaSuccess) return cuda_status(e, "finalize_act");
  }
  UmmaArgs u2{(const unsigned char*)pool, blob_bytes, (long long)2 * f * d * 2, d, f, n_groups, group_buf,
              group_off, b2, y, N * d, split2};
  u2.gmask = gm;
  u2.early_a = 1;  // W13 (whose own wait ordered it after the schedule) precedes W2
  CK(launch_umma_grouped(u2, max_groups, BN, st), "umma W2");
}
int mspq_moe_bf16_tc(const int32_t* n_groups, const int32_t* group_expert, const int32_t* group_buf,
                     const int32_t* group_off, const int32_t* entry_tok, const int32_t* entry_group,
                     const void* xn, const void* pool, long long blob_bytes, int d, int f, int T, int K,
                     int max_groups, int split1, int split2, void* ws, float* y, void* stream) {
  return mspq_moe_bf16_tc_part(n_groups, group_expert, group_buf, group_off, entry_tok, entry_group, xn, pool,
                               blob_bytes, d, f, T, K, max_groups, split1, split2, ws, y, nullptr, 1, stream);
}
// dense projection = K3 with one group holding all T tokens; dsched packed per T:
// [n_groups = 1, group_buf = 0, group_off = {0, T}, entry_tok = 0..T-1]
long long mspq_dense_ws_bytes(int kdim, int T) { return (long long)(kdim / 64) * tc_bn(T) * 128 + 1024; }
int mspq_dense_sched_fill(int32_t* host_packed, int T) {
  host_packed[0] = 1;
  host_packed[1] = 0;
  host_packed[2] = 0;
  host_packed[3] = T;
  for (int t = 0; t < T; ++t) host_packed[4 + t] = t;
  return MSPQ_OK;
}
int mspq_dense_bf16_tc(const int32_t* dsched, const void* x, const void* w_tiled, int rows, int kdim, int T,
                       int split, void* ws, float* out, long long out_split_stride, void* stream) {
  if (rows % 128 || kdim % 64 || T < 1 || T > 32 || split < 1 || split > kdim / 64)
    return set_error(MSPQ_ERR_SHAPE_MISMATCH, "dense_bf16_tc: rows % 128, kdim % 64, 1 <= T <= 32, 1 <= split <= kdim/64");
  const int BN = tc_bn(T);
  int32_t* p = (int32_t*)dsched;
  SchedPtrs s{p, nullptr, p + 1, p + 2, p + 4, nullptr, nullptr};
  cudaStream_t st = ST(stream);
  unsigned char* b1 = (unsigned char*)ws;
  if (x) {  // x == NULL: the producer already wrote the B image into ws (K1 / attention epilogue)
    cudaError_t e = launch_gather_b((const uint16_t*)x, kdim, s, 1, kdim, BN, b1, st);
    if (e != cudaSuccess) return cuda_status(e, "dense gather");
  }
  UmmaArgs u{(const unsigned char*)w_tiled, 0, 0, rows, kdim, p, p + 1, p + 2, b1, out, out_split_stride, split};
  u.early_a = 1;  // weights and dsched are static: the A stream starts under the predecessor's tail
  CK(launch_umma_grouped(u, 1, BN, st), "dense umma");
}
long long mspq_attention_ws_bytes(int T, int H, int Hkv, int Dh) {
  return (long long)attn_part_floats(T, H, Hkv, Dh) * 4;
}
int mspq_attention_batched(const float* qkv, int splits, long long split_stride, int T, int H, int Hkv, int Dh, int P,
                           const int32_t* meta, long long kv_stream_stride, void* kc, void* vc, void* out, void* oimg,
                           void* ws, void* stream) {
  if (H < 1 || Hkv < 1 || H % Hkv || H / Hkv > 8 || (Dh != 64 && Dh != 128) || T < 1 || P > 4096 || !ws || !meta ||
      T * Hkv > AT_CNT)
    return set_error(MSPQ_ERR_SHAPE_MISMATCH,
                     "attention_batched: Hkv | H, H/Hkv <= 8, Dh in {64, 128}, P <= 4096, T * Hkv <= 2048");
  AttnArgs a{qkv, splits, split_stride, T, H, Hkv, Dh, P, nullptr, (uint16_t*)kc, (uint16_t*)vc, (uint16_t*)out,
             1.0f / sqrtf((float)Dh), (unsigned char*)oimg, tc_bn(T), (float*)ws, meta, kv_stream_stride};
  CK(launch_attn_window(a, ST(stream)), "attention_batched");
}
int mspq_attention(const float* qkv, int splits, long long split_stride, int T, int H, int Hkv, int Dh, int P,
                   const int32_t* pos0, void* kc, void* vc, void* out, void* oimg, void* ws, void* stream) {
  if (H < 1 || Hkv < 1 || H % Hkv || H / Hkv > 8 || (Dh != 64 && Dh != 128) || T < 1 || P < T || P > 4096 || !ws ||
      T * Hkv > AT_CNT)
    return set_error(MSPQ_ERR_SHAPE_MISMATCH,
                     "attention: Hkv | H, H/Hkv <= 8, Dh in {64, 128}, 1 <= T <= P <= 4096, T * Hkv <= 2048, workspace");
  AttnArgs a{qkv, splits, split_stride, T, H, Hkv, Dh, P, pos0, (uint16_t*)kc, (uint16_t*)vc, (uint16_t*)out,
             1.0f / sqrtf((float)Dh), (unsigned char*)oimg, tc_bn(T), (float*)ws};
  CK(launch_attn_window(a, ST(stream)), "attention");
}
int mspq_debug_gemv_variant(int v) {
  gemv_set_variant(v);
  return MSPQ_OK;
}
int mspq_fragtile_int4(const void* q, int rows, int cols, void* fq, void* stream) {
  if (rows % 32 || cols % 128) return set_error(MSPQ_ERR_SHAPE_MISMATCH, "fragtile_int4: rows % 32, cols % 128");
  CK(launch_fragtile_int4((const uint32_t*)q, rows, cols, (uint32_t*)fq, ST(stream)), "fragtile_int4");
}
int mspq_moe_int4_gemv(const int32_t* n_groups, const int32_t* group_expert, const void* xn, const void* blobs,
                       long long blob_bytes, int layer, int E, int d, int f, int K, int split2, void* act, float* y,
                       void* stream) {
  if (d % 128 || f % 128 || K < 1 || split2 < 1 || split2 > f / 128)
    return set_error(MSPQ_ERR_SHAPE_MISMATCH, "moe_int4_gemv: d, f multiples of 128, 1 <= split2 <= f/128");
  const long long q13 = (long long)2 * f * d / 2, s13 = (long long)2 * f * (d / 128) * 2, q2 = (long long)d * f / 2;
  cudaStream_t st = ST(stream);
  GemvArgs g1{(const unsigned char*)blobs, blob_bytes, 0, q13, 2 * f, d, layer, E, n_groups, group_expert,
              (const uint16_t*)xn, 0, nullptr, (uint16_t*)act};
  cudaError_t e = launch_int4_gemv(g1, K, 1, st);
  if (e != cudaSuccess) return cuda_status(e, "int4 gemv W13");
  GemvArgs g2{(const unsigned char*)blobs, blob_bytes, q13 + s13, q13 + s13 + q2, d, f, layer, E, n_groups,
              group_expert, (const uint16_t*)act, 1, y, nullptr};
  CK(launch_int4_gemv(g2, K, split2, st), "int4 gemv W2");
}
int mspq_moe_int4_tc(const int32_t* n_groups, const int32_t* group_expert, const int32_t* group_buf,
                     const int32_t* group_off, const int32_t* entry_tok, const int32_t* entry_group,
                     const void* xn, const void* blobs, long long blob_bytes, int layer, int E, int d, int f, int T,
                     int K, int max_groups, int split1, int split2, void* ws, float* y, void* stream) {
  if (d % 128 || f % 256 || T > 32 || split1 < 1 || split2 < 1)
    return set_error(MSPQ_ERR_SHAPE_MISMATCH, "moe_int4_tc: d % 128, f % 256, T <= 32, splits >= 1");
  const int BN = tc_bn(T);
  const int IR = (BN == 16 && T <= 8) ? 8 : BN;  // B image rows (8: aliased 8-row token tiles)
  const long long N = (long long)T * K;
  auto al = [](long long b) { return (b + 1023) / 1024 * 1024; };
  unsigned char* b1 = (unsigned char*)ws;
  float* p1 = (float*)(b1 + al(max_groups * (d / 64) * BN * 128));
  unsigned char* b2 = (unsigned char*)p1 + al((long long)split1 * N * 2 * f * 4);
  float* c1 = (float*)(b2 + al(max_groups * (f / 64) * BN * 128));  // [G][IR][d/64]
  float* c2 = c1 + al(max_groups * BN * (d / 64) * 4) / 4;            // [G][IR][f/64]
  SchedPtrs s{(int32_t*)n_groups, (int32_t*)group_expert, (int32_t*)group_buf, (int32_t*)group_off,
              (int32_t*)entry_tok, nullptr, (int32_t*)entry_group};
  cudaStream_t st = ST(stream);
  const long long q13 = (long long)2 * f * d / 2, s13 = (long long)2 * f * (d / 128) * 2, q2 = (long long)d * f / 2;
  if (T == 1 && IR == 8 && split1 == 1) {
    // draft shape: both GEMMs build their token tiles from the bf16 rows themselves and W13's
    // epilogue applies SiLU*up (no gather / finalize kernels, no fp32 W13 plane)
    uint16_t* act = (uint16_t*)b2;  // [N][f] bf16
    UmmaArgs u1{(const unsigned char*)blobs, blob_bytes, 0, 2 * f, d, n_groups, group_buf, group_off, nullptr, p1,
                N * 2 * f, 1, q13, layer * E, IR, nullptr, (const uint16_t*)xn, 0, entry_tok, act};
    cudaError_t e = launch_umma_int4p(u1, max_groups, st);
    if (e != cudaSuccess) return cuda_status(e, "umma_int4 W13 (fused act)");
    UmmaArgs u2{(const unsigned char*)blobs, blob_bytes, q13 + s13, d, f, n_groups, group_buf, group_off, nullptr, y,
                N * d, split2, q13 + s13 + q2, layer * E, IR, nullptr, act, 1, entry_tok, nullptr};
    CK(launch_umma_int4p(u2, max_groups, st), "umma_int4 W2 (self-gather)");
  }
  cudaError_t e = launch_gather_b((const uint16_t*)xn, d, s, max_groups, d, IR, b1, st, c1);
  if (e != cudaSuccess) return cuda_status(e, "gather_b");
  UmmaArgs u1{(const unsigned char*)blobs, blob_bytes, 0, 2 * f, d, n_groups, group_buf, group_off, b1, p1,
              N * 2 * f, split1, q13, layer * E, IR, c1};
  e = launch_umma_int4(u1, max_groups, BN, st);
  if (e != cudaSuccess) return cuda_status(e, "umma_int4 W13");
  e = launch_finalize_act(p1, split1, N * 2 * f, s, entry_group, (int)N, f, IR, b2, st, c2);
  if (e != cudaSuccess) return cuda_status(e, "finalize_act");
  UmmaArgs u2{(const unsigned char*)blobs, blob_bytes, q13 + s13, d, f, n_groups, group_buf, group_off, b2, y,
              N * d, split2, q13 + s13 + q2, layer * E, IR, c2};
  CK(launch_umma_int4(u2, max_groups, BN, st), "umma_int4 W2");
}
int mspq_tile_int4(const void* q, const void* s, int rows, int cols, void* tq, void* ts, void* stream) {
  if (rows % 128 || cols % 128) return set_error(MSPQ_ERR_SHAPE_MISMATCH, "tile_int4: rows%128, cols%128");
  CK(launch_tile_int4((const uint32_t*)q, (const uint16_t*)s, rows, cols, (uint32_t*)tq, (uint16_t*)ts, ST(stream)),
     "tile_int4");
}
int mspq_debug_timeline(long long* dst, int n) { CK(debug_int4_timeline(dst, n), "debug_timeline"); }
int mspq_tile_bf16(const void* src, int rows, int cols, void* dst, void* stream) {
  if (rows % 128 || cols % 64) return set_error(MSPQ_ERR_SHAPE_MISMATCH, "tile_bf16: rows%128, cols%64");
  CK(launch_tile_bf16((const uint16_t*)src, rows, cols, (unsigned char*)dst, ST(stream)), "tile_bf16");
}
int mspq_lm_head(const void* xn, const void* lm, int T, int V, int d, float* logits, void* stream) {
  CK(launch_lm_head((const uint16_t*)xn, (const uint16_t*)lm, T, V, d, logits, ST(stream)), "lm_head");
}
int mspq_argmax(const float* logits, int T, int V, int32_t* out, void* stream) {
  DraftState ds{nullptr, nullptr, nullptr, nullptr};
  CK(launch_argmax(logits, T, V, out, ds, ST(stream)), "argmax");
}
int mspq_accept_scan(const int32_t* draft, const int32_t* tgt, int k, int32_t* res, void* stream) {
  CK(launch_accept(draft, tgt, k, res, nullptr, nullptr, 0, ST(stream)), "accept_scan");
}

int mspq_argmax_advance(const float* logits, int V, int32_t* out, int32_t* row,
                        int32_t* draft_toks, int32_t* cur_tok, int32_t* cur_pos, void* stream) {
  DraftState ds{row, draft_toks, cur_tok, cur_pos};
  CK(launch_argmax(logits, 1, V, out, ds, ST(stream)), "argmax_advance");
}
int mspq_accept_advance(const int32_t* draft, const int32_t* tgt, int k, int32_t* res,
                        int32_t* cur_tok, int32_t* cur_pos, int head_pos, void* stream) {
  CK(launch_accept(draft, tgt, k, res, cur_tok, cur_pos, head_pos, ST(stream)), "accept_advance");
}

// ------------------------------------------------------------------ K4
struct mspq_cache {
  CtlDev C;
  int kmax, nbuf;
  void* blk;
  void* hblk;  // mapped pinned: [0,256) status mirror, then requests
};

int mspq_cache_create(int L, int E, int K, int kmax, int nbuf, int log_cap, mspq_cache** out) {
  // K <= 64: the controller's per-step key scratch (ctl.cu sorted_keys) and gate_topk's limit
  if (L < 1 || E < 1 || K < 1 || K > E || K > 64 || L * E > 8192 || E > 1024)
    return set_error(MSPQ_ERR_SHAPE_VIOLATION, "cache: need 1<=K<=min(E,64), E<=1024, L*E<=8192");
  mspq_cache* c = new mspq_cache();
  c->kmax = kmax;
  c->nbuf = nbuf;
  CtlDev& C = c->C;
  C.L = L;
  C.E = E;
  C.K = K;
  C.nbuf = nbuf;
  C.kmax = kmax;
  const int n = L * E;
  C.req_cap = 4 * n + 64;
  C.log_cap = log_cap > 0 ? log_cap : (kmax + 1) * L * K * 4 + 4 * n + 64;
  C.plan_cap = n + 64;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  size_t o_cap = take(L * 4), o_res = take(n * 4), o_stamp = take(n * 8), o_clock = take(8),
         o_lsize = take(L * 4), o_scal = take(S_COUNT * 4), o_free = take(nbuf * 4 + 4),
         o_pend = take(nbuf * 4 + 4), o_snap = take(n), o_sched = take(n), o_cf = take(n * 4),
         o_cc = take(n * 8), o_eids = take((size_t)kmax * L * K * 4),
         o_eg = take((size_t)kmax * L * K * 4),
         o_log = take((size_t)C.log_cap * 24), o_plan = take((size_t)C.plan_cap * 12),
         o_reqd = take((size_t)C.req_cap * 12),
         o_cov = take(L * 8), o_step = take((size_t)L * (kmax + 1) * 8);
  cudaError_t e = cudaMalloc(&c->blk, off);
  if (e != cudaSuccess) {
    delete c;
    return cuda_status(e, "cache_create");
  }
  // copy requests + status are written by the controller straight into mapped pinned memory
  const size_t hbytes = 256 + (size_t)(E + 8) * 4 + (size_t)C.req_cap * 12;
  e = cudaHostAlloc(&c->hblk, hbytes, cudaHostAllocMapped);
  if (e != cudaSuccess) {
    cudaFree(c->blk);
    delete c;
    return cuda_status(e, "cache_create(host)");
  }
  memset(c->hblk, 0, hbytes);
  void* dptr = nullptr;
  cudaHostGetDevicePointer(&dptr, c->hblk, 0);
  // the block is zeroed synchronously: callers drive the cache on their own (possibly
  // non-blocking) streams, which do not order against the legacy stream
  e = cudaMemset(c->blk, 0, off);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    cudaFree(c->blk);
    cudaFreeHost(c->hblk);
    delete c;
    return cuda_status(e, "cache_create(zero)");
  }
  char* b = (char*)c->blk;
  C.cap = (int*)(b + o_cap);
  C.res = (int*)(b + o_res);
  C.stamp = (unsigned long long*)(b + o_stamp);
  C.clock = (unsigned long long*)(b + o_clock);
  C.lsize = (int*)(b + o_lsize);
  C.scal = (int*)(b + o_scal);
  C.free_stack = (int*)(b + o_free);
  C.pending = (int*)(b + o_pend);
  C.snap = (unsigned char*)(b + o_snap);
  C.sched = (unsigned char*)(b + o_sched);
  C.cand_first = (int*)(b + o_cf);
  C.cand_conf = (double*)(b + o_cc);
  C.elb_ids = (int32_t*)(b + o_eids);
  C.elb_gates = (float*)(b + o_eg);
  C.hstat = (int*)dptr;
  C.hsched = (int*)((char*)dptr + 256);
  C.req = (int*)((char*)dptr + 256 + (size_t)(E + 8) * 4);
  C.log = (int*)(b + o_log);
  C.req_dev = (int*)(b + o_reqd);
  C.plan = (int*)(b + o_plan);
  C.cov = (int*)(b + o_cov);
  C.step = (int*)(b + o_step);
  C.stage = ctl_stage_bytes(C, true) > 0 ? 1 : 0;  // mspq_cache_set_staging(0) turns it off (tests)
  *out = c;
  return MSPQ_OK;
}

int mspq_cache_destroy(mspq_cache* c) {
  if (!c) return MSPQ_OK;
  cudaFree(c->blk);
  cudaFreeHost(c->hblk);
  delete c;
  return MSPQ_OK;
}

int mspq_cache_configure(mspq_cache* c, int mode, int policy, const int* caps, int cap_global,
                         int budget, double f1, double f2, void* stream) {
  if (policy < 0 || policy > 4) return set_error(MSPQ_ERR_UNKNOWN_POLICY, "policy ordinal");
  CtlDev& C = c->C;
  C.mode = mode;
  C.policy = policy;
  C.cap_global = cap_global;
  C.budget = budget;
  C.f1 = f1;
  C.f2 = f2;
  cudaError_t e = cudaMemcpyAsync(C.cap, caps, C.L * sizeof(int), cudaMemcpyHostToDevice, ST(stream));
  if (e != cudaSuccess) return cuda_status(e, "cache_configure");
  CK(ctl_reset(C, c->nbuf, ST(stream)), "cache_reset");
}

int mspq_cache_view_get(mspq_cache* c, mspq_cache_view* v) {
  const CtlDev& C = c->C;
  *v = mspq_cache_view{C.elb_ids, C.elb_gates, C.scal, C.req, C.log, C.plan, C.cov, C.step, C.res,
                       (int32_t*)c->hblk, (int32_t*)((char*)c->hblk + 256 + (size_t)(C.E + 8) * 4),
                       (int32_t*)((char*)c->hblk + 256),
                       C.req_cap, C.log_cap, C.plan_cap, c->nbuf};
  return MSPQ_OK;
}

int mspq_cache_set_staging(mspq_cache* c, int on) {
  c->C.stage = on && ctl_stage_bytes(c->C, true) > 0 ? 1 : 0;
  return MSPQ_OK;
}
int mspq_cache_begin_cycle(mspq_cache* c, int k, void* stream) {
  if (k < 0 || k > c->kmax) return set_error(MSPQ_ERR_K_OUT_OF_RANGE, "k > kmax");
  CK(ctl_begin_cycle(c->C, k, ST(stream)), "cache_begin_cycle");
}
int mspq_cache_plan_row(mspq_cache* c, int row, void* stream) {
  CK(ctl_plan_row(c->C, row, ST(stream)), "cache_plan_row");
}
int mspq_cache_verify_layer(mspq_cache* c, int layer, int nslots, const int32_t* tgt,
                            int32_t* gbuf, void* stream) {
  if (nslots > c->kmax + 1) return set_error(MSPQ_ERR_K_OUT_OF_RANGE, "nslots > kmax+1");
  CK(ctl_verify_layer(c->C, layer, nslots, tgt, gbuf, ST(stream)), "cache_verify_layer");
}
int mspq_cache_replay_cycle(mspq_cache* c, const int32_t* target, const int32_t* draft,
                            const double* gates, int pos, int k_eff, int head_pos,
                            int32_t* out_counts, int32_t* out_batches, int32_t* out_jit_rows,
                            int32_t* out_cov, int32_t* out_step, int32_t* out_flush_keys,
                            void* stream) {
  if (k_eff > c->kmax) return set_error(MSPQ_ERR_K_OUT_OF_RANGE, "k_eff > kmax");
  ReplayTrace tr{target, draft, gates};
  ReplayOut o{out_counts, out_batches, out_jit_rows, out_cov, out_step, out_flush_keys};
  CK(ctl_replay_cycle(c->C, tr, pos, k_eff, head_pos, o, ST(stream)), "cache_replay_cycle");
}

// whole-trace replay (one launch, governor on the device); see include/mspq_capi.h
int mspq_cache_replay_all(mspq_cache* c, const int32_t* target, const int32_t* draft, const double* gates,
                          const unsigned char* acc, int n, const int32_t* gov_ints, const double* gov_reals,
                          int nvs, const double* vs_xy, int32_t* slices, int stride, const int32_t* offsets,
                          int32_t* k_eff, int32_t* n_cycles, int32_t* flush_keys, void* stream) {
  if (nvs < 2 || nvs > 16) return set_error(MSPQ_ERR_INSUFFICIENT_SAMPLES, "replay_all: 2..16 verify samples");
  GovDev g{};
  g.use_gov = gov_ints[0];
  g.fixed_k = gov_ints[1];
  g.k_min = gov_ints[2];
  g.k_max = gov_ints[3];
  g.k_slo = gov_ints[4];
  g.kcap = gov_ints[5];
  if (g.kcap > 64 || g.kcap > c->kmax) return set_error(MSPQ_ERR_K_OUT_OF_RANGE, "replay_all: k above kmax");
  g.alpha = gov_reals[0];
  g.initial_accept = gov_reals[1];
  g.pcie_bw = gov_reals[2];
  g.init_lat = gov_reals[3];
  g.overhead = gov_reals[4];
  g.expert_bytes = gov_reals[5];
  g.draft_base = gov_reals[6];
  g.draft_tok = gov_reals[7];
  g.nvs = nvs;
  for (int i = 0; i < nvs; ++i) {
    g.vs_x[i] = vs_xy[2 * i];
    g.vs_y[i] = vs_xy[2 * i + 1];
  }
  ReplayTrace tr{target, draft, gates};
  ReplayAllOut o{slices, stride, offsets[0], offsets[1], offsets[2], offsets[3], k_eff, n_cycles, flush_keys};
  CK(ctl_replay_all(c->C, tr, acc, n, g, o, ST(stream)), "cache_replay_all");
}

}  // extern "C"
