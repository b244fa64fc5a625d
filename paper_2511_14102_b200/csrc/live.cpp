// Live speculative decode engine (the generate() drop-in next to run_simulation, sim.hpp:86).
//
// Per cycle:
//   governor: k = select_k(profile re-fit on this B200, EMA acceptance, g)   perfmodel.cpp:166-183
//   draft:    k replays of a captured CUDA graph (embed -> L x [K1 gate/top-k + ELB row -> K2
//             INT4 grouped FFN] -> norm -> LM head -> argmax/advance); after each row the device
//             planner (K4 plan_row) decides Phase-II/III prefetches; the host issues those H2D
//             copies on the copy-engine stream while the next draft row runs.
//   verify:   layer-major over the k+1 window slots: K1 (target routing) -> K4 verify_layer
//             (refill / demand policy steps, slot-pool buffers, grouped-GEMM schedule) -> demand
//             H2D -> wait on the copies this layer's experts need (= exposed stall) -> K3 bf16
//             grouped FFN -> ... -> LM head -> argmax -> K5 accept/advance.
//   record:   CycleRecord in the reference schema (sim.cpp:468-510) with measured times.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mspq_capi.h"
#include "json.hpp"
#include "status.h"

using json = nlohmann::ordered_json;

#include "host_common.h"

using namespace mspq_host;

#define CUDA_OK(x)                                                                                  \
  do {                                                                                              \
    cudaError_t _e = (x);                                                                           \
    if (_e != cudaSuccess) fail(MSPQ_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e));   \
  } while (0)
#define CAPI_OK(x)                                                     \
  do {                                                                 \
    int _s = (x);                                                      \
    if (_s) fail(_s, std::string(#x) + ": " + mspq_last_error());      \
  } while (0)

namespace {

enum : int { S_TOTAL = 0, S_NFREE, S_NPEND, S_K, S_T1, S_T2, S_NREQ, S_NLOG, S_NPLAN, S_FETCHED, S_DEMAND, S_JIT, S_OVERFLOW };

struct Sched {
  int32_t* base = nullptr;
  int32_t *n_groups, *group_expert, *group_buf, *group_off, *entry_tok, *entry_of, *entry_group;
  void carve(int32_t* p, int G, int N) {
    base = p;
    n_groups = p;
    group_expert = p + 4;
    group_buf = group_expert + G;
    group_off = group_buf + G;
    entry_tok = group_off + G + 1;
    entry_of = entry_tok + N;
    entry_group = entry_of + N;
  }
  static size_t ints(int G, int N) { return 4 + 3 * (size_t)G + 1 + 3 * (size_t)N + 8; }
};

double elapsed_s(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e-3;
}

}  // namespace

struct mspq_engine {
  mspq_model_desc m{};
  mspq_engine_opts o{};
  std::string store_path;
  cudaStream_t sc = nullptr, sx = nullptr;
  int64_t S16 = 0, S4 = 0;
  int Tmax = 0, G = 0, N = 0;
  // device weights
  void* wblk = nullptr;
  uint16_t *embed = nullptr, *pos = nullptr, *lm = nullptr, *gfinal = nullptr, *gamma = nullptr, *router = nullptr;
  unsigned char* draft4 = nullptr;
  // host store (expert_codec 1: one XC blob per payload in a region of Sreg bytes)
  unsigned char* host = nullptr;
  size_t host_bytes = 0;
  int codec = 0;
  int64_t Sreg = 0;        // host bytes reserved per payload (S16 raw; worst-case blob with the codec)
  int n_tiles = 0;         // 16 KB tile images per bf16 expert
  uint64_t xc_bytes_total = 0;
  cudaStream_t sdec = nullptr;        // codec: decode stream (copy chunks land on sx, decode here)
  unsigned char* stage[2] = {nullptr, nullptr};
  cudaEvent_t ev_stage[2] = {nullptr, nullptr};
  char stage_rec[2] = {0, 0};
  int stage_next = 0;
  // deferred prefetch (run-config "prefetch_defer", default on; per-layer capacity only): a plan
  // prefetch for layer j >= 1 is issued on the demand stream right after layer j-1's demand
  // copies, so it covers the layer boundary (GEMM, K1, controller) when the link would otherwise
  // idle.  FIFO order on the stream keeps it ahead of any later demand write to the same slot.
  bool pf_defer = false;
  // decode grid per chunk: <= one CTA per SM, so a decode never holds a whole SM register file
  // and the verify GEMM (higher stream priority) co-resides on every SM (256: K3 0.66 of HBM at cap 4)
  static constexpr int dec_ctas = 128;
  std::vector<std::pair<int, int>> deferred;  // (key, buf), plan order
  int n_payload = 0;
  bool host_is_shm = false;
  // slot pool
  unsigned char* pool = nullptr;
  int nbuf = 0;
  mspq_cache* cache = nullptr;
  mspq_cache_view view{};
  // workspaces
  void* ws = nullptr;
  float* h = nullptr;
  uint16_t* xn = nullptr;
  int32_t* ids_t = nullptr;
  float* wts_t = nullptr;
  int32_t* ids_d = nullptr;
  float* wts_d = nullptr;
  Sched sv[2], sd[2];
  float *yv[2] = {nullptr, nullptr}, *yd[2] = {nullptr, nullptr};
  int yv_splits[2] = {1, 1};
  int yd_split1 = 1, yd_split2 = 1;
  void* tcws = nullptr;
  void* tcws_d = nullptr;
  static constexpr int kMaxSplit = 8;
  uint16_t* act = nullptr;
  uint16_t* act_d = nullptr;  // draft GEMV: [K][f] SiLU(gate) * up
  float* logits = nullptr;
  int32_t* amax = nullptr;
  int32_t* gbuf = nullptr;  // [E] first-request buffer per expert of the current verify layer
  std::vector<int> layer_bufs;
  int32_t* dst = nullptr;  // device state: [0] row [1] cur_tok [2] cur_pos [3] accepted [4] bonus [8..] win_tok [8+Tmax+1..] win_pos
  int32_t* hpin = nullptr;  // pinned host mirror for small transfers
  size_t hpin_ints = 0;
  // draft graph
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  // copy bookkeeping
  std::vector<cudaEvent_t> ev_ready;
  std::vector<char> ready_rec;
  std::vector<int> last_cycle, last_layer;
  std::vector<cudaEvent_t> ev_gemm, ev_w0, ev_w1, ev_row, ev_k0, ev_g0, ev_g1, ev_ka1, ev_rt;
  std::vector<char> layer_parts;  // verify layer ran its GEMM in two parts (resident / in flight)
  int graph_nodes = 0;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_pool_next = 0;
  cudaEvent_t ev_c0 = nullptr, ev_dend = nullptr, ev_end = nullptr, ev_t0 = nullptr;
  // config
  bool configured = false;
  HostCfg cfg;
  std::vector<int> caps;
  double pcie_bw_measured = 0.0, draft_step_s = 0.0, home_bw_measured = 0.0;
  std::pair<double, double> pcie_fixed{0.0, -1.0};             // (init latency, per-copy overhead) s
  std::vector<std::pair<double, double>> verify_measured;       // (window, s) timed verify passes
  std::vector<std::pair<double, double>> verify_fit;
  int cycle_serial = 0;
  // "elb" estimator state: per (layer, expert) routing frequency from the draft's
  // ELB rows (decayed per row) and the residency table snapshotted at the end of each cycle.
  // Both persist across generate() calls, like the cache itself.
  std::vector<double> elb_freq;
  std::vector<int32_t> res_host;
  std::vector<double> elb_calib;  // [kmax+1] EMA of fetched / estimated for the k actually run
  // the governor's learned state (EMA acceptance p_i, g) persists across generate() calls of one
  // configuration, as in serving; configure() resets it
  std::vector<double> gov_accept;
  double gov_g = -1.0;
  // trace_level >= 3 (parity tests): the fp32 residual entering every layer (index L = final),
  // for the verify window [L+1][T][d] and each draft row [k][L+1][d], kept per cycle of the
  // last generate() and read back with mspq_engine_read("hcap_v:<cycle>" / "hcap_d:<cycle>")
  float *hcap_v = nullptr, *hcap_dstage = nullptr, *hcap_d = nullptr;
  float *hmid_v = nullptr, *hmid_dstage = nullptr, *hmid_d = nullptr;  // after the attention residual
  std::vector<std::vector<float>> hmid_v_hist, hmid_d_hist;
  // attention: bf16 weights shared by draft and target, tile-major per layer
  // [Wqkv (H+2Hkv)Dh x d | Wo d x H Dh]; one KV cache [L][P][Hkv][Dh] shared by both
  bool attn = false;
  int Nq = 0, Nkv = 0, Nqkv = 0;
  unsigned char* wattn = nullptr;
  size_t wattn_layer = 0;
  uint16_t* gamma_a = nullptr;
  uint16_t *kcache = nullptr, *vcache = nullptr;
  float *qkv = nullptr, *oproj = nullptr;  // split planes [kMaxSplit][Tmax][Nqkv | d]
  uint16_t* ao = nullptr;                  // [Tmax][Nq] attention output
  int32_t* dsched = nullptr;               // [Tmax + 1][4 + Tmax] packed dense schedules per T
  void* dws = nullptr;
  float* attn_part = nullptr;  // split-K attention partials
  // several request streams (mspq_generate_batch): stream s has its own device decode state, KV
  // cache (kv_base + s * L * kv_layer) and captured draft graph; E->dst / E->kcache / E->vcache /
  // E->gexec point at the current one (stream 0 outside a batch)
  int S = 1;
  std::vector<int32_t*> dst_s;
  uint16_t *kv_base_k = nullptr, *kv_base_v = nullptr;
  std::vector<cudaGraph_t> graph_s;
  std::vector<cudaGraphExec_t> gexec_s;
  int32_t* bmeta = nullptr;  // [Tmax][3] batch window metadata (window base row, stream, position)
  int32_t* btok = nullptr;   // [Tmax] batch tokens
  int32_t* bpos = nullptr;   // [Tmax] batch positions
  void use_stream(int st) {
    dst = dst_s[st];
    if (kv_base_k) {
      kcache = kv_base_k + (size_t)st * m.L * kv_layer();
      vcache = kv_base_v + (size_t)st * m.L * kv_layer();
    }
    gexec = gexec_s.empty() ? gexec : gexec_s[st];
  }
  // prefill (§2.2 of DESIGN.md): every expert of a layer streamed into one of two layer buffers
  unsigned char* pf_buf[2] = {nullptr, nullptr};
  cudaEvent_t pf_ready[2] = {nullptr, nullptr}, pf_done[2] = {nullptr, nullptr};
  float* pf_h = nullptr;                 // [n][d] residual of every prompt token
  float* pf_y[2] = {nullptr, nullptr};   // [chunk][kMaxSplit][32 K][d] MoE planes by layer parity
  int32_t* pf_gbuf = nullptr;            // [E] identity expert -> layer-buffer slot
  int32_t* pf_eo = nullptr;              // [chunk][32 K] each chunk's entry_of, kept for the next layer
  int pf_n = 0;                          // prompt capacity of pf_h / pf_y
  int32_t* dsched_of(int T) { return dsched + (size_t)T * (4 + Tmax); }
  size_t kv_layer() const { return (size_t)m.P * m.Hkv * m.Dh; }
  int32_t* sched_cap = nullptr;  // collect_plans: each verify layer's device schedule [L][Sched::ints]
  // peer-expert tier (home partitioning, include/mspq_capi.h (3)): expert (l, e) lives in the home
  // region of engine e % peer_G at slot l * home_per_layer + e / peer_G
  int peer_G = 0, peer_rank = 0, home_per_layer = 0;
  unsigned char* home = nullptr;
  size_t home_bytes = 0;
  std::vector<unsigned char*> peer_home;  // [G] base of each engine's home region (nullptr = not attached)
  std::vector<char> peer_ipc;             // [G] mapped with cudaIpcOpenMemHandle (closed on destroy)
  uint64_t gen_peer_bytes = 0, gen_home_local_bytes = 0;
  uint64_t n_peer = 0, n_home_local = 0;
  uint64_t n_refetch = 0;  // fetches served from the key's first-request buffer of the layer
  std::vector<int> fill_at;
  const unsigned char* home_src(int key) const {
    if (peer_G <= 0) return nullptr;
    const int l = key / m.E, e = key % m.E, owner = e % peer_G;
    const unsigned char* base = peer_home[owner];
    return base ? base + ((size_t)l * home_per_layer + e / peer_G) * (size_t)S16 : nullptr;
  }
  std::vector<std::vector<float>> hcap_v_hist, hcap_d_hist;

  int32_t* win_tok() { return dst + 8; }
  int32_t* win_pos() { return dst + 8 + Tmax + 1; }
  int64_t payload(int key) const { return m.unique_experts > 0 ? key % m.unique_experts : key; }
  const unsigned char* host_blob(int64_t p) const { return host + (size_t)p * Sreg; }
  // bytes the copy engine moves for payload p (the blob size with the codec)
  uint64_t wire_bytes(int64_t p) const {
    return codec ? reinterpret_cast<const uint32_t*>(host_blob(p) + 64)[n_tiles] : (uint64_t)S16;
  }

  cudaEvent_t pool_event() {
    if (ev_pool_next >= ev_pool.size()) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_pool_next++];
  }
};

namespace {

void make_weights(mspq_engine* E) {
  const auto& m = E->m;
  const int64_t d = m.d;
  size_t n_embed = (size_t)m.V * d, n_pos = (size_t)m.P * d, n_lm = n_embed, n_g = (size_t)(m.L + 1) * d,
         n_r = (size_t)m.L * m.E * d;
  size_t total = (n_embed + n_pos + n_lm + n_g + n_r) * 2;
  CUDA_OK(cudaMalloc(&E->wblk, total));
  uint16_t* p = (uint16_t*)E->wblk;
  E->embed = p;
  p += n_embed;
  E->pos = p;
  p += n_pos;
  E->lm = p;
  p += n_lm;
  E->gamma = p;
  p += (size_t)m.L * d;
  E->gfinal = p;
  p += d;
  E->router = p;
  void* s = E->sc;
  CAPI_OK(mspq_fill_bf16(m.seed, 1, m.embed_scale, 0, E->embed, (long long)n_embed, 0, s));
  CAPI_OK(mspq_fill_bf16(m.seed, 2, m.pos_scale, 0, E->pos, (long long)n_pos, 0, s));
  CAPI_OK(mspq_fill_bf16(m.seed, 3, m.a_lm, 0, E->lm, (long long)n_lm, 0, s));
  CAPI_OK(mspq_fill_bf16(m.seed, 4, 0.f, 1, E->gfinal, d, 0, s));
  if (E->attn) {  // tensor ids 0x800000 + 16 l + {0: Wqkv, 1: Wo, 2: attention RMSNorm gamma}
    const size_t nqkv = (size_t)E->Nqkv * d, no = (size_t)d * E->Nq;
    E->wattn_layer = (nqkv + no) * 2;
    CUDA_OK(cudaMalloc(&E->wattn, (size_t)m.L * E->wattn_layer));
    CUDA_OK(cudaMalloc(&E->gamma_a, (size_t)m.L * d * 2));
    uint16_t* stg;
    CUDA_OK(cudaMalloc(&stg, std::max(nqkv, no) * 2));
    for (int l = 0; l < m.L; ++l) {
      const uint64_t tb = 0x800000ull + (uint64_t)l * 16;
      unsigned char* wl = E->wattn + (size_t)l * E->wattn_layer;
      CAPI_OK(mspq_fill_bf16(m.seed, tb + 0, m.a_qkv, 0, stg, (long long)nqkv, 0, s));
      CAPI_OK(mspq_tile_bf16(stg, E->Nqkv, d, wl, s));
      CAPI_OK(mspq_fill_bf16(m.seed, tb + 1, m.a_o, 0, stg, (long long)no, 0, s));
      CAPI_OK(mspq_tile_bf16(stg, d, E->Nq, wl + nqkv * 2, s));
      CAPI_OK(mspq_fill_bf16(m.seed, tb + 2, 0.f, 1, E->gamma_a + (size_t)l * d, d, 0, s));
    }
    CUDA_OK(cudaStreamSynchronize((cudaStream_t)s));
    cudaFree(stg);
    const size_t kvb = (size_t)E->S * m.L * E->kv_layer() * 2;  // one cache per request stream
    CUDA_OK(cudaMalloc(&E->kcache, kvb));
    CUDA_OK(cudaMalloc(&E->vcache, kvb));
    CUDA_OK(cudaMemset(E->kcache, 0, kvb));
    CUDA_OK(cudaMemset(E->vcache, 0, kvb));
    E->kv_base_k = E->kcache;
    E->kv_base_v = E->vcache;
  }
  for (int l = 0; l < m.L; ++l) {
    CAPI_OK(mspq_fill_bf16(m.seed, 0x100ull + (uint64_t)l * 16, 0.f, 1, E->gamma + (size_t)l * d, d, 0, s));
    CAPI_OK(mspq_fill_bf16(m.seed, 0x100ull + (uint64_t)l * 16 + 1, m.a_router, 0, E->router + (size_t)l * m.E * d,
                           (long long)m.E * d, 0, s));
  }
}

void alloc_host_store(mspq_engine* E) {
  E->host_bytes = (size_t)E->n_payload * E->Sreg;
  if (E->store_path.empty()) {
    CUDA_OK(cudaHostAlloc((void**)&E->host, E->host_bytes, cudaHostAllocPortable));
    return;
  }
  // shared pinned store: a /dev/shm file mapped by every rank and registered with CUDA
  const bool create = E->o.host_store_role == 0;
  const std::string ready = E->store_path + ".ready";
  int fd;
  if (create) {
    unlink(ready.c_str());
    fd = open(E->store_path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
    if (fd < 0) fail(MSPQ_ERR_IO, "cannot create host store " + E->store_path);
    if (ftruncate(fd, (off_t)E->host_bytes) != 0) fail(MSPQ_ERR_IO, "ftruncate host store");
  } else {
    // the owner publishes "<magic> <bytes> <payloads> <codec>" by an atomic rename once the store
    // is filled; an attacher maps it only if that record and the file size match this engine
    char want[160];
    snprintf(want, sizeof(want), "MSPQSTORE1 %zu %d %d", E->host_bytes, E->n_payload, E->codec);
    bool ok = false;
    for (int i = 0; i < 36000 && !ok; ++i) {
      FILE* f = fopen(ready.c_str(), "r");
      if (f) {
        char got[160] = {0};
        const size_t n = fread(got, 1, sizeof(got) - 1, f);
        fclose(f);
        got[n] = 0;
        if (strncmp(got, "MSPQSTORE1 ", 11) == 0) {
          if (strcmp(got, want) != 0) fail(MSPQ_ERR_IO, std::string("host store record mismatch: ") + got);
          ok = true;
          break;
        }
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(50));
    }
    if (!ok) fail(MSPQ_ERR_IO, "host store never became ready");
    fd = open(E->store_path.c_str(), O_RDWR);
    if (fd < 0) fail(MSPQ_ERR_IO, "cannot open host store " + E->store_path);
    struct stat st;
    if (fstat(fd, &st) != 0 || (size_t)st.st_size != E->host_bytes) {
      close(fd);
      fail(MSPQ_ERR_IO, "host store size does not match this model");
    }
  }
  void* p = mmap(nullptr, E->host_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) fail(MSPQ_ERR_IO, "mmap host store");
  E->host = (unsigned char*)p;
  E->host_is_shm = true;
  CUDA_OK(cudaHostRegister(E->host, E->host_bytes, cudaHostRegisterPortable));
}

// Generates every expert once on the GPU: bf16 blob -> pinned host store (payload) and the
// INT4 draft of every key that maps to it.
void make_experts(mspq_engine* E) {
  const auto& m = E->m;
  const int LE = m.L * m.E;
  const int64_t S16 = E->S16, S4 = E->S4;
  CUDA_OK(cudaMalloc(&E->draft4, (size_t)LE * S4));
  unsigned char* stage[2];
  unsigned char* tiled[2];
  CUDA_OK(cudaMalloc(&stage[0], S16));
  CUDA_OK(cudaMalloc(&stage[1], S16));
  CUDA_OK(cudaMalloc(&tiled[0], S16));
  CUDA_OK(cudaMalloc(&tiled[1], S16));
  const bool fill_host = !(E->host_is_shm && E->o.host_store_role != 0);
  const int64_t q13 = (int64_t)2 * m.f * m.d / 2, s13 = (int64_t)2 * m.f * (m.d / 128) * 2, q2 = (int64_t)m.d * m.f / 2;
  unsigned char* rq;  // row-major quantised staging, tiled into the draft blob below
  CUDA_OK(cudaMalloc(&rq, S4));
  unsigned char *xscr = nullptr, *xout = nullptr;
  if (E->codec && fill_host) {
    CUDA_OK(cudaMalloc(&xscr, (size_t)mspq_xc_scratch_bytes(E->n_tiles)));
    CUDA_OK(cudaMalloc(&xout, (size_t)E->Sreg));
  }
  for (int p = 0; p < E->n_payload; ++p) {
    unsigned char* st = stage[p & 1];
    const int cl = p / m.E, ce = p % m.E;
    CAPI_OK(mspq_fill_expert(m.seed, cl, ce, m.d, m.f, m.a_up, m.a_down, st, E->sc));
    CAPI_OK(mspq_quantize_int4(st, 2 * m.f, m.d, rq, rq + q13, E->sc));
    CAPI_OK(mspq_quantize_int4(st + (size_t)2 * m.f * m.d * 2, m.d, m.f, rq + q13 + s13, rq + q13 + s13 + q2, E->sc));
    for (int key = p; key < LE; key += E->n_payload) {
      // draft blob for the T = 1 GEMV (gemv_int4.cu): fragment-major q words, row-major scales
      unsigned char* b4 = E->draft4 + (size_t)key * S4;
      CAPI_OK(mspq_fragtile_int4(rq, 2 * m.f, m.d, b4, E->sc));
      CUDA_OK(cudaMemcpyAsync(b4 + q13, rq + q13, (size_t)s13, cudaMemcpyDeviceToDevice, E->sc));
      CAPI_OK(mspq_fragtile_int4(rq + q13 + s13, m.d, m.f, b4 + q13 + s13, E->sc));
      CUDA_OK(cudaMemcpyAsync(b4 + q13 + s13 + q2, rq + q13 + s13 + q2, (size_t)(S4 - q13 - s13 - q2),
                              cudaMemcpyDeviceToDevice, E->sc));
    }
    if (fill_host) {
      // host store keeps the tile-major SW128 images K3 streams with one bulk copy per tile
      unsigned char* tl = tiled[p & 1];
      CAPI_OK(mspq_tile_bf16(st, 2 * m.f, m.d, tl, E->sc));
      CAPI_OK(mspq_tile_bf16(st + (size_t)2 * m.f * m.d * 2, m.d, m.f, tl + (size_t)2 * m.f * m.d * 2, E->sc));
      if (E->codec) {
        long long nb = 0;
        CAPI_OK(mspq_xc_encode(tl, E->n_tiles, xscr, xout, E->Sreg, &nb, E->sc));
        CUDA_OK(cudaMemcpyAsync(E->host + (size_t)p * E->Sreg, xout, (size_t)nb, cudaMemcpyDeviceToHost, E->sc));
        CUDA_OK(cudaStreamSynchronize(E->sc));  // xout is reused by the next payload
      } else {
        CUDA_OK(cudaMemcpyAsync(E->host + (size_t)p * S16, tl, S16, cudaMemcpyDeviceToHost, E->sc));
      }
    }
  }
  if (xscr) cudaFree(xscr);
  if (xout) cudaFree(xout);
  CUDA_OK(cudaStreamSynchronize(E->sc));
  cudaFree(rq);
  cudaFree(stage[0]);
  cudaFree(stage[1]);
  cudaFree(tiled[0]);
  cudaFree(tiled[1]);
  if (E->codec)
    for (int p = 0; p < E->n_payload; ++p) E->xc_bytes_total += E->wire_bytes(p);
  if (E->host_is_shm && E->o.host_store_role == 0) {
    const std::string ready = E->store_path + ".ready", tmp = ready + ".tmp";
    FILE* f = fopen(tmp.c_str(), "w");
    if (!f) fail(MSPQ_ERR_IO, "cannot write " + tmp);
    fprintf(f, "MSPQSTORE1 %zu %d %d", E->host_bytes, E->n_payload, E->codec);
    fclose(f);
    if (rename(tmp.c_str(), ready.c_str()) != 0) fail(MSPQ_ERR_IO, "cannot publish " + ready);
  }
}

void make_workspaces(mspq_engine* E) {
  const auto& m = E->m;
  const int T = E->Tmax, K = m.K, L = m.L, d = m.d, f = m.f;
  E->G = std::min(m.E, T * K);
  E->N = T * K;
  const size_t sched_ints = Sched::ints(E->G, E->N);
  size_t off = 0;
  auto take = [&](size_t b) {
    size_t o = off;
    off += (b + 255) & ~size_t(255);
    return o;
  };
  size_t o_h = take((size_t)T * d * 4), o_xn = take((size_t)T * d * 2), o_it = take((size_t)L * T * K * 4),
         o_wt = take((size_t)L * T * K * 4), o_id = take((size_t)L * K * 4), o_wd = take((size_t)L * K * 4),
         o_sv0 = take(sched_ints * 4), o_sv1 = take(sched_ints * 4), o_sd0 = take(Sched::ints(K, K) * 4),
         o_sd1 = take(Sched::ints(K, K) * 4), o_yv0 = take((size_t)mspq_engine::kMaxSplit * E->N * d * 4),
         o_yv1 = take((size_t)mspq_engine::kMaxSplit * E->N * d * 4),
         o_yd0 = take((size_t)mspq_engine::kMaxSplit * K * d * 4), o_yd1 = take((size_t)mspq_engine::kMaxSplit * K * d * 4),
         o_act = take((size_t)E->N * f * 2),
         o_lg = take((size_t)T * m.V * 4), o_am = take((size_t)T * 4), o_dst = take((size_t)(8 + 2 * (T + 1)) * 4),
         o_gb = take((size_t)m.E * 4),
         o_tc = take((size_t)mspq_moe_bf16_tc_ws_bytes(d, f, T, K, E->G, mspq_engine::kMaxSplit)),
         o_tcd = take((size_t)mspq_moe_bf16_tc_ws_bytes(d, f, 1, K, K, mspq_engine::kMaxSplit));
  CUDA_OK(cudaMalloc(&E->ws, off));
  CUDA_OK(cudaMemset(E->ws, 0, off));
  CUDA_OK(cudaDeviceSynchronize());  // the engine's streams are non-blocking w.r.t. the legacy stream
  char* b = (char*)E->ws;
  E->h = (float*)(b + o_h);
  E->xn = (uint16_t*)(b + o_xn);
  E->ids_t = (int32_t*)(b + o_it);
  E->wts_t = (float*)(b + o_wt);
  E->ids_d = (int32_t*)(b + o_id);
  E->wts_d = (float*)(b + o_wd);
  E->sv[0].carve((int32_t*)(b + o_sv0), E->G, E->N);
  E->sv[1].carve((int32_t*)(b + o_sv1), E->G, E->N);
  E->sd[0].carve((int32_t*)(b + o_sd0), K, K);
  E->sd[1].carve((int32_t*)(b + o_sd1), K, K);
  E->yv[0] = (float*)(b + o_yv0);
  E->yv[1] = (float*)(b + o_yv1);
  E->yd[0] = (float*)(b + o_yd0);
  E->yd[1] = (float*)(b + o_yd1);
  E->act = (uint16_t*)(b + o_act);
  E->logits = (float*)(b + o_lg);
  E->amax = (int32_t*)(b + o_am);
  E->dst = (int32_t*)(b + o_dst);
  E->dst_s.assign(E->S, nullptr);
  E->dst_s[0] = E->dst;
  for (int st = 1; st < E->S; ++st) {
    CUDA_OK(cudaMalloc(&E->dst_s[st], (size_t)(8 + 2 * (T + 1)) * 4));
    CUDA_OK(cudaMemset(E->dst_s[st], 0, (size_t)(8 + 2 * (T + 1)) * 4));
  }
  CUDA_OK(cudaMalloc(&E->bmeta, (size_t)T * 3 * 4));
  CUDA_OK(cudaMalloc(&E->btok, (size_t)T * 4));
  CUDA_OK(cudaMalloc(&E->bpos, (size_t)T * 4));
  E->gbuf = (int32_t*)(b + o_gb);
  E->tcws = (void*)(b + o_tc);
  E->tcws_d = (void*)(b + o_tcd);
  E->hpin_ints = 64 + (size_t)L * T * K * 2 + (size_t)E->Tmax * L * K * 3 + 4 * T + (size_t)L * 2 + (size_t)L * T * 2 +
                 (size_t)L * m.E + 64;
  CUDA_OK(cudaHostAlloc((void**)&E->hpin, E->hpin_ints * 4, 0));
  CUDA_OK(cudaMalloc(&E->sched_cap, (size_t)L * sched_ints * 4));
  CUDA_OK(cudaMalloc(&E->act_d, (size_t)K * f * 2));
  if (E->attn) {
    const int KS = mspq_engine::kMaxSplit;
    CUDA_OK(cudaMalloc(&E->qkv, (size_t)KS * T * E->Nqkv * 4));
    CUDA_OK(cudaMalloc(&E->oproj, (size_t)KS * T * d * 4));
    CUDA_OK(cudaMalloc(&E->ao, (size_t)T * E->Nq * 2));
    CUDA_OK(cudaMalloc(&E->dws, (size_t)mspq_dense_ws_bytes(std::max(d, E->Nq), T)));
    CUDA_OK(cudaMalloc(&E->attn_part, (size_t)mspq_attention_ws_bytes(T, m.H, m.Hkv, m.Dh)));
    CUDA_OK(cudaMemset(E->attn_part, 0, (size_t)mspq_attention_ws_bytes(T, m.H, m.Hkv, m.Dh)));  // merge counters
    std::vector<int32_t> ds((size_t)(T + 1) * (4 + T), 0);
    for (int t = 1; t <= T; ++t) mspq_dense_sched_fill(ds.data() + (size_t)t * (4 + T), t);
    CUDA_OK(cudaMalloc(&E->dsched, ds.size() * 4));
    CUDA_OK(cudaMemcpy(E->dsched, ds.data(), ds.size() * 4, cudaMemcpyHostToDevice));
  }
  if (E->o.trace_level >= 3) {
    CUDA_OK(cudaMalloc(&E->hcap_v, (size_t)(L + 1) * T * d * 4));
    CUDA_OK(cudaMalloc(&E->hcap_dstage, (size_t)(L + 1) * d * 4));
    CUDA_OK(cudaMalloc(&E->hcap_d, (size_t)E->o.kmax * (L + 1) * d * 4));
    if (E->attn) {
      CUDA_OK(cudaMalloc(&E->hmid_v, (size_t)L * T * d * 4));
      CUDA_OK(cudaMalloc(&E->hmid_dstage, (size_t)L * d * 4));
      CUDA_OK(cudaMalloc(&E->hmid_d, (size_t)E->o.kmax * L * d * 4));
    }
  }
}

// One draft step for a single token, captured once as a CUDA graph.
// K splits for a draft GEMM: the most that still give every SM at most one unit of the
// persistent K2 (one CTA per SM)
int split_for(int units_per_split1, int kblocks) {
  const int units = std::max(1, units_per_split1);
  const int sp = std::max(1, 148 / units);  // persistent K2: one CTA per SM
  return std::max(1, std::min({sp, mspq_engine::kMaxSplit, std::max(1, kblocks / 2)}));
}

// K splits for a dense projection: >= ~2 CTAs per SM of tcgen05 units
// K split of a dense projection: the fewest k-blocks on the busiest SM, counting at least 2 CTAs
// per SM (one CTA's 3-stage ring alone does not cover the HBM latency); ties -> fewer planes.
// Phi QKV (48 row tiles x 64 k-blocks): 6 splits = 288 CTAs, <= 2 per SM (7 put 3 on 40 SMs).
int dense_split(int rows, int kdim) {
  const int rt = std::max(1, rows / 128), kb = std::max(1, kdim / 64);
  int best = 1;
  long best_cost = -1;
  for (int sp = 1; sp <= std::min(mspq_engine::kMaxSplit, kb); ++sp) {
    const int per = (kb + sp - 1) / sp, eff = (kb + per - 1) / per;  // non-empty splits
    const long per_sm = std::max(2L, ((long)rt * eff + 147) / 148);
    const long cost = per_sm * per;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = eff;
    }
  }
  return best;
}

// Attention block of layer l for the T tokens in E->h (positions *pos0 ..): K1 (the previous
// layer's MoE combine + attention RMSNorm) -> QKV projection -> shared-KV attention -> O
// projection into E->oproj (split planes).  The caller's next K1 adds them (dense combine) and
// routes.  Returns the O projection's split count.  cap_in (nullable): copy of the residual
// entering the layer (trace_level 3).
int enqueue_attn(mspq_engine* E, int l, int T, const int32_t* pos0, const float* y, const int32_t* entry_of,
                 const float* wts, int y_splits, long long y_stride, float* cap_in, cudaStream_t s,
                 const int32_t* meta = nullptr) {
  const auto& m = E->m;
  const int d = m.d;
  // the normed rows go straight into the QKV GEMM's B image and the attention output into the O
  // GEMM's (one workspace, used in stream order): no gather kernels
  CAPI_OK(mspq_gate_topk_img(E->h, y, entry_of, wts, y_splits, y_stride, E->gamma_a + (size_t)l * d, nullptr, E->xn,
                             nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, l, m.L, T, d, m.E, m.K,
                             m.eps, E->dws, s));
  if (cap_in) CUDA_OK(cudaMemcpyAsync(cap_in, E->h, (size_t)T * d * 4, cudaMemcpyDeviceToDevice, s));
  const unsigned char* wl = E->wattn + (size_t)l * E->wattn_layer;
  const int spq = dense_split(E->Nqkv, d), spo = dense_split(d, E->Nq);
  CAPI_OK(mspq_dense_bf16_tc(E->dsched_of(T), nullptr, wl, E->Nqkv, d, T, spq, E->dws, E->qkv, (long long)T * E->Nqkv, s));
  if (meta)  // batched request streams: per-token window / stream / position, one KV cache per stream
    CAPI_OK(mspq_attention_batched(E->qkv, spq, (long long)T * E->Nqkv, T, m.H, m.Hkv, m.Dh, m.P, meta,
                                   (long long)m.L * (long long)E->kv_layer(), E->kv_base_k + (size_t)l * E->kv_layer(),
                                   E->kv_base_v + (size_t)l * E->kv_layer(), nullptr, E->dws, E->attn_part, s));
  else
    CAPI_OK(mspq_attention(E->qkv, spq, (long long)T * E->Nqkv, T, m.H, m.Hkv, m.Dh, m.P, pos0,
                           E->kcache + (size_t)l * E->kv_layer(), E->vcache + (size_t)l * E->kv_layer(), nullptr,
                           E->dws, E->attn_part, s));
  CAPI_OK(mspq_dense_bf16_tc(E->dsched_of(T), nullptr, wl + (size_t)E->Nqkv * d * 2, d, E->Nq, T, spo, E->dws,
                             E->oproj, (long long)T * d, s));
  return spo;
}

void enqueue_draft_step(mspq_engine* E, cudaStream_t s) {
  const auto& m = E->m;
  const int K = m.K, L = m.L, d = m.d;
  // the draft GEMV: W13 in one pass (SiLU*up fused), W2 over K splits so a layer launches >= ~3
  // CTAs per SM (d/64 row blocks x K experts x split2)
  E->yd_split1 = 1;
  E->yd_split2 = std::max(1, std::min(m.f / 128, (3 * 148 + (d / 64) * K - 1) / ((d / 64) * K)));
  int32_t* row = E->dst + 0;
  int32_t* cur_tok = E->dst + 1;
  int32_t* cur_pos = E->dst + 2;
  CAPI_OK(mspq_embed(E->embed, E->pos, cur_tok, cur_pos, 1, d, E->h, s));
  for (int l = 0; l < L; ++l) {
    const int pl = (l - 1) & 1;
    const float* y = l ? E->yd[pl] : nullptr;
    const int32_t* eo = l ? E->sd[pl].entry_of : nullptr;
    const float* pw = l ? E->wts_d + (size_t)(l - 1) * K : nullptr;
    int ysp = E->yd_split2;
    long long yst = (long long)K * d;
    if (E->attn) {  // attention first: its K1 takes the MoE combine, the MoE K1 the dense one
      ysp = enqueue_attn(E, l, 1, cur_pos, y, eo, pw, ysp, yst, E->hcap_dstage ? E->hcap_dstage + (size_t)l * d : nullptr,
                         s);
      y = E->oproj;
      eo = nullptr;
      pw = nullptr;
      yst = d;
    }
    CAPI_OK(mspq_gate_topk(E->h, y, eo, pw, ysp, yst, E->gamma + (size_t)l * d,
                           E->router + (size_t)l * m.E * d, E->xn, E->ids_d + (size_t)l * K, E->wts_d + (size_t)l * K,
                           nullptr, E->view.elb_ids, E->view.elb_gates, row, E->sd[l & 1].base, l, L, 1, d, m.E, K,
                           m.eps, s));
    if (E->hmid_dstage)
      CUDA_OK(cudaMemcpyAsync(E->hmid_dstage + (size_t)l * d, E->h, (size_t)d * 4, cudaMemcpyDeviceToDevice, s));
    else if (E->hcap_dstage && !E->attn)
      CUDA_OK(cudaMemcpyAsync(E->hcap_dstage + (size_t)l * d, E->h, (size_t)d * 4, cudaMemcpyDeviceToDevice, s));
    Sched& sc = E->sd[l & 1];
    CAPI_OK(mspq_moe_int4_gemv(sc.n_groups, sc.group_expert, E->xn, E->draft4, E->S4, l, m.E, d, m.f, K,
                               E->yd_split2, E->act_d, E->yd[l & 1], s));
  }
  const int pl = (L - 1) & 1;
  CAPI_OK(mspq_gate_topk(E->h, E->yd[pl], E->sd[pl].entry_of, E->wts_d + (size_t)(L - 1) * K, E->yd_split2,
                         (long long)K * d, E->gfinal, nullptr,
                         E->xn, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, L, L, 1, d, m.E, K, m.eps,
                         s));
  if (E->hcap_dstage)
    CUDA_OK(cudaMemcpyAsync(E->hcap_dstage + (size_t)L * d, E->h, (size_t)d * 4, cudaMemcpyDeviceToDevice, s));
  CAPI_OK(mspq_lm_head(E->xn, E->lm, 1, m.V, d, E->logits, s));
  CAPI_OK(mspq_argmax_advance(E->logits, m.V, E->amax, row, E->win_tok() + 1, cur_tok, cur_pos, s));
}

// Norm gammas + routers (contiguous, ~4 MB for Phi) are re-read every draft step while 2.6 GB
// of expert/LM weights stream past; mark them L2-persisting for the captured graph's kernels.
void l2_persist(mspq_engine* E, cudaGraph_t g) {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess || prop.persistingL2CacheMaxSize <= 0) return;
  const size_t want = ((size_t)(E->m.L + 1) * E->m.d + (size_t)E->m.L * E->m.E * E->m.d) * 2;
  const size_t win = std::min<size_t>(want, prop.accessPolicyMaxWindowSize);
  cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(win, prop.persistingL2CacheMaxSize));
  cudaKernelNodeAttrValue v{};
  v.accessPolicyWindow.base_ptr = E->gamma;
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = 1.0f;
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  size_t n = 0;
  cudaGraphGetNodes(g, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n);
  cudaGraphGetNodes(g, nodes.data(), &n);
  for (auto nd : nodes) {
    cudaGraphNodeType t;
    cudaGraphNodeGetType(nd, &t);
    if (t == cudaGraphNodeTypeKernel) cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributeAccessPolicyWindow, &v);
  }
  cudaGetLastError();  // the window is a hint: never fail the engine over it
}

void capture_draft_graph(mspq_engine* E) {
  CUDA_OK(cudaStreamBeginCapture(E->sc, cudaStreamCaptureModeThreadLocal));
  try {
    enqueue_draft_step(E, E->sc);
  } catch (...) {
    cudaGraph_t g;
    cudaStreamEndCapture(E->sc, &g);
    throw;
  }
  CUDA_OK(cudaStreamEndCapture(E->sc, &E->graph));
  l2_persist(E, E->graph);
  CUDA_OK(cudaGraphInstantiate(&E->gexec, E->graph, 0));
  size_t nn = 0;
  CUDA_OK(cudaGraphGetNodes(E->graph, nullptr, &nn));
  E->graph_nodes = (int)nn;
}

// PCIe fixed costs (perfmodel.hpp:15-30 T_pcie,init and T_pcie,overhead), measured on the copy
// stream: init = one 4 KB pinned H2D copy from idle (the first byte's latency); overhead = the
// per-copy constant of t(n) = overhead + n / B fitted on two copy sizes (32 MB and 8 MB, or the
// store's size and a quarter of it for small models)
std::pair<double, double> measure_pcie_fixed(mspq_engine* E) {
  const size_t n2 = std::min<size_t>(32u << 20, E->host_bytes & ~(size_t)4095), n1 = n2 / 4;
  void* dbuf;
  CUDA_OK(cudaMalloc(&dbuf, n2));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timed = [&](size_t n, int reps) {
    CUDA_OK(cudaMemcpyAsync(dbuf, E->host, n, cudaMemcpyHostToDevice, E->sx));  // warm
    CUDA_OK(cudaStreamSynchronize(E->sx));
    double best = 1e30;
    for (int r = 0; r < reps; ++r) {
      cudaEventRecord(a, E->sx);
      CUDA_OK(cudaMemcpyAsync(dbuf, E->host, n, cudaMemcpyHostToDevice, E->sx));
      cudaEventRecord(b, E->sx);
      CUDA_OK(cudaEventSynchronize(b));
      best = std::min(best, elapsed_s(a, b));
    }
    return best;
  };
  const double t0 = timed(4096, 8), t1 = timed(n1, 4), t2 = timed(n2, 4);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(dbuf);
  const double over = std::max(0.0, (t1 * (double)n2 - t2 * (double)n1) / (double)(n2 - n1));
  return {t0, over};
}

// Verify samples (perfmodel.hpp:26 t_verify(window)), MEASURED: for window w in {1, 5, 9, 17} (<= kmax+1),
// one full target pass over w tokens with u = round(E (1 - (1 - K/E)^w)) distinct experts per layer
// resident (the expected union) -- embed, per layer [attention] + K1 + schedule + K3 grouped GEMM
// (+ the final norm and LM head), exactly the kernels a verify runs, on the compute stream, no
// copies.  The experts are the first u slot-pool buffers (timing does not depend on their values).
std::vector<std::pair<double, double>> measure_verify(mspq_engine* E) {
  const auto& m = E->m;
  const int L = m.L, K = m.K, Ex = m.E, d = m.d;
  std::vector<std::pair<double, double>> out;
  std::vector<int32_t> gb(Ex), ids;
  for (int e = 0; e < Ex; ++e) gb[e] = e < E->nbuf ? e : E->nbuf - 1;
  int32_t* dgb;
  int32_t* dids;
  CUDA_OK(cudaMalloc(&dgb, Ex * 4));
  CUDA_OK(cudaMalloc(&dids, (size_t)E->Tmax * K * 4));
  CUDA_OK(cudaMemcpy(dgb, gb.data(), Ex * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w : {1, 5, 9, 17}) {
    if (w > E->o.kmax + 1) break;  // decode windows are k + 1 <= kmax + 1
    const int u = std::max(K, std::min(Ex, (int)std::lround((double)Ex * (1.0 - std::pow(1.0 - (double)K / Ex, w)))));
    ids.assign((size_t)w * K, 0);
    for (int t = 0; t < w; ++t)
      for (int j = 0; j < K; ++j) ids[(size_t)t * K + j] = (t * K + j) % u;  // distinct within a token (K <= u)
    for (int s2 = 0; s2 < w; ++s2) {
      E->hpin[s2] = s2 % m.V;
      E->hpin[E->Tmax + 1 + s2] = s2;
    }
    CUDA_OK(cudaMemcpyAsync(dids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, E->sc));
    CUDA_OK(cudaMemcpyAsync(E->win_tok(), E->hpin, w * 4, cudaMemcpyHostToDevice, E->sc));
    CUDA_OK(cudaMemcpyAsync(E->win_pos(), E->hpin + E->Tmax + 1, w * 4, cudaMemcpyHostToDevice, E->sc));
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
      CUDA_OK(cudaEventRecord(a, E->sc));
      CAPI_OK(mspq_embed(E->embed, E->pos, E->win_tok(), E->win_pos(), w, d, E->h, E->sc));
      int ysp = 1;
      for (int l = 0; l < L; ++l) {
        const float* y = l ? E->yv[(l - 1) & 1] : nullptr;
        const int32_t* eo = l ? E->sv[(l - 1) & 1].entry_of : nullptr;
        const float* pw = l ? E->wts_t : nullptr;
        long long yst = (long long)w * K * d;
        if (E->attn) {
          ysp = enqueue_attn(E, l, w, E->win_pos(), y, eo, pw, ysp, yst, nullptr, E->sc);
          y = E->oproj;
          eo = nullptr;
          pw = nullptr;
          yst = (long long)w * d;
        }
        CAPI_OK(mspq_gate_topk(E->h, y, eo, pw, ysp, yst, E->gamma + (size_t)l * d, E->router + (size_t)l * Ex * d,
                               E->xn, E->ids_t, E->wts_t, nullptr, nullptr, nullptr, nullptr, nullptr, l, L, w, d, Ex,
                               K, m.eps, E->sc));
        Sched& sv = E->sv[l & 1];
        CAPI_OK(mspq_build_schedule(dids, w, K, Ex, dgb, sv.n_groups, sv.group_expert, sv.group_buf, sv.group_off,
                                    sv.entry_tok, sv.entry_of, sv.entry_group, E->sc));
        const int units = std::max(1, u * (2 * m.f / 128));
        const int sp1 = std::max(1, std::min({(296 + units - 1) / units, mspq_engine::kMaxSplit, d / 64}));
        const int units2 = std::max(1, u * (d / 128));
        const int sp2 = std::max(1, std::min({(296 + units2 - 1) / units2, mspq_engine::kMaxSplit, m.f / 64}));
        CAPI_OK(mspq_moe_bf16_tc(sv.n_groups, sv.group_expert, sv.group_buf, sv.group_off, sv.entry_tok,
                                 sv.entry_group, E->xn, E->pool, E->S16, d, m.f, w, K, E->G, sp1, sp2, E->tcws,
                                 E->yv[l & 1], E->sc));
        ysp = sp2;
      }
      CAPI_OK(mspq_gate_topk(E->h, E->yv[(L - 1) & 1], E->sv[(L - 1) & 1].entry_of, E->wts_t, ysp,
                             (long long)w * K * d, E->gfinal, nullptr, E->xn, nullptr, nullptr, nullptr, nullptr,
                             nullptr, nullptr, nullptr, L, L, w, d, Ex, K, m.eps, E->sc));
      CAPI_OK(mspq_lm_head(E->xn, E->lm, w, m.V, d, E->logits, E->sc));
      CUDA_OK(cudaEventRecord(b, E->sc));
      CUDA_OK(cudaEventSynchronize(b));
      best = std::min(best, elapsed_s(a, b));
    }
    out.push_back({(double)w, best});
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(dgb);
  cudaFree(dids);
  return out;
}

double measure_pcie(mspq_engine* E) {
  const size_t bytes = std::min<size_t>(E->S16, 64u << 20);
  void* dbuf;
  CUDA_OK(cudaMalloc(&dbuf, bytes));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) CUDA_OK(cudaMemcpyAsync(dbuf, E->host, bytes, cudaMemcpyHostToDevice, E->sx));
  cudaEventRecord(a, E->sx);
  for (int i = 0; i < 8; ++i) CUDA_OK(cudaMemcpyAsync(dbuf, E->host, bytes, cudaMemcpyHostToDevice, E->sx));
  cudaEventRecord(b, E->sx);
  cudaEventSynchronize(b);
  const double bw = 8.0 * bytes / elapsed_s(a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(dbuf);
  return bw;
}

}  // namespace

// ============================================================================ configure
static void configure(mspq_engine* E, const std::string& text) {
  const auto& m = E->m;
  HostCfg c = parse_host_cfg(text);
  validate_host_cfg(c, m.K);
  if (c.entropy_weighted) fail(MSPQ_ERR_INVALID_CONFIG, "entropy_weighted_capacity needs a trace (replay only)");
  const int kcap = std::max(c.use_governor ? c.k_max : c.fixed_k, 1);
  if (kcap > E->o.kmax) fail(MSPQ_ERR_K_OUT_OF_RANGE, "k above the engine's kmax");
  E->caps.assign(m.L, (int)std::min<long>(c.cache_capacity, m.E));
  const long cap_total = c.mode == 0 ? (long)m.L * std::min<long>(c.cache_capacity, m.E)
                                     : std::min<long>(c.cache_capacity, (long)m.L * m.E);
  const int extra = E->o.slot_extra > 0 ? E->o.slot_extra : std::min(m.E, E->Tmax * m.K) + 4;
  const int nbuf = (int)cap_total + extra;
  if (nbuf > E->nbuf) {
    if (E->cache) mspq_cache_destroy(E->cache);
    if (E->pool) cudaFree(E->pool);
    E->pool = nullptr;
    E->cache = nullptr;
    CUDA_OK(cudaMalloc(&E->pool, (size_t)nbuf * E->S16));
    E->nbuf = nbuf;
    CAPI_OK(mspq_cache_create(m.L, m.E, m.K, E->Tmax - 1, nbuf, E->o.log_cap, &E->cache));
    CAPI_OK(mspq_cache_view_get(E->cache, &E->view));
    for (auto ev : E->ev_ready) cudaEventDestroy(ev);
    E->ev_ready.assign(nbuf, nullptr);
    for (auto& ev : E->ev_ready) CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    for (size_t st = 0; st < E->gexec_s.size(); ++st) {
      cudaGraphExecDestroy(E->gexec_s[st]);
      cudaGraphDestroy(E->graph_s[st]);
    }
    E->gexec_s.clear();
    E->graph_s.clear();
    E->gexec = nullptr;
    for (int st = 0; st < E->S; ++st) {  // one draft graph per request stream (its state, its KV cache)
      E->gexec_s.push_back(nullptr);
      E->use_stream(st);
      E->gexec = nullptr;
      capture_draft_graph(E);
      E->gexec_s[st] = E->gexec;
      E->graph_s.push_back(E->graph);
    }
    E->use_stream(0);
  }
  E->ready_rec.assign(E->nbuf, 0);
  E->elb_freq.assign((size_t)m.L * m.E, (double)m.K / m.E);  // uniform prior: K of E experts per token
  E->res_host.assign((size_t)m.L * m.E, -1);                  // mspq_cache_configure empties the cache
  E->elb_calib.assign((size_t)E->o.kmax + 1, 1.0);
  E->gov_accept.clear();
  E->gov_g = -1.0;
  E->last_cycle.assign(E->nbuf, -1);
  E->last_layer.assign(E->nbuf, -1);
  CAPI_OK(mspq_cache_configure(E->cache, c.mode, c.policy, E->caps.data(), (int)std::min<long>(c.cache_capacity, (long)m.L * m.E),
                               c.budget, c.f1, c.f2, E->sc));
  CUDA_OK(cudaStreamSynchronize(E->sc));
  // ---- HardwareProfile re-fit on this B200 (unless the config pins one)
  if (E->pcie_bw_measured == 0.0) E->pcie_bw_measured = measure_pcie(E);
  if (E->draft_step_s == 0.0) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int32_t init[3] = {0, 0, 0};
    CUDA_OK(cudaMemcpyAsync(E->dst, init, sizeof(init), cudaMemcpyHostToDevice, E->sc));
    for (int i = 0; i < 2; ++i) CUDA_OK(cudaGraphLaunch(E->gexec, E->sc));
    int32_t z[3] = {0, 0, 0};
    CUDA_OK(cudaMemcpyAsync(E->dst, z, sizeof(z), cudaMemcpyHostToDevice, E->sc));
    cudaEventRecord(a, E->sc);
    for (int i = 0; i < 4; ++i) CUDA_OK(cudaGraphLaunch(E->gexec, E->sc));
    cudaEventRecord(b, E->sc);
    CUDA_OK(cudaEventSynchronize(b));
    E->draft_step_s = elapsed_s(a, b) / 4.0;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  if (E->home && E->home_bw_measured == 0.0) {
    // peer tier: a fetch is an HBM -> HBM copy of the bf16 tile images from a home region
    // (measured on this GPU's own home; a peer's over NVLink is not measurable on one GPU)
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int nb = std::min(E->nbuf, 8);
    for (int i = 0; i < nb; ++i)
      CUDA_OK(cudaMemcpyAsync(E->pool + (size_t)i * E->S16, E->home, E->S16, cudaMemcpyDeviceToDevice, E->sx));
    cudaEventRecord(a, E->sx);
    for (int i = 0; i < nb; ++i)
      CUDA_OK(cudaMemcpyAsync(E->pool + (size_t)i * E->S16, E->home, E->S16, cudaMemcpyDeviceToDevice, E->sx));
    cudaEventRecord(b, E->sx);
    CUDA_OK(cudaEventSynchronize(b));
    E->home_bw_measured = (double)nb * E->S16 / elapsed_s(a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
  if (E->pcie_fixed.second < 0.0) E->pcie_fixed = measure_pcie_fixed(E);
  if (E->verify_measured.empty()) E->verify_measured = measure_verify(E);
  if (!c.profile_given) {
    Profile p;
    p.pcie_bandwidth = E->home ? E->home_bw_measured : E->pcie_bw_measured;
    p.pcie_init_latency = E->home ? 0.0 : E->pcie_fixed.first;
    p.pcie_overhead = E->home ? 0.0 : E->pcie_fixed.second;
    // bytes one fetch puts on the link: the mean XC blob with the codec (raw tiles from a home)
    p.expert_size_bytes = E->home ? (uint64_t)E->S16
                                  : E->codec ? (uint64_t)(E->xc_bytes_total / E->n_payload) : (uint64_t)E->S16;
    p.draft_base = 0.0;
    p.draft_per_token = E->draft_step_s;
    // verify samples: timed target passes with the expected per-layer expert union resident
    p.verify_samples = E->verify_measured;
    if (p.verify_samples.size() < 2) {  // kmax < 4: extend linearly from the measured point(s)
      const double w0 = p.verify_samples.empty() ? 1.0 : p.verify_samples.back().first;
      const double t0 = p.verify_samples.empty() ? E->draft_step_s : p.verify_samples.back().second;
      p.verify_samples.push_back({w0 + 4.0, t0 * 1.5});
    }
    c.profile = p;
  }
  E->cfg = c;
  E->configured = true;
}

// ============================================================================ generate
struct CopyBatch {
  cudaEvent_t a = nullptr, b = nullptr;
  int count = 0;
  bool demand = false;  // a verify layer's demand misses (the reference's synchronous fetch)
  const char* label = "io_new";
};

// The controller's copy requests are on the critical path of the copy engine (a layer's demand
// fetches cannot start before the host has read them), so the host polls the event instead of
// sleeping in cudaEventSynchronize (the blocking-sync wake-up costs tens of microseconds).
static void spin_wait(cudaEvent_t ev) {
  for (;;) {
    const cudaError_t e = cudaEventQuery(ev);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) fail(MSPQ_ERR_CUDA, std::string("cudaEventQuery: ") + cudaGetErrorString(e));
  }
}

// one expert's bf16 tile images into dst: raw H2D on the copy stream, or the XC blob in chunks
// through a staging buffer and decoded as each chunk lands (the same pipeline as issue_copies)
static uint64_t copy_expert(mspq_engine* E, int key, unsigned char* dst) {
  if (const unsigned char* hs = E->home_src(key)) {  // peer tier: HBM -> HBM from the key's home
    cudaStream_t hst = E->codec ? E->sdec : E->sx;
    CUDA_OK(cudaMemcpyAsync(dst, hs, E->S16, cudaMemcpyDeviceToDevice, hst));
    return 0;  // no PCIe bytes
  }
  const unsigned char* hb = E->host_blob(E->payload(key));
  if (!E->codec) {
    CUDA_OK(cudaMemcpyAsync(dst, hb, E->S16, cudaMemcpyHostToDevice, E->sx));
    return (uint64_t)E->S16;
  }
  const uint32_t* toff = reinterpret_cast<const uint32_t*>(hb + 64);
  const int sb = E->stage_next;
  E->stage_next ^= 1;
  unsigned char* stg = E->stage[sb];
  if (E->stage_rec[sb]) CUDA_OK(cudaStreamWaitEvent(E->sx, E->ev_stage[sb], 0));
  const int nt = E->n_tiles;
  const int nm = std::max(1, std::min(8, (int)(toff[nt] / (24u << 20))));
  const int tail = nm > 1 ? nt / 32 : 0, nc = nm + (tail ? 1 : 0);
  for (int c = 0; c < nc; ++c) {
    const int t0 = c < nm ? (int)((int64_t)(nt - tail) * c / nm) : nt - tail;
    const int t1 = c < nm ? (int)((int64_t)(nt - tail) * (c + 1) / nm) : nt;
    const uint32_t b0 = c ? toff[t0] : 0u, b1 = toff[t1];
    CUDA_OK(cudaMemcpyAsync(stg + b0, hb + b0, b1 - b0, cudaMemcpyHostToDevice, E->sx));
    cudaEvent_t ev = E->pool_event();
    CUDA_OK(cudaEventRecord(ev, E->sx));
    CUDA_OK(cudaStreamWaitEvent(E->sdec, ev, 0));
    CAPI_OK(mspq_xc_decode(stg, t0, t1, dst, E->dec_ctas, E->sdec));
  }
  CUDA_OK(cudaEventRecord(E->ev_stage[sb], E->sdec));
  E->stage_rec[sb] = 1;
  return toff[nt];
}

static int issue_copies(mspq_engine* E, int cycle, CopyBatch& batch, uint64_t& bytes, bool prefetch = false,
                        const std::vector<std::pair<int, int>>* list = nullptr, int layer = -1) {
  cudaStream_t sx = E->sx, sdec = E->sdec;
  unsigned char** stage = E->stage;
  cudaEvent_t* ev_stage = E->ev_stage;
  char* stage_rec = E->stage_rec;
  int& stage_next = E->stage_next;
  const int n = list ? (int)list->size() : E->view.host_stat[S_NREQ];
  if (!list) {
    if (E->view.host_stat[S_OVERFLOW]) fail(MSPQ_ERR_OVERFLOW, "device controller ran out of buffers / queue");
    if (n > E->view.req_cap) fail(MSPQ_ERR_OVERFLOW, "copy request queue overflow");
  }
  // refetch_from_hbm: per request, the index in this list of the request that fills the key's
  // first-request buffer (-1 = filled before this list); a refetch may copy from it only after it
  std::vector<int>& fill_at = E->fill_at;
  if (layer >= 0 && E->cfg.refetch_from_hbm) {
    fill_at.assign(n, -1);
    for (int i = 0; i < n; ++i) {
      const int key = E->view.host_req[i * 3];
      if (key / E->m.E == layer && E->view.host_req[i * 3 + 1] == E->view.host_sched[1 + key % E->m.E])
        fill_at[i] = i;
    }
  }
  auto filled_before = [&](int i, int key, int b0) {
    for (int j = 0; j < n; ++j)
      if (fill_at[j] >= 0 && E->view.host_req[j * 3] == key && E->view.host_req[j * 3 + 1] == b0) return j < i;
    return true;
  };
  for (int i = 0; i < n; ++i) {
    const int key = list ? (*list)[i].first : E->view.host_req[i * 3];
    const int buf = list ? (*list)[i].second : E->view.host_req[i * 3 + 1];
    if (buf < 0 || buf >= E->nbuf) fail(MSPQ_ERR_OVERFLOW, "invalid slot buffer");
    if (prefetch && !list && E->pf_defer && key / E->m.E >= 1) {
      E->deferred.push_back({key, buf});
      continue;
    }
    if (!batch.a) {
      batch.a = E->pool_event();
      CUDA_OK(cudaEventRecord(batch.a, sx));
    }
    const bool reused = E->last_cycle[buf] == cycle;  // the slot's last reader is this cycle's GEMM
    unsigned char* slot = E->pool + (size_t)buf * E->S16;
    if (layer >= 0 && key / E->m.E == layer && E->cfg.refetch_from_hbm) {
      // evicted and requested again inside this verify layer: the key's first-request buffer
      // (host_sched, published by the controller with this request list) is parked until the
      // layer's GEMM has read it (ctl.cu erase), so it still holds the expert -- copy it HBM -> HBM
      // on the writer lane, in order after the write that filled it.  Same decision, no link bytes.
      const int b0 = E->view.host_sched[1 + key % E->m.E];
      if (b0 >= 0 && b0 < E->nbuf && b0 != buf && !list && filled_before(i, key, b0)) {
        cudaStream_t w = E->codec ? sdec : sx;
        if (reused) CUDA_OK(cudaStreamWaitEvent(w, E->ev_gemm[E->last_layer[buf]], 0));
        if (E->ready_rec[b0]) CUDA_OK(cudaStreamWaitEvent(w, E->ev_ready[b0], 0));
        CUDA_OK(cudaMemcpyAsync(slot, E->pool + (size_t)b0 * E->S16, E->S16, cudaMemcpyDeviceToDevice, w));
        CUDA_OK(cudaEventRecord(E->ev_ready[buf], w));
        E->ready_rec[buf] = 1;
        ++E->n_refetch;
        ++batch.count;
        continue;
      }
    }
    if (const unsigned char* hs = E->home_src(key)) {
      // peer-expert tier: HBM -> HBM from the key's home region (a peer's over NVLink, or this
      // GPU's own), in the decode stream's order so it follows any earlier write into the slot
      cudaStream_t hst = E->codec ? sdec : sx;
      if (reused) CUDA_OK(cudaStreamWaitEvent(hst, E->ev_gemm[E->last_layer[buf]], 0));
      if (E->ready_rec[buf]) CUDA_OK(cudaStreamWaitEvent(hst, E->ev_ready[buf], 0));
      CUDA_OK(cudaMemcpyAsync(slot, hs, E->S16, cudaMemcpyDeviceToDevice, hst));
      CUDA_OK(cudaEventRecord(E->ev_ready[buf], hst));
      const int owner = (key % E->m.E) % E->peer_G;
      if (owner == E->peer_rank) {
        E->gen_home_local_bytes += (uint64_t)E->S16;
        ++E->n_home_local;
      } else {
        E->gen_peer_bytes += (uint64_t)E->S16;
        ++E->n_peer;
      }
      E->ready_rec[buf] = 1;
      ++batch.count;
      continue;
    }
    // two lanes: a slot may still be under a write issued on the other lane (a prefetch the
    // controller evicted before its use), so the new writer orders after it
    if (!E->codec) {
      if (reused) CUDA_OK(cudaStreamWaitEvent(sx, E->ev_gemm[E->last_layer[buf]], 0));
      CUDA_OK(cudaMemcpyAsync(slot, E->host_blob(E->payload(key)), E->S16, cudaMemcpyHostToDevice, sx));
      CUDA_OK(cudaEventRecord(E->ev_ready[buf], sx));
      bytes += (uint64_t)E->S16;
    } else {
      // compressed blob -> staging (copy engine, chunked) -> decode kernel -> slot.  Chunk c's
      // decode starts as soon as its bytes land, so only the last chunk's decode is exposed.
      const unsigned char* hb = E->host_blob(E->payload(key));
      const uint32_t* toff = reinterpret_cast<const uint32_t*>(hb + 64);
      const int sb = stage_next;
      stage_next ^= 1;
      unsigned char* stg = stage[sb];
      if (stage_rec[sb]) CUDA_OK(cudaStreamWaitEvent(sx, ev_stage[sb], 0));
      if (reused) CUDA_OK(cudaStreamWaitEvent(sdec, E->ev_gemm[E->last_layer[buf]], 0));
      const int nt = E->n_tiles;
      // ~24 MB chunks: a pinned H2D chunk pays a fixed start cost (tools/h2d_chunks.py: 54.9 GB/s at
      // 4 x 25 MB vs 53.6 at 16 x 6 MB), while the exposed tail is one tile per decode warp either way
      // The last chunk is a small one (1/32 of the tiles), so less decode work is left once the link
      // goes quiet.
      const int nm = std::max(1, std::min(8, (int)(toff[nt] / (24u << 20))));
      const int tail = nm > 1 ? nt / 32 : 0, nc = nm + (tail ? 1 : 0);
      for (int c = 0; c < nc; ++c) {
        const int t0 = c < nm ? (int)((int64_t)(nt - tail) * c / nm) : nt - tail;
        const int t1 = c < nm ? (int)((int64_t)(nt - tail) * (c + 1) / nm) : nt;
        const uint32_t b0 = c ? toff[t0] : 0u, b1 = toff[t1];
        CUDA_OK(cudaMemcpyAsync(stg + b0, hb + b0, b1 - b0, cudaMemcpyHostToDevice, sx));
        cudaEvent_t ev = E->pool_event();
        CUDA_OK(cudaEventRecord(ev, sx));
        CUDA_OK(cudaStreamWaitEvent(sdec, ev, 0));
        CAPI_OK(mspq_xc_decode(stg, t0, t1, slot, E->dec_ctas, sdec));
      }
      CUDA_OK(cudaEventRecord(ev_stage[sb], sdec));
      stage_rec[sb] = 1;
      CUDA_OK(cudaEventRecord(E->ev_ready[buf], sdec));
      bytes += toff[nt];
    }
    E->ready_rec[buf] = 1;
    ++batch.count;
  }
  if (batch.a) {
    batch.b = E->pool_event();
    CUDA_OK(cudaEventRecord(batch.b, E->codec ? sdec : sx));
  }
  return n;
}

// Prefill of one prompt's tokens 0 .. n_prompt-2 (attention models): the target,
// layer-major over the whole prompt in chunks of up to 32 tokens, so their KV rows exist before the
// first cycle.  A prompt routes to (nearly) every expert of every layer, so each layer's E experts
// are streamed from the host store (or the peer tier's homes) into one of two layer buffers, two
// layers ahead of the compute, outside the capped cache (whose state the prefill leaves alone).
// Writes the KV rows of the engine's current stream (E->kcache / E->vcache).
static json run_prefill(mspq_engine* E, const int32_t* prompt, int n_prompt) {
  const auto& m = E->m;
  const int L = m.L, K = m.K, Ex = m.E, d = m.d;
  json prefill = json::object();
  const auto pw0 = std::chrono::steady_clock::now();
  const int n = n_prompt - 1, CH = 32, nch = (n + CH - 1) / CH;
  if (nch > L) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "prompt longer than 32 x layers tokens");
  const size_t plane = (size_t)mspq_engine::kMaxSplit * CH * K * d;  // floats per chunk planes
  if (!E->pf_buf[0]) {
    for (int i = 0; i < 2; ++i) {
      CUDA_OK(cudaMalloc(&E->pf_buf[i], (size_t)Ex * E->S16));
      CUDA_OK(cudaEventCreateWithFlags(&E->pf_ready[i], cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&E->pf_done[i], cudaEventDisableTiming));
    }
    std::vector<int32_t> idn(Ex);
    for (int e = 0; e < Ex; ++e) idn[e] = e;
    CUDA_OK(cudaMalloc(&E->pf_gbuf, Ex * 4));
    CUDA_OK(cudaMemcpy(E->pf_gbuf, idn.data(), Ex * 4, cudaMemcpyHostToDevice));
  }
  if (n > E->pf_n) {
    for (float* p : {E->pf_h, E->pf_y[0], E->pf_y[1]})
      if (p) cudaFree(p);
    CUDA_OK(cudaMalloc(&E->pf_h, (size_t)n * d * 4));
    CUDA_OK(cudaMalloc(&E->pf_y[0], (size_t)nch * plane * 4));
    CUDA_OK(cudaMalloc(&E->pf_y[1], (size_t)nch * plane * 4));
    if (E->pf_eo) cudaFree(E->pf_eo);
    CUDA_OK(cudaMalloc(&E->pf_eo, (size_t)nch * CH * K * 4 * 2));
    E->pf_n = n;
  }
  std::vector<int32_t> pos_all(n), tok_all(prompt, prompt + n);
  for (int i = 0; i < n; ++i) pos_all[i] = i;
  int32_t *d_tok = nullptr, *d_pos = nullptr;
  CUDA_OK(cudaMalloc(&d_tok, (size_t)n * 4));
  CUDA_OK(cudaMalloc(&d_pos, (size_t)n * 4));
  CUDA_OK(cudaMemcpyAsync(d_tok, tok_all.data(), (size_t)n * 4, cudaMemcpyHostToDevice, E->sc));
  CUDA_OK(cudaMemcpyAsync(d_pos, pos_all.data(), (size_t)n * 4, cudaMemcpyHostToDevice, E->sc));
  CAPI_OK(mspq_embed(E->embed, E->pos, d_tok, d_pos, n, d, E->pf_h, E->sc));
  uint64_t pf_bytes = 0;
  E->ev_pool_next = 0;
  auto stream_layer = [&](int l) {  // layer l's experts into buffer l & 1, after layer l-2's GEMMs
    const int bi = l & 1;
    if (l >= 2) {  // every stream that writes the buffer (copy; decode / home copies) waits for its readers
      CUDA_OK(cudaStreamWaitEvent(E->sx, E->pf_done[bi], 0));
      if (E->sdec) CUDA_OK(cudaStreamWaitEvent(E->sdec, E->pf_done[bi], 0));
    }
    for (int e = 0; e < Ex; ++e) pf_bytes += copy_expert(E, l * Ex + e, E->pf_buf[bi] + (size_t)e * E->S16);
    CUDA_OK(cudaEventRecord(E->pf_ready[bi], E->codec ? E->sdec : E->sx));
  };
  stream_layer(0);
  if (L > 1) stream_layer(1);
  std::vector<int> ysp_ch(nch, 1);
  for (int l = 0; l < L; ++l) {
    if (E->ev_pool_next > E->ev_pool.size() / 2 + 256) E->ev_pool_next = 0;  // events of finished layers
    bool waited = false;
    for (int c = 0; c < nch; ++c) {
      const int t0 = c * CH, T = std::min(CH, n - t0);
      float* hc = E->pf_h + (size_t)t0 * d;
      float* yprev = E->pf_y[(l - 1) & 1] + (size_t)c * plane;
      float* ycur = E->pf_y[l & 1] + (size_t)c * plane;
      Sched& sv = E->sv[c & 1];
      // attention block of chunk c (the residual lives in pf_h; E->h is the window workspace)
      CUDA_OK(cudaMemcpyAsync(E->h, hc, (size_t)T * d * 4, cudaMemcpyDeviceToDevice, E->sc));
      int32_t* eo_prev = E->pf_eo + ((size_t)((l - 1) & 1) * nch + c) * CH * K;
      int32_t* eo_cur = E->pf_eo + ((size_t)(l & 1) * nch + c) * CH * K;
      const int ysp = enqueue_attn(E, l, T, d_pos + t0, l ? yprev : nullptr, l ? eo_prev : nullptr,
                                   l ? E->wts_t + (size_t)c * CH * K : nullptr, ysp_ch[c], (long long)T * K * d,
                                   nullptr, E->sc);
      int32_t* ids = E->ids_t;  // [T][K] of this chunk
      CAPI_OK(mspq_gate_topk(E->h, E->oproj, nullptr, nullptr, ysp, (long long)T * d, E->gamma + (size_t)l * d,
                             E->router + (size_t)l * Ex * d, E->xn, ids, E->wts_t + (size_t)c * CH * K, nullptr,
                             nullptr, nullptr, nullptr, nullptr, l, L, T, d, Ex, K, m.eps, E->sc));
      CAPI_OK(mspq_build_schedule(ids, T, K, Ex, E->pf_gbuf, sv.n_groups, sv.group_expert, sv.group_buf,
                                  sv.group_off, sv.entry_tok, sv.entry_of, sv.entry_group, E->sc));
      if (!waited) {  // the layer's experts have landed
        CUDA_OK(cudaStreamWaitEvent(E->sc, E->pf_ready[l & 1], 0));
        waited = true;
      }
      const int G = std::min(Ex, T * K);
      const int units = std::max(1, G * (2 * m.f / 128));
      const int sp1 = std::max(1, std::min({(296 + units - 1) / units, mspq_engine::kMaxSplit, d / 64}));
      const int units2 = std::max(1, G * (d / 128));
      const int sp2 = std::max(1, std::min({(296 + units2 - 1) / units2, mspq_engine::kMaxSplit, m.f / 64}));
      CAPI_OK(mspq_moe_bf16_tc(sv.n_groups, sv.group_expert, sv.group_buf, sv.group_off, sv.entry_tok,
                               sv.entry_group, E->xn, E->pf_buf[l & 1], E->S16, d, m.f, T, K, E->G, sp1, sp2,
                               E->tcws, ycur, E->sc));
      CUDA_OK(cudaMemcpyAsync(hc, E->h, (size_t)T * d * 4, cudaMemcpyDeviceToDevice, E->sc));
      ysp_ch[c] = sp2;
      // the chunk's entry_of must survive until layer l+1's combine of this chunk (the Sched
      // double buffer holds two chunks); its routing weights stay at wts_t + c * 32 K
      CUDA_OK(cudaMemcpyAsync(eo_cur, sv.entry_of, (size_t)T * K * 4, cudaMemcpyDeviceToDevice, E->sc));
    }
    CUDA_OK(cudaEventRecord(E->pf_done[l & 1], E->sc));
    if (l + 2 < L) stream_layer(l + 2);
  }
  CUDA_OK(cudaStreamSynchronize(E->sc));
  CUDA_OK(cudaStreamSynchronize(E->sx));
  if (E->sdec) CUDA_OK(cudaStreamSynchronize(E->sdec));
  cudaFree(d_tok);
  cudaFree(d_pos);
  prefill["tokens"] = n;
  prefill["windows"] = nch;
  prefill["expert_copies"] = (uint64_t)L * Ex;
  prefill["h2d_bytes"] = pf_bytes;
  prefill["time_s"] = std::chrono::duration<double>(std::chrono::steady_clock::now() - pw0).count();
  return prefill;
}

static std::string generate(mspq_engine* E, const int32_t* prompt, int n_prompt, int max_new) {
  if (!E->configured) fail(MSPQ_ERR_INVALID_CONFIG, "engine not configured");
  if (n_prompt < 1) fail(MSPQ_ERR_EMPTY_RANGE, "empty prompt");
  const auto& m = E->m;
  const HostCfg& c = E->cfg;
  const Profile& prof = c.profile;
  const int L = m.L, K = m.K, Ex = m.E, d = m.d;
  if (n_prompt - 1 + max_new + E->Tmax >= m.P) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "positions exceed the positional table");
  for (int i = 0; i < n_prompt; ++i)
    if (prompt[i] < 0 || prompt[i] >= m.V) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "prompt token out of vocab");
  const int level = E->o.trace_level;
  int head_pos = n_prompt - 1;
  // device decode state
  E->hpin[0] = 0;
  E->hpin[1] = prompt[n_prompt - 1];
  E->hpin[2] = head_pos;
  CUDA_OK(cudaMemcpyAsync(E->dst, E->hpin, 12, cudaMemcpyHostToDevice, E->sc));
  CUDA_OK(cudaMemcpyAsync(E->win_tok(), E->hpin + 1, 4, cudaMemcpyHostToDevice, E->sc));
  const int kcap = std::max(c.use_governor ? c.k_max : c.fixed_k, 1);
  if (E->gov_accept.empty()) E->gov_accept.assign(kcap, c.initial_accept);
  if (E->gov_g < 0.0) E->gov_g = static_cast<double>(L) * static_cast<double>(K);
  std::vector<double>& accept = E->gov_accept;
  double& g = E->gov_g;
  // |E_new(k)| for the governor.  linear (reference, sim.cpp:75-78): g*k with g = fetched/k of the
  // last cycle.  elb: the ELB analysed against the current cache state -- per layer,
  // every non-resident expert e is fetched if any of the k+1 window tokens routes to it, which the
  // ELB's per-(layer, expert) frequency p puts at 1-(1-p)^(k+1); summed over layers.  A per-k
  // factor (EMA of fetched / estimate for the k last run at) absorbs what the union misses: at
  // small caps the planner's prefetches evict experts the window still needs, and they come back
  // on demand (Phi cap 4/16: ~2x the union at k = 16).
  auto elb_raw = [E, Ex, L](int k) {
    double s = 0.0;
    for (int i = 0; i < L * Ex; ++i)
      if (E->res_host[i] < 0) s += 1.0 - std::pow(1.0 - E->elb_freq[i], static_cast<double>(k + 1));
    return s;
  };
  auto est = [&]() {
    if (c.estimator == 1)
      return Est([E, elb_raw](int k) { return static_cast<int>(std::llround(E->elb_calib[k] * elb_raw(k))); });
    return Est([gg = g](int k) { return static_cast<int>(std::llround(gg * static_cast<double>(k))); });
  };
  int k_slo = c.k_slo;
  if (c.use_governor && c.ttft_budget > 0.0) k_slo = std::min(k_slo, k_slo_from_ttft(prof, c.ttft_budget, est(), c.k_min, c.k_max));
  CUDA_OK(cudaEventRecord(E->ev_t0, E->sc));
  CUDA_OK(cudaStreamWaitEvent(E->sx, E->ev_t0, 0));
  E->pf_defer = c.prefetch_defer && c.mode == 0;  // run-config "prefetch_defer" (default on)
  E->deferred.clear();
  E->hcap_v_hist.clear();
  E->hcap_d_hist.clear();
  E->hmid_v_hist.clear();
  E->hmid_d_hist.clear();
  E->gen_peer_bytes = E->gen_home_local_bytes = 0;
  E->n_peer = E->n_home_local = 0;
  E->n_refetch = 0;
  std::vector<int> committed;
  json cycles = json::array();
  double stall_total = 0.0, layer_cov_total = 0.0, step_cov_total = 0.0;
  uint64_t h2d_bytes = 0, total_new = 0, layer_cov_count = 0, step_total = 0, acc_total = 0;
  const auto wall0 = std::chrono::steady_clock::now();
  int ci = 0;
  // trace_level >= 1: the committed positions of the reference trace this run exports
  // (to_reference_trace): target routing + the draft's routing of the same token
  std::vector<std::vector<int>> an_target, an_draft;  // [pos][L*K]
  long k3_groups = 0, draft_steps = 0;
  double k3_time = 0.0, k3_bytes = 0.0, draft_time = 0.0;
  // verify layers of one window of T tokens (positions head .. head+T-1 in E->win_pos(), tokens
  // in E->win_tok(), residual embedded in E->h): per layer [attention] -> K1 route -> controller
  // verify step -> copies -> K3.  Also runs prefill chunks (prefill: no captures / plans).
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> stall_ev;
  long launches = 0;
  std::vector<int> layer_groups(L, 0);
  auto verify_layers = [&](int T, int cycle, bool prefill, std::vector<CopyBatch>& batches, uint64_t& cyc_bytes) {
    for (int l = 0; l < L; ++l) {
      const int pl = (l - 1) & 1;
      int32_t* tgt = E->ids_t + (size_t)l * T * K;
      const float* y = l ? E->yv[pl] : nullptr;
      const int32_t* eo = l ? E->sv[pl].entry_of : nullptr;
      const float* pw = l ? E->wts_t + (size_t)(l - 1) * T * K : nullptr;
      int ysp = E->yv_splits[pl];
      long long yst = (long long)T * K * d;
      const bool cap = E->hcap_v && !prefill;
      if (E->attn) {
        ysp = enqueue_attn(E, l, T, E->win_pos(), y, eo, pw, ysp, yst, cap ? E->hcap_v + (size_t)l * T * d : nullptr,
                           E->sc);
        y = E->oproj;
        eo = nullptr;
        pw = nullptr;
        yst = (long long)T * d;
        launches += 4;
      }
      CAPI_OK(mspq_gate_topk(E->h, y, eo, pw, ysp, yst, E->gamma + (size_t)l * d,
                             E->router + (size_t)l * Ex * d, E->xn, tgt, E->wts_t + (size_t)l * T * K, nullptr, nullptr,
                             nullptr, nullptr, nullptr, l, L, T, d, Ex, K, m.eps, E->sc));
      Sched& sv = E->sv[l & 1];
      if (cap && E->attn)
        CUDA_OK(cudaMemcpyAsync(E->hmid_v + (size_t)l * T * d, E->h, (size_t)T * d * 4, cudaMemcpyDeviceToDevice, E->sc));
      else if (cap)
        CUDA_OK(cudaMemcpyAsync(E->hcap_v + (size_t)l * T * d, E->h, (size_t)T * d * 4, cudaMemcpyDeviceToDevice, E->sc));
      if (level >= 1) CUDA_OK(cudaEventRecord(E->ev_rt[l], E->sc));
      CAPI_OK(mspq_cache_verify_layer(E->cache, l, T, tgt, E->gbuf, E->sc));
      CUDA_OK(cudaEventRecord(E->ev_w0[l], E->sc));
      CAPI_OK(mspq_build_schedule(tgt, T, K, Ex, E->gbuf, sv.n_groups, sv.group_expert, sv.group_buf, sv.group_off,
                                  sv.entry_tok, sv.entry_of, sv.entry_group, E->sc));
      if (c.collect_plans && !prefill)
        CUDA_OK(cudaMemcpyAsync(E->sched_cap + (size_t)l * Sched::ints(E->G, E->N), sv.base,
                                Sched::ints(E->G, E->N) * 4, cudaMemcpyDeviceToDevice, E->sc));
      spin_wait(E->ev_w0[l]);
      CopyBatch b;
      b.label = "io_new";
      b.demand = true;
      issue_copies(E, cycle, b, cyc_bytes, false, nullptr, l);
      if (b.count) batches.push_back(b);
      if (!E->deferred.empty()) {
        // deferred plan prefetches for layer l+1 go right behind layer l's demand copies; when l+1
        // has none, the earliest remaining layer's are pulled forward so the boundary stays covered
        int lim = l + 1;
        bool any = false;
        for (auto& kb : E->deferred) any |= kb.first / Ex <= lim;
        if (!any) {
          lim = L;
          for (auto& kb : E->deferred) lim = std::min(lim, kb.first / Ex);
        }
        std::vector<std::pair<int, int>> now, keep;
        for (auto& kb : E->deferred) (kb.first / Ex <= lim ? now : keep).push_back(kb);
        E->deferred.swap(keep);
        CopyBatch bp;
        issue_copies(E, cycle, bp, cyc_bytes, true, &now);
        if (bp.count) batches.push_back(bp);
      }
      // the layer's groups (ascending expert = the device schedule's order) split into experts
      // already resident (part A: their GEMM runs while the copies are still on the link) and
      // experts whose copy is in flight (part B: after a stream wait on their ready events)
      std::vector<int>& gb = E->layer_bufs;
      gb.clear();
      for (int e = 0; e < Ex; ++e)
        if (E->view.host_sched[1 + e] >= 0) gb.push_back(E->view.host_sched[1 + e]);
      const int ng = (int)gb.size();
      uint32_t mA[8] = {0, 0, 0, 0, 0, 0, 0, 0}, mB[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      std::vector<int> pend;
      for (int gi = 0; gi < ng; ++gi) {
        const int buf = gb[gi];
        if (buf < 0 || buf >= E->nbuf) fail(MSPQ_ERR_OVERFLOW, "schedule buffer out of range");
        bool pending = false;
        if (E->ready_rec[buf]) {
          if (cudaEventQuery(E->ev_ready[buf]) == cudaErrorNotReady) pending = true;
          else E->ready_rec[buf] = 0;
        }
        if (pending) pend.push_back(buf);
        if (gi < 256) (pending ? mB : mA)[gi >> 5] |= 1u << (gi & 31);
      }
      // K splits so each tcgen05 GEMM has >= ~2 CTAs per SM
      auto pick_split = [&](int rows, int kdim) {
        const int units = std::max(1, ng * (rows / 128));
        int sp = (296 + units - 1) / units;
        return std::max(1, std::min({sp, mspq_engine::kMaxSplit, kdim / 64}));
      };
      const int sp1 = pick_split(2 * m.f, d), sp2 = pick_split(d, m.f);
      E->yv_splits[l & 1] = sp2;
      const bool parts = c.verify_overlap && !pend.empty() && (int)pend.size() < ng && ng <= 256;
      E->layer_parts[l] = parts ? 1 : 0;
      if (!parts && !pend.empty()) {  // everything waits
        for (int buf : pend) CUDA_OK(cudaStreamWaitEvent(E->sc, E->ev_ready[buf], 0));
        CUDA_OK(cudaEventRecord(E->ev_w1[l], E->sc));
        stall_ev.push_back({E->ev_w0[l], E->ev_w1[l]});
      }
      CUDA_OK(cudaEventRecord(E->ev_k0[l], E->sc));
      if (!parts) {
        CAPI_OK(mspq_moe_bf16_tc(sv.n_groups, sv.group_expert, sv.group_buf, sv.group_off, sv.entry_tok,
                                 sv.entry_group, E->xn, E->pool, E->S16, d, m.f, T, K, E->G, sp1, sp2, E->tcws,
                                 E->yv[l & 1], E->sc));
      } else {
        CAPI_OK(mspq_moe_bf16_tc_part(sv.n_groups, sv.group_expert, sv.group_buf, sv.group_off, sv.entry_tok,
                                      sv.entry_group, E->xn, E->pool, E->S16, d, m.f, T, K, E->G, sp1, sp2, E->tcws,
                                      E->yv[l & 1], mA, 1, E->sc));
        CUDA_OK(cudaEventRecord(E->ev_ka1[l], E->sc));
        for (int buf : pend) CUDA_OK(cudaStreamWaitEvent(E->sc, E->ev_ready[buf], 0));
        CUDA_OK(cudaEventRecord(E->ev_w1[l], E->sc));
        stall_ev.push_back({E->ev_ka1[l], E->ev_w1[l]});
        CAPI_OK(mspq_moe_bf16_tc_part(sv.n_groups, sv.group_expert, sv.group_buf, sv.group_off, sv.entry_tok,
                                      sv.entry_group, E->xn, E->pool, E->S16, d, m.f, T, K, E->G, sp1, sp2, E->tcws,
                                      E->yv[l & 1], mB, 0, E->sc));
        launches += 3;
      }
      CUDA_OK(cudaEventRecord(E->ev_gemm[l], E->sc));
      launches += 7;  // gate_topk, verify_layer, schedule, gather, 2 x tcgen05 GEMM, finalize
      layer_groups[l] = ng;
      for (int gi = 0; gi < ng; ++gi) {
        const int buf = gb[gi];
        E->last_cycle[buf] = cycle;
        E->last_layer[buf] = l;
      }
    }
  };
  // ---------------- prefill (attention models): the prompt's tokens 0 .. n_prompt-2 through the
  // target, layer-major over the whole prompt in chunks of up to 32 tokens, so their KV rows exist
  // before the first cycle.  A prompt routes to (nearly) every expert of every layer, so the
  // prefill streams each layer's E experts from the host store into one of two layer buffers,
  // two layers ahead of the compute, outside the capped cache (whose state the prefill leaves
  // alone) -- each expert crosses the link once instead of once per window slot.  Its time is
  // reported apart from the decode metric (TTFT vs TPOT).
  json prefill = json::object();
  if (E->attn && n_prompt > 1) {
    prefill = run_prefill(E, prompt, n_prompt);
    // the decode state (head token / position) the prefill's embed left alone, and the decode's clock
    CUDA_OK(cudaEventRecord(E->ev_t0, E->sc));  // the decode's clock starts after the prefill
    CUDA_OK(cudaStreamWaitEvent(E->sx, E->ev_t0, 0));
    if (E->sdec) CUDA_OK(cudaStreamWaitEvent(E->sdec, E->ev_t0, 0));
  }
  const auto wall_dec0 = std::chrono::steady_clock::now();
  while ((int)committed.size() < max_new) {
    const int rem = max_new - (int)committed.size();
    const int cycle = ++E->cycle_serial;
    E->ev_pool_next = 0;
    const int kk = c.use_governor ? select_k(prof, accept, c.k_min, c.k_max, k_slo, est()) : c.fixed_k;
    const int k = std::max(1, std::min({kk, rem, E->o.kmax}));
    const int T = k + 1;
    const int est_new = c.use_governor ? est()(k) : -1;
    const uint64_t refetch0 = E->n_refetch;
    const double est_raw = c.estimator == 1 ? elb_raw(k) : 0.0;
    uint64_t cyc_bytes = 0;
    std::vector<CopyBatch> batches;
    // ---------------- draft + planner
    CUDA_OK(cudaEventRecord(E->ev_c0, E->sc));
    CUDA_OK(cudaMemsetAsync(E->dst, 0, 4, E->sc));  // row = 0
    CAPI_OK(mspq_cache_begin_cycle(E->cache, k, E->sc));
    CUDA_OK(cudaEventRecord(E->ev_g0[0], E->sc));
    CUDA_OK(cudaGraphLaunch(E->gexec, E->sc));
    CUDA_OK(cudaEventRecord(E->ev_g1[0], E->sc));
    if (E->hcap_d) CUDA_OK(cudaMemcpyAsync(E->hcap_d, E->hcap_dstage, (size_t)(L + 1) * d * 4, cudaMemcpyDeviceToDevice, E->sc));
    if (E->hmid_d) CUDA_OK(cudaMemcpyAsync(E->hmid_d, E->hmid_dstage, (size_t)L * d * 4, cudaMemcpyDeviceToDevice, E->sc));
    launches += E->graph_nodes;
    for (int i = 0; i < k; ++i) {
      CAPI_OK(mspq_cache_plan_row(E->cache, i, E->sc));
      CUDA_OK(cudaEventRecord(E->ev_row[i], E->sc));
      ++launches;
      if (i + 1 < k) {
        CUDA_OK(cudaEventRecord(E->ev_g0[i + 1], E->sc));
        CUDA_OK(cudaGraphLaunch(E->gexec, E->sc));
        CUDA_OK(cudaEventRecord(E->ev_g1[i + 1], E->sc));
        if (E->hcap_d)
          CUDA_OK(cudaMemcpyAsync(E->hcap_d + (size_t)(i + 1) * (L + 1) * d, E->hcap_dstage, (size_t)(L + 1) * d * 4,
                                  cudaMemcpyDeviceToDevice, E->sc));
        if (E->hmid_d)
          CUDA_OK(cudaMemcpyAsync(E->hmid_d + (size_t)(i + 1) * L * d, E->hmid_dstage, (size_t)L * d * 4,
                                  cudaMemcpyDeviceToDevice, E->sc));
        launches += E->graph_nodes;
      }
      spin_wait(E->ev_row[i]);
      CopyBatch b;
      issue_copies(E, cycle, b, cyc_bytes, true);
      if (b.count) batches.push_back(b);
    }
    CUDA_OK(cudaEventRecord(E->ev_dend, E->sc));
    // ---------------- verify (layer-major)
    for (int s = 0; s < T; ++s) E->hpin[s] = head_pos + s;
    CUDA_OK(cudaMemcpyAsync(E->win_pos(), E->hpin, T * 4, cudaMemcpyHostToDevice, E->sc));
    CAPI_OK(mspq_embed(E->embed, E->pos, E->win_tok(), E->win_pos(), T, d, E->h, E->sc));
    double stall = 0.0;
    int demand_total = 0;
    stall_ev.clear();
    verify_layers(T, cycle, false, batches, cyc_bytes);
    if (!E->deferred.empty()) fail(MSPQ_ERR_OVERFLOW, "deferred prefetch left at the end of the verify pass");
    const int pl = (L - 1) & 1;
    launches += 6;  // embed, final norm, lm head, argmax, accept, begin_cycle
    CAPI_OK(mspq_gate_topk(E->h, E->yv[pl], E->sv[pl].entry_of, E->wts_t + (size_t)(L - 1) * T * K, E->yv_splits[pl],
                           (long long)T * K * d, E->gfinal, nullptr,
                           E->xn, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, L, L, T, d, Ex, K, m.eps,
                           E->sc));
    if (E->hcap_v)
      CUDA_OK(cudaMemcpyAsync(E->hcap_v + (size_t)L * T * d, E->h, (size_t)T * d * 4, cudaMemcpyDeviceToDevice, E->sc));
    CAPI_OK(mspq_lm_head(E->xn, E->lm, T, m.V, d, E->logits, E->sc));
    CAPI_OK(mspq_argmax(E->logits, T, m.V, E->amax, E->sc));
    CAPI_OK(mspq_accept_advance(E->win_tok() + 1, E->amax, k, E->dst + 3, E->dst + 1, E->dst + 2, head_pos, E->sc));
    // next head = bonus
    CUDA_OK(cudaMemcpyAsync(E->win_tok(), E->dst + 1, 4, cudaMemcpyDeviceToDevice, E->sc));
    // results back: accepted, bonus, window tokens, target argmax (+ traces)
    int32_t* hp = E->hpin;
    size_t o = 0;
    const size_t o_res = o;
    CUDA_OK(cudaMemcpyAsync(hp + o, E->dst + 3, 8, cudaMemcpyDeviceToHost, E->sc));
    o += 2;
    const size_t o_win = o;
    CUDA_OK(cudaMemcpyAsync(hp + o, E->dst + 8 + 1, k * 4, cudaMemcpyDeviceToHost, E->sc));  // draft tokens
    o += k;
    const size_t o_am = o;
    CUDA_OK(cudaMemcpyAsync(hp + o, E->amax, T * 4, cudaMemcpyDeviceToHost, E->sc));
    o += T;
    const size_t o_cov = o;
    CUDA_OK(cudaMemcpyAsync(hp + o, E->view.cov, (size_t)L * 8, cudaMemcpyDeviceToHost, E->sc));
    o += (size_t)L * 2;
    const size_t o_step = o;
    CUDA_OK(cudaMemcpyAsync(hp + o, E->view.step, (size_t)L * T * 8, cudaMemcpyDeviceToHost, E->sc));
    o += (size_t)L * T * 2;
    const size_t o_tr = o;
    if (level >= 1) {
      CUDA_OK(cudaMemcpyAsync(hp + o, E->ids_t, (size_t)L * T * K * 4, cudaMemcpyDeviceToHost, E->sc));
      o += (size_t)L * T * K;
      CUDA_OK(cudaMemcpyAsync(hp + o, E->view.elb_ids, (size_t)k * L * K * 4, cudaMemcpyDeviceToHost, E->sc));
      o += (size_t)k * L * K;
      CUDA_OK(cudaMemcpyAsync(hp + o, E->view.elb_gates, (size_t)k * L * K * 4, cudaMemcpyDeviceToHost, E->sc));
      o += (size_t)k * L * K;
    }
    const size_t o_res_tab = o;
    if (c.estimator == 1) {  // residency snapshot + this cycle's ELB rows for the elb estimator
      CUDA_OK(cudaMemcpyAsync(hp + o, E->view.res, (size_t)L * Ex * 4, cudaMemcpyDeviceToHost, E->sc));
      o += (size_t)L * Ex;
      CUDA_OK(cudaMemcpyAsync(hp + o, E->view.elb_ids, (size_t)k * L * K * 4, cudaMemcpyDeviceToHost, E->sc));
      o += (size_t)k * L * K;
    }
    CUDA_OK(cudaEventRecord(E->ev_end, E->sc));
    CUDA_OK(cudaEventSynchronize(E->ev_end));
    if (E->hcap_v) {
      std::vector<float> hv((size_t)(L + 1) * T * d), hd((size_t)k * (L + 1) * d);
      CUDA_OK(cudaMemcpy(hv.data(), E->hcap_v, hv.size() * 4, cudaMemcpyDeviceToHost));
      CUDA_OK(cudaMemcpy(hd.data(), E->hcap_d, hd.size() * 4, cudaMemcpyDeviceToHost));
      E->hcap_v_hist.push_back(std::move(hv));
      E->hcap_d_hist.push_back(std::move(hd));
      if (E->hmid_v) {
        std::vector<float> mv((size_t)L * T * d), md((size_t)k * L * d);
        CUDA_OK(cudaMemcpy(mv.data(), E->hmid_v, mv.size() * 4, cudaMemcpyDeviceToHost));
        CUDA_OK(cudaMemcpy(md.data(), E->hmid_d, md.size() * 4, cudaMemcpyDeviceToHost));
        E->hmid_v_hist.push_back(std::move(mv));
        E->hmid_d_hist.push_back(std::move(md));
      }
    }
    const int fetched = E->view.host_stat[S_FETCHED], demand = E->view.host_stat[S_DEMAND];
    const int n_log = E->view.host_stat[S_NLOG];
    for (auto& [a, b] : stall_ev) stall += elapsed_s(a, b);
    for (int l = 0; l < L; ++l) {  // K3 device time, the stream wait between the two parts excluded
      const double t = E->layer_parts[l] ? elapsed_s(E->ev_k0[l], E->ev_ka1[l]) + elapsed_s(E->ev_w1[l], E->ev_gemm[l])
                                         : elapsed_s(E->ev_k0[l], E->ev_gemm[l]);
      k3_time += t;
      k3_bytes += (double)layer_groups[l] * E->S16;
      k3_groups += layer_groups[l];
    }
    for (int i = 0; i < k; ++i) draft_time += elapsed_s(E->ev_g0[i], E->ev_g1[i]);
    draft_steps += k;
    const int accepted = hp[o_res], bonus_tok = hp[o_res + 1];
    std::vector<int> new_toks;
    for (int i = 0; i < accepted; ++i) new_toks.push_back(hp[o_win + i]);
    new_toks.push_back(bonus_tok);
    if ((int)new_toks.size() > rem) new_toks.resize(rem);
    const int consumed = (int)new_toks.size();
    const int bonus = consumed > accepted ? 1 : 0;
    // ---- record (reference CycleRecord schema + measured extensions)
    json rec;
    rec["cycle"] = ci;
    rec["k"] = k;
    rec["accepted"] = consumed - bonus;
    rec["bonus"] = bonus;
    const double t_start = elapsed_s(E->ev_t0, E->ev_c0), t_dend = elapsed_s(E->ev_t0, E->ev_dend),
                 t_end = elapsed_s(E->ev_t0, E->ev_end);
    rec["start_s"] = t_start;
    rec["span_s"] = t_end - t_start;
    json cov = json::array();
    for (int l = 0; l < L; ++l) {
      const double v = static_cast<double>(hp[o_cov + l * 2]) / static_cast<double>(hp[o_cov + l * 2 + 1]);
      cov.push_back(v);
      layer_cov_total += v;
      ++layer_cov_count;
    }
    rec["coverage"] = cov;
    double sc_sum = 0.0;
    for (int s = 0; s < T; ++s)
      for (int l = 0; l < L; ++l)
        sc_sum += static_cast<double>(hp[o_step + (l * T + s) * 2]) / static_cast<double>(hp[o_step + (l * T + s) * 2 + 1]);
    rec["step_coverage"] = sc_sum / (T * L);
    rec["steps"] = T * L;
    rec["new_experts"] = fetched;
    rec["refetch_hbm"] = E->n_refetch - refetch0;
    if (c.use_governor) rec["est_new_experts"] = est_new;
    rec["bytes"] = cyc_bytes;
    rec["io_wait_s"] = stall;
    double sync_s = 0.0;
    json segs = json::array();
    segs.push_back(segment("compute", "draft", t_start, t_dend - t_start));
    int io_pending = 0;
    for (auto& b : batches) {
      // a mispredicted prefetch may still be on the copy/decode streams at ev_end: its batch is
      // left out of the segments (and counted) rather than read from an incomplete event
      if (cudaEventQuery(b.b) != cudaSuccess) {
        cudaGetLastError();
        ++io_pending;
        continue;
      }
      const double bs = elapsed_s(E->ev_t0, b.a), be = elapsed_s(E->ev_t0, b.b);
      segs.push_back(segment("io", b.label, bs, be - bs));
    }
    rec["io_pending_batches"] = io_pending;
    segs.push_back(segment("compute", "verify", t_dend, t_end - t_dend));
    // sync fetch = the demand misses' copy (+ decode) time, measured (sim.cpp:338-344 models it as
    // t_pcie_new(demand_count) queued after the channel traffic)
    for (auto& b : batches)
      if (b.demand && cudaEventQuery(b.b) == cudaSuccess) sync_s += elapsed_s(b.a, b.b);
    cudaGetLastError();
    rec["sync_fetch_s"] = sync_s;
    rec["sync_count"] = demand;
    rec["segments"] = segs;
    if (c.collect_plans) {  // sim.cpp:377-392: the device planner's items and the verify schedules
      const int np = std::min(E->view.host_stat[S_NPLAN], E->view.plan_cap);
      std::vector<int32_t> pl((size_t)np * 3);
      if (np) CUDA_OK(cudaMemcpy(pl.data(), E->view.plan, pl.size() * 4, cudaMemcpyDeviceToHost));
      json pj = json::array();
      for (int i = 0; i < np; ++i)
        pj.push_back({{"issue_after_token", pl[i * 3]}, {"layer", pl[i * 3 + 1] / Ex}, {"expert", pl[i * 3 + 1] % Ex},
                      {"phase", pl[i * 3 + 2]}});
      rec["prefetch_plan"] = pj;
      const size_t si = Sched::ints(E->G, E->N);
      std::vector<int32_t> sc((size_t)L * si);
      CUDA_OK(cudaMemcpy(sc.data(), E->sched_cap, sc.size() * 4, cudaMemcpyDeviceToHost));
      json ej = json::array();
      for (int l = 0; l < L; ++l) {
        const int32_t* b = sc.data() + (size_t)l * si;
        const int ng = b[0];
        const int32_t *gexp = b + 4, *goff = b + 4 + 2 * E->G, *etok = goff + E->G + 1;
        json groups = json::array();
        for (int g2 = 0; g2 < ng; ++g2) {
          json toks = json::array();
          for (int i = goff[g2]; i < goff[g2 + 1]; ++i) toks.push_back(head_pos + etok[i]);
          groups.push_back({{"expert", gexp[g2]}, {"tokens", toks}});
        }
        ej.push_back({{"layer", l}, {"groups", groups}});
      }
      rec["execution_plan"] = ej;
    }
    rec["tokens"] = new_toks;
    if (level >= 1) {
      json dt = json::array(), ta = json::array();
      for (int i = 0; i < k; ++i) dt.push_back(hp[o_win + i]);
      for (int s = 0; s < T; ++s) ta.push_back(hp[o_am + s]);
      rec["draft_tokens"] = dt;
      rec["target_argmax"] = ta;
      json tgt = json::array();  // [slot][layer][K]
      for (int s = 0; s < T; ++s) {
        json sl = json::array();
        for (int l = 0; l < L; ++l) {
          json c2 = json::array();
          for (int j = 0; j < K; ++j) c2.push_back(hp[o_tr + ((size_t)l * T + s) * K + j]);
          sl.push_back(c2);
        }
        tgt.push_back(sl);
      }
      rec["target"] = tgt;
      const size_t o_e = o_tr + (size_t)L * T * K, o_g = o_e + (size_t)k * L * K;
      json elb = json::array(), gates = json::array();
      for (int r = 0; r < k; ++r) {
        json rl = json::array(), gl = json::array();
        for (int l = 0; l < L; ++l) {
          json c2 = json::array(), g2 = json::array();
          for (int j = 0; j < K; ++j) {
            c2.push_back(hp[o_e + ((size_t)r * L + l) * K + j]);
            float gv;
            memcpy(&gv, &hp[o_g + ((size_t)r * L + l) * K + j], 4);
            g2.push_back(gv);
          }
          rl.push_back(c2);
          gl.push_back(g2);
        }
        elb.push_back(rl);
        gates.push_back(gl);
      }
      rec["elb"] = elb;
      {  // positions this cycle commits to the exported trace: slot 0 (cycle > 0), slots 1..accepted
        const int acc_c = consumed - bonus;
        for (int s2 = (ci > 0 ? 0 : 1); s2 <= acc_c; ++s2) {
          std::vector<int> tg((size_t)L * K), dr((size_t)L * K);
          for (int l = 0; l < L; ++l)
            for (int j = 0; j < K; ++j) {
              tg[(size_t)l * K + j] = hp[o_tr + ((size_t)l * T + s2) * K + j];
              dr[(size_t)l * K + j] = s2 < k ? hp[o_e + ((size_t)s2 * L + l) * K + j] : tg[(size_t)l * K + j];
            }
          an_target.push_back(std::move(tg));
          an_draft.push_back(std::move(dr));
        }
      }
      rec["elb_gates"] = gates;
      // per verify layer (s from the run start): controller done, GEMM start (after any wait on
      // in-flight copies), GEMM end, K1 (route) done
      json lt = json::array();
      for (int l = 0; l < L; ++l)
        lt.push_back({elapsed_s(E->ev_t0, E->ev_w0[l]), elapsed_s(E->ev_t0, E->ev_k0[l]),
                      elapsed_s(E->ev_t0, E->ev_gemm[l]), elapsed_s(E->ev_t0, E->ev_rt[l])});
      rec["layer_times"] = lt;
    }
    if (level >= 2) {
      const int nl = std::min(n_log, E->view.log_cap);
      std::vector<int32_t> lg((size_t)nl * 6);
      if (nl) CUDA_OK(cudaMemcpy(lg.data(), E->view.log, (size_t)nl * 24, cudaMemcpyDeviceToHost));
      json lj = json::array();
      for (int i = 0; i < nl; ++i) {
        const int32_t* ev = &lg[(size_t)i * 6];
        lj.push_back({ev[0], ev[1], ev[2] / Ex, ev[2] % Ex, ev[3], ev[4] < 0 ? -1 : ev[4] / Ex,
                      ev[4] < 0 ? -1 : ev[4] % Ex, ev[5]});
      }
      rec["log"] = lj;
    }
    cycles.push_back(rec);
    // ---- governor state (sim.cpp:394-404 semantics on the live outcomes)
    std::vector<bool> outcomes;
    for (int i = 0; i < k; ++i) {
      const bool ok = i < accepted;
      outcomes.push_back(ok);
      if (!ok) break;
    }
    if (outcomes.size() > accept.size()) outcomes.resize(accept.size());
    accept = update_acceptance(accept, c.ema_alpha, outcomes);
    g = static_cast<double>(fetched) / static_cast<double>(k);
    if (c.estimator == 1) {
      constexpr double beta = 1.0 / 32.0;
      // calibrated against the fetches that crossed the link: an in-layer refetch served from HBM
      // (refetch_from_hbm) is exactly what the union model leaves out
      const double moved = static_cast<double>(fetched) - static_cast<double>(E->n_refetch - refetch0);
      if (est_raw > 0.0) E->elb_calib[k] = (1.0 - 0.25) * E->elb_calib[k] + 0.25 * (moved / est_raw);
      // per drafted row: p <- (1-beta) p + beta [e in row's top-K at layer l]
      const int32_t* rows = hp + o_res_tab + (size_t)L * Ex;
      for (int r = 0; r < k; ++r)
        for (int l = 0; l < L; ++l) {
          double* pl = &E->elb_freq[(size_t)l * Ex];
          for (int e = 0; e < Ex; ++e) pl[e] *= 1.0 - beta;
          for (int j = 0; j < K; ++j) {
            const int e = rows[((size_t)r * L + l) * K + j];
            if (e >= 0 && e < Ex) pl[e] += beta;
          }
        }
      std::copy(hp + o_res_tab, hp + o_res_tab + (size_t)L * Ex, E->res_host.begin());
    }
    stall_total += stall;
    step_cov_total += sc_sum;
    step_total += (uint64_t)T * L;
    acc_total += (uint64_t)(consumed - bonus);
    total_new += fetched;
    h2d_bytes += cyc_bytes;
    for (int t2 : new_toks) committed.push_back(t2);
    head_pos += accepted + 1;
    ++ci;
    demand_total += demand;
  }
  // everything (including trailing prefetches) has landed before we report
  CUDA_OK(cudaStreamSynchronize(E->sx));
  if (E->sdec) CUDA_OK(cudaStreamSynchronize(E->sdec));
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall0).count();
  json rep;
  const double total_time = cycles.empty() ? 0.0
                                           : cycles.back()["start_s"].get<double>() + cycles.back()["span_s"].get<double>();
  rep["total_tokens"] = committed.size();
  rep["total_time_s"] = total_time;
  rep["tpot_s"] = committed.empty() ? 0.0 : total_time / committed.size();
  rep["ttft_s"] = cycles.empty() ? 0.0 : cycles[0]["span_s"].get<double>();
  rep["mean_coverage"] = layer_cov_count ? layer_cov_total / layer_cov_count : 0.0;
  rep["mean_step_coverage"] = step_total ? step_cov_total / step_total : 0.0;
  rep["mean_accepted"] = cycles.empty() ? 0.0 : (double)acc_total / cycles.size();
  rep["stall_time_s"] = stall_total;
  rep["total_new_experts"] = total_new;
  rep["cycles"] = cycles;
  rep["tokens"] = committed;
  rep["h2d_bytes"] = h2d_bytes;
  rep["h2d_bytes_bf16"] = (uint64_t)total_new * (uint64_t)E->S16;
  rep["refetch_hbm"] = E->n_refetch;
  if (E->peer_G > 0) {  // peer-expert tier: where the fetched experts' bytes came from
    json pt;
    pt["group"] = E->peer_G;
    pt["rank"] = E->peer_rank;
    pt["peer_bytes"] = E->gen_peer_bytes;
    pt["home_local_bytes"] = E->gen_home_local_bytes;
    pt["peer_fetches"] = E->n_peer;
    pt["home_local_fetches"] = E->n_home_local;
    pt["pcie_fetches"] = (uint64_t)total_new - E->n_peer - E->n_home_local - E->n_refetch;
    rep["peer_tier"] = pt;
  }
  rep["expert_codec"] = E->codec ? "xc" : "none";
  if (!an_target.empty()) {
    // draft -> target routing fidelity and per-layer routing entropy of the run
    // (classify_fidelity / layer_entropy, trace.cpp:401-462, on the exported trace's positions)
    auto cell = [&](size_t p, int l) {
      std::vector<int> a(an_target[p].begin() + (size_t)l * K, an_target[p].begin() + (size_t)(l + 1) * K);
      std::vector<int> b(an_draft[p].begin() + (size_t)l * K, an_draft[p].begin() + (size_t)(l + 1) * K);
      if (a == b) return 0;
      std::sort(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      return a == b ? 1 : 2;
    };
    auto stats = [&](bool per_token) {
      uint64_t cnt[3] = {0, 0, 0};
      for (size_t p = 0; p < an_target.size(); ++p) {
        if (!per_token) {
          for (int l = 0; l < L; ++l) ++cnt[cell(p, l)];
        } else {
          int worst = 0;
          for (int l = 0; l < L && worst < 2; ++l) worst = std::max(worst, cell(p, l));
          ++cnt[worst];
        }
      }
      const double n = static_cast<double>(cnt[0] + cnt[1] + cnt[2]);
      json f;
      f["hard_rate"] = static_cast<double>(cnt[0]) / n;
      f["soft_rate"] = static_cast<double>(cnt[1]) / n;
      f["mismatch_rate"] = 1.0 - static_cast<double>(cnt[0]) / n - static_cast<double>(cnt[1]) / n;
      f["hard_count"] = cnt[0];
      f["soft_count"] = cnt[1];
      f["mismatch_count"] = cnt[2];
      f["total"] = cnt[0] + cnt[1] + cnt[2];
      return f;
    };
    json fid;
    fid["token_layer"] = stats(false);
    fid["token"] = stats(true);
    rep["fidelity"] = fid;
    json ent = json::array();
    for (int l = 0; l < L; ++l) {
      std::vector<uint64_t> cnt(Ex, 0);
      uint64_t tot = 0;
      for (auto& tg : an_target)
        for (int j = 0; j < K; ++j) {
          ++cnt[tg[(size_t)l * K + j]];
          ++tot;
        }
      double h = 0.0;
      for (uint64_t c2 : cnt) {
        if (c2 == 0) continue;
        const double pr = static_cast<double>(c2) / static_cast<double>(tot);
        h -= pr * std::log2(pr);
      }
      ent.push_back(h);
    }
    rep["layer_entropy"] = ent;
  }
  rep["wall_s"] = wall;
  rep["decode_wall_s"] = std::chrono::duration<double>(std::chrono::steady_clock::now() - wall_dec0).count();
  if (!prefill.empty()) rep["prefill"] = prefill;
  rep["profile"] = c.profile.to_json();
  rep["policy"] = policy_name(c.policy);
  // kernel evidence: K3 (bf16 grouped verify FFN, tcgen05) per-launch device time (CUDA events
  // on the launching stream) and algorithmic bytes (expert weights streamed); draft step = one
  // graph replay (L x (K1 + K2 tcgen05 INT4) + LM head).
  json ks;
  ks["kernel_launches"] = launches;
  ks["k3_launches"] = (long)L * (long)cycles.size();
  ks["k3_time_s"] = k3_time;
  ks["k3_weight_bytes"] = k3_bytes;
  ks["k3_groups"] = k3_groups;
  ks["draft_steps"] = draft_steps;
  ks["draft_time_s"] = draft_time;
  ks["draft_step_bytes"] = (double)m.L * m.K * E->S4 + (double)m.V * m.d * 2 + (double)m.L * m.E * m.d * 2 +
                           (double)m.L * E->wattn_layer;
  rep["kernels"] = ks;
  return rep.dump();
}

// ============================================================================ generate_batch
// Several request streams decoded together (include/mspq_capi.h mspq_generate_batch).  Each cycle:
// every active stream drafts k tokens with its own captured draft graph (its state, its KV cache);
// their verify windows are concatenated into ONE batch of n (k+1) tokens that goes through a single
// layer-major verify pass -- K1 over the batch, attention with per-token (window, stream, position)
// metadata, one controller step over all slots, one grouped GEMM per layer, so the streams share
// the expert weight reads and the fetches -- then each stream's accept runs on its slice.
static std::string generate_batch(mspq_engine* E, const int32_t* prompts, const int32_t* lens, int n_streams,
                                  int max_new) {
  if (!E->configured) fail(MSPQ_ERR_INVALID_CONFIG, "engine not configured");
  const auto& m = E->m;
  const HostCfg& c = E->cfg;
  if (n_streams < 1 || n_streams > E->S) fail(MSPQ_ERR_INVALID_CONFIG, "more streams than the engine's max_streams");
  if (c.policy != 0) fail(MSPQ_ERR_INVALID_CONFIG, "generate_batch needs the lru policy");
  const int L = m.L, K = m.K, Ex = m.E, d = m.d, n = n_streams;
  std::vector<const int32_t*> pr(n);
  std::vector<int> plen(n), head(n);
  for (int i = 0, off = 0; i < n; off += lens[i], ++i) {
    pr[i] = prompts + off;
    plen[i] = lens[i];
    if (plen[i] < 1) fail(MSPQ_ERR_EMPTY_RANGE, "empty prompt");
    if (plen[i] - 1 + max_new + E->Tmax >= m.P) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "positions exceed the positional table");
    for (int j = 0; j < plen[i]; ++j)
      if (pr[i][j] < 0 || pr[i][j] >= m.V) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "prompt token out of vocab");
    head[i] = plen[i] - 1;
  }
  const int level = E->o.trace_level;
  const auto wall0 = std::chrono::steady_clock::now();
  E->n_refetch = 0;
  json prefills = json::array();
  for (int i = 0; i < n; ++i) {  // prefill + device decode state of every stream
    E->use_stream(i);
    if (E->attn && plen[i] > 1) prefills.push_back(run_prefill(E, pr[i], plen[i]));
    E->hpin[0] = 0;
    E->hpin[1] = pr[i][plen[i] - 1];
    E->hpin[2] = head[i];
    CUDA_OK(cudaMemcpyAsync(E->dst, E->hpin, 12, cudaMemcpyHostToDevice, E->sc));
    CUDA_OK(cudaMemcpyAsync(E->win_tok(), E->hpin + 1, 4, cudaMemcpyHostToDevice, E->sc));
    CUDA_OK(cudaStreamSynchronize(E->sc));
  }
  E->use_stream(0);
  const auto wall_dec0 = std::chrono::steady_clock::now();
  CUDA_OK(cudaEventRecord(E->ev_t0, E->sc));
  CUDA_OK(cudaStreamWaitEvent(E->sx, E->ev_t0, 0));
  if (E->sdec) CUDA_OK(cudaStreamWaitEvent(E->sdec, E->ev_t0, 0));
  std::vector<std::vector<int>> committed(n);
  json cycles = json::array();
  uint64_t h2d = 0, total_new = 0;
  double stall_total = 0.0;
  std::vector<double> accept(std::max(c.use_governor ? c.k_max : c.fixed_k, 1), c.initial_accept);
  double g = static_cast<double>(L) * static_cast<double>(K);
  auto est = [&]() { return Est([gg = g](int k) { return static_cast<int>(std::llround(gg * static_cast<double>(k))); }); };
  std::vector<int32_t> hbuf;
  std::vector<int> layer_groups(L, 0);
  long launches = 0, k3_groups = 0, draft_steps = 0;
  double k3_time = 0.0, k3_bytes = 0.0, draft_time = 0.0;
  int ci = 0;
  while (true) {
    std::vector<int> act;
    for (int i = 0; i < n; ++i)
      if ((int)committed[i].size() < max_new) act.push_back(i);
    if (act.empty()) break;
    const int na = (int)act.size();
    int rem = max_new;
    for (int i : act) rem = std::min(rem, max_new - (int)committed[i].size());
    const int kk = c.use_governor ? select_k(c.profile, accept, c.k_min, c.k_max, c.k_slo, est()) : c.fixed_k;
    const int k = std::max(1, std::min({kk, rem, E->o.kmax, E->Tmax / na - 1}));
    if (k < 1 || na * (k + 1) > E->Tmax) fail(MSPQ_ERR_K_OUT_OF_RANGE, "batch window exceeds 32 slots");
    const int Tw = k + 1, T = na * Tw;
    const int cycle = ++E->cycle_serial;
    E->ev_pool_next = 0;
    uint64_t cyc_bytes = 0;
    CUDA_OK(cudaEventRecord(E->ev_c0, E->sc));
    CAPI_OK(mspq_cache_begin_cycle(E->cache, k, E->sc));
    // ---- drafts (each stream's own graph; lru: no planner)
    for (int j = 0; j < na; ++j) {
      E->use_stream(act[j]);
      CUDA_OK(cudaMemsetAsync(E->dst, 0, 4, E->sc));  // row = 0
      for (int i = 0; i < k; ++i) CUDA_OK(cudaGraphLaunch(E->gexec, E->sc));
    }
    CUDA_OK(cudaEventRecord(E->ev_dend, E->sc));
    // ---- the batch: windows back to back, per-token metadata
    hbuf.assign((size_t)T * 3 + T, 0);
    for (int j = 0; j < na; ++j)
      for (int sl = 0; sl < Tw; ++sl) {
        const int t = j * Tw + sl;
        hbuf[(size_t)t * 3] = j * Tw;
        hbuf[(size_t)t * 3 + 1] = act[j];
        hbuf[(size_t)t * 3 + 2] = head[act[j]] + sl;
        hbuf[(size_t)T * 3 + t] = head[act[j]] + sl;
      }
    std::memcpy(E->hpin, hbuf.data(), hbuf.size() * 4);  // the previous cycle's reads are synchronised
    CUDA_OK(cudaMemcpyAsync(E->bmeta, E->hpin, (size_t)T * 12, cudaMemcpyHostToDevice, E->sc));
    CUDA_OK(cudaMemcpyAsync(E->bpos, E->hpin + (size_t)T * 3, (size_t)T * 4, cudaMemcpyHostToDevice, E->sc));
    for (int j = 0; j < na; ++j)
      CUDA_OK(cudaMemcpyAsync(E->btok + j * Tw, E->dst_s[act[j]] + 8, (size_t)Tw * 4, cudaMemcpyDeviceToDevice, E->sc));
    E->use_stream(0);
    CAPI_OK(mspq_embed(E->embed, E->pos, E->btok, E->bpos, T, d, E->h, E->sc));
    // ---- one layer-major verify pass over the whole batch
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> stall_ev;
    int ysp_prev = 1;
    for (int l = 0; l < L; ++l) {
      const int pl = (l - 1) & 1;
      int32_t* tgt = E->ids_t + (size_t)l * T * K;
      const float* y = l ? E->yv[pl] : nullptr;
      const int32_t* eo = l ? E->sv[pl].entry_of : nullptr;
      const float* pw = l ? E->wts_t + (size_t)(l - 1) * T * K : nullptr;
      int ysp = ysp_prev;
      long long yst = (long long)T * K * d;
      if (E->attn) {
        ysp = enqueue_attn(E, l, T, nullptr, y, eo, pw, ysp, yst, nullptr, E->sc, E->bmeta);
        y = E->oproj;
        eo = nullptr;
        pw = nullptr;
        yst = (long long)T * d;
      }
      CAPI_OK(mspq_gate_topk(E->h, y, eo, pw, ysp, yst, E->gamma + (size_t)l * d, E->router + (size_t)l * Ex * d,
                             E->xn, tgt, E->wts_t + (size_t)l * T * K, nullptr, nullptr, nullptr, nullptr, nullptr, l,
                             L, T, d, Ex, K, m.eps, E->sc));
      Sched& sv = E->sv[l & 1];
      CAPI_OK(mspq_cache_verify_layer(E->cache, l, T, tgt, E->gbuf, E->sc));
      CUDA_OK(cudaEventRecord(E->ev_w0[l], E->sc));
      CAPI_OK(mspq_build_schedule(tgt, T, K, Ex, E->gbuf, sv.n_groups, sv.group_expert, sv.group_buf, sv.group_off,
                                  sv.entry_tok, sv.entry_of, sv.entry_group, E->sc));
      spin_wait(E->ev_w0[l]);
      CopyBatch b;
      b.demand = true;
      issue_copies(E, cycle, b, cyc_bytes, false, nullptr, l);
      std::vector<int> gb;
      for (int e = 0; e < Ex; ++e)
        if (E->view.host_sched[1 + e] >= 0) gb.push_back(E->view.host_sched[1 + e]);
      bool waited = false;
      for (int buf : gb) {
        if (buf < 0 || buf >= E->nbuf) fail(MSPQ_ERR_OVERFLOW, "schedule buffer out of range");
        if (E->ready_rec[buf]) {
          if (cudaEventQuery(E->ev_ready[buf]) == cudaErrorNotReady) {
            CUDA_OK(cudaStreamWaitEvent(E->sc, E->ev_ready[buf], 0));
            waited = true;
          } else {
            E->ready_rec[buf] = 0;
          }
        }
      }
      if (waited) {
        CUDA_OK(cudaEventRecord(E->ev_w1[l], E->sc));
        stall_ev.push_back({E->ev_w0[l], E->ev_w1[l]});
      }
      const int ng = std::max(1, (int)gb.size());
      auto pick_split = [&](int rows, int kdim) {
        const int units = std::max(1, ng * (rows / 128));
        return std::max(1, std::min({(296 + units - 1) / units, mspq_engine::kMaxSplit, kdim / 64}));
      };
      const int sp1 = pick_split(2 * m.f, d), sp2 = pick_split(d, m.f);
      CUDA_OK(cudaEventRecord(E->ev_k0[l], E->sc));
      CAPI_OK(mspq_moe_bf16_tc(sv.n_groups, sv.group_expert, sv.group_buf, sv.group_off, sv.entry_tok, sv.entry_group,
                               E->xn, E->pool, E->S16, d, m.f, T, K, E->G, sp1, sp2, E->tcws, E->yv[l & 1], E->sc));
      CUDA_OK(cudaEventRecord(E->ev_gemm[l], E->sc));
      launches += (E->attn ? 4 : 0) + 7;
      layer_groups[l] = (int)gb.size();
      for (int buf : gb) {
        E->last_cycle[buf] = cycle;
        E->last_layer[buf] = l;
      }
      ysp_prev = sp2;
    }
    const int pl = (L - 1) & 1;
    CAPI_OK(mspq_gate_topk(E->h, E->yv[pl], E->sv[pl].entry_of, E->wts_t + (size_t)(L - 1) * T * K, ysp_prev,
                           (long long)T * K * d, E->gfinal, nullptr, E->xn, nullptr, nullptr, nullptr, nullptr, nullptr,
                           nullptr, nullptr, L, L, T, d, Ex, K, m.eps, E->sc));
    CAPI_OK(mspq_lm_head(E->xn, E->lm, T, m.V, d, E->logits, E->sc));
    CAPI_OK(mspq_argmax(E->logits, T, m.V, E->amax, E->sc));
    for (int j = 0; j < na; ++j) {  // accept per stream on its slice; next head = its bonus
      int32_t* ds = E->dst_s[act[j]];
      CAPI_OK(mspq_accept_advance(ds + 8 + 1, E->amax + j * Tw, k, ds + 3, ds + 1, ds + 2, head[act[j]], E->sc));
      CUDA_OK(cudaMemcpyAsync(ds + 8, ds + 1, 4, cudaMemcpyDeviceToDevice, E->sc));
    }
    // results back: per stream (accepted, bonus, drafts), target argmax, routing (level >= 1)
    int32_t* hp = E->hpin;
    for (int j = 0; j < na; ++j) {
      CUDA_OK(cudaMemcpyAsync(hp + j * (2 + k), E->dst_s[act[j]] + 3, 8, cudaMemcpyDeviceToHost, E->sc));
      CUDA_OK(cudaMemcpyAsync(hp + j * (2 + k) + 2, E->dst_s[act[j]] + 8 + 1, (size_t)k * 4, cudaMemcpyDeviceToHost, E->sc));
    }
    const size_t o_tr = (size_t)na * (2 + k);
    if (level >= 1)
      CUDA_OK(cudaMemcpyAsync(hp + o_tr, E->ids_t, (size_t)L * T * K * 4, cudaMemcpyDeviceToHost, E->sc));
    CUDA_OK(cudaEventRecord(E->ev_end, E->sc));
    CUDA_OK(cudaEventSynchronize(E->ev_end));
    const int fetched = E->view.host_stat[S_FETCHED];
    double stall = 0.0;
    for (auto& [a, b2] : stall_ev) stall += elapsed_s(a, b2);
    for (int l = 0; l < L; ++l) {  // K3 device time per layer (as generate())
      k3_time += elapsed_s(E->ev_k0[l], E->ev_gemm[l]);
      k3_bytes += (double)layer_groups[l] * E->S16;
      k3_groups += layer_groups[l];
    }
    draft_time += elapsed_s(E->ev_c0, E->ev_dend);
    draft_steps += (long)na * k;
    launches += (long)na * k * E->graph_nodes + 2 + 3 + 2 * na;  // drafts, begin/embed, final norm/lm/argmax, accepts
    json rec;
    rec["cycle"] = ci;
    rec["k"] = k;
    rec["streams"] = act;
    rec["new_experts"] = fetched;
    rec["bytes"] = cyc_bytes;
    rec["io_wait_s"] = stall;
    rec["start_s"] = elapsed_s(E->ev_t0, E->ev_c0);
    rec["span_s"] = elapsed_s(E->ev_c0, E->ev_end);
    json toks = json::array(), accs = json::array();
    int acc_sum = 0;
    for (int j = 0; j < na; ++j) {
      const int sidx = act[j];
      const int accepted = hp[j * (2 + k)], bonus_tok = hp[j * (2 + k) + 1];
      std::vector<int> nt;
      for (int i = 0; i < accepted; ++i) nt.push_back(hp[j * (2 + k) + 2 + i]);
      nt.push_back(bonus_tok);
      const int remi = max_new - (int)committed[sidx].size();
      if ((int)nt.size() > remi) nt.resize(remi);
      for (int t2 : nt) committed[sidx].push_back(t2);
      head[sidx] += accepted + 1;
      toks.push_back(nt);
      accs.push_back(accepted);
      acc_sum += accepted;
      // governor EMA over every stream's outcomes
      std::vector<bool> outcomes;
      for (int i = 0; i < k; ++i) {
        outcomes.push_back(i < accepted);
        if (i >= accepted) break;
      }
      if (outcomes.size() > accept.size()) outcomes.resize(accept.size());
      accept = update_acceptance(accept, c.ema_alpha, outcomes);
    }
    rec["tokens"] = toks;
    rec["accepted"] = accs;
    if (level >= 1) {
      json tgt = json::array();  // [slot][layer][K] over the batch
      for (int t = 0; t < T; ++t) {
        json sl = json::array();
        for (int l = 0; l < L; ++l) {
          json c2 = json::array();
          for (int j2 = 0; j2 < K; ++j2) c2.push_back(hp[o_tr + ((size_t)l * T + t) * K + j2]);
          sl.push_back(c2);
        }
        tgt.push_back(sl);
      }
      rec["target"] = tgt;
    }
    if (level >= 2) {
      const int nl = std::min(E->view.host_stat[S_NLOG], E->view.log_cap);
      std::vector<int32_t> lg((size_t)nl * 6);
      if (nl) CUDA_OK(cudaMemcpy(lg.data(), E->view.log, (size_t)nl * 24, cudaMemcpyDeviceToHost));
      json lj = json::array();
      for (int i = 0; i < nl; ++i) {
        const int32_t* ev = &lg[(size_t)i * 6];
        lj.push_back({ev[0], ev[1], ev[2] / Ex, ev[2] % Ex, ev[3], ev[4] < 0 ? -1 : ev[4] / Ex,
                      ev[4] < 0 ? -1 : ev[4] % Ex, ev[5]});
      }
      rec["log"] = lj;
    }
    cycles.push_back(rec);
    g = static_cast<double>(fetched) / static_cast<double>(k * na);
    total_new += fetched;
    h2d += cyc_bytes;
    stall_total += stall;
    ++ci;
  }
  CUDA_OK(cudaStreamSynchronize(E->sx));
  if (E->sdec) CUDA_OK(cudaStreamSynchronize(E->sdec));
  E->use_stream(0);
  json rep;
  size_t tot = 0;
  json st = json::array();
  for (int i = 0; i < n; ++i) {
    st.push_back(committed[i]);
    tot += committed[i].size();
  }
  const double total_time = cycles.empty() ? 0.0
                                           : cycles.back()["start_s"].get<double>() + cycles.back()["span_s"].get<double>();
  rep["streams"] = n;
  rep["tokens"] = st;
  rep["total_tokens"] = tot;
  rep["total_time_s"] = total_time;
  rep["stall_time_s"] = stall_total;
  rep["total_new_experts"] = total_new;
  rep["h2d_bytes"] = h2d;
  rep["h2d_bytes_bf16"] = total_new * (uint64_t)E->S16;
  rep["refetch_hbm"] = E->n_refetch;
  rep["cycles"] = cycles;
  rep["prefill"] = prefills;
  json ks;  // same kernel evidence as generate(); the draft span covers every stream's k graph replays
  ks["kernel_launches"] = launches;
  ks["k3_launches"] = (long)L * (long)cycles.size();
  ks["k3_time_s"] = k3_time;
  ks["k3_weight_bytes"] = k3_bytes;
  ks["k3_groups"] = k3_groups;
  ks["draft_steps"] = draft_steps;
  ks["draft_time_s"] = draft_time;
  ks["draft_step_bytes"] = (double)m.L * m.K * E->S4 + (double)m.V * m.d * 2 + (double)m.L * m.E * m.d * 2 +
                           (double)m.L * E->wattn_layer;
  rep["kernels"] = ks;
  const auto wall1 = std::chrono::steady_clock::now();
  rep["wall_s"] = std::chrono::duration<double>(wall1 - wall0).count();
  rep["decode_wall_s"] = std::chrono::duration<double>(wall1 - wall_dec0).count();
  return rep.dump();
}

// ============================================================================ C-ABI
namespace {
template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const Err& e) {
    return mspq::set_error(e.code, e.msg);
  } catch (const nlohmann::json::exception& e) {
    return mspq::set_error(MSPQ_ERR_INVALID_CONFIG, e.what());
  } catch (const std::exception& e) {
    return mspq::set_error(MSPQ_ERR_INTERNAL, e.what());
  }
}
char* dupstr(const std::string& s) {
  char* p = (char*)malloc(s.size() + 1);
  memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
void destroy(mspq_engine* E) {
  if (!E) return;
  cudaDeviceSynchronize();
  for (size_t st = 0; st < E->gexec_s.size(); ++st) {
    if (E->gexec_s[st]) cudaGraphExecDestroy(E->gexec_s[st]);
    if (E->graph_s[st]) cudaGraphDestroy(E->graph_s[st]);
  }
  for (size_t st = 1; st < E->dst_s.size(); ++st)
    if (E->dst_s[st]) cudaFree(E->dst_s[st]);
  for (void* p : {(void*)E->bmeta, (void*)E->btok, (void*)E->bpos})
    if (p) cudaFree(p);
  E->kcache = E->kv_base_k;  // the allocations (stream 0)
  E->vcache = E->kv_base_v;
  for (auto v : {&E->ev_ready, &E->ev_gemm, &E->ev_w0, &E->ev_w1, &E->ev_row, &E->ev_pool, &E->ev_k0, &E->ev_g0, &E->ev_g1,
                 &E->ev_ka1, &E->ev_rt})
    for (auto ev : *v)
      if (ev) cudaEventDestroy(ev);
  for (auto ev : {E->ev_c0, E->ev_dend, E->ev_end, E->ev_t0})
    if (ev) cudaEventDestroy(ev);
  if (E->cache) mspq_cache_destroy(E->cache);
  if (E->pool) cudaFree(E->pool);
  if (E->ws) cudaFree(E->ws);
  if (E->draft4) cudaFree(E->draft4);
  if (E->wblk) cudaFree(E->wblk);
  if (E->hpin) cudaFreeHost(E->hpin);
  for (float* p : {E->hcap_v, E->hcap_dstage, E->hcap_d})
    if (p) cudaFree(p);
  if (E->sched_cap) cudaFree(E->sched_cap);
  if (E->act_d) cudaFree(E->act_d);
  for (int i = 0; i < 2; ++i) {
    if (E->pf_buf[i]) cudaFree(E->pf_buf[i]);
    if (E->pf_y[i]) cudaFree(E->pf_y[i]);
    if (E->pf_ready[i]) cudaEventDestroy(E->pf_ready[i]);
    if (E->pf_done[i]) cudaEventDestroy(E->pf_done[i]);
  }
  if (E->pf_h) cudaFree(E->pf_h);
  if (E->pf_gbuf) cudaFree(E->pf_gbuf);
  if (E->pf_eo) cudaFree(E->pf_eo);
  for (void* p : {(void*)E->wattn, (void*)E->gamma_a, (void*)E->kcache, (void*)E->vcache, (void*)E->qkv, (void*)E->oproj,
                  (void*)E->ao, (void*)E->dsched, E->dws, (void*)E->attn_part, (void*)E->hmid_v, (void*)E->hmid_dstage, (void*)E->hmid_d})
    if (p) cudaFree(p);
  for (size_t r = 0; r < E->peer_ipc.size(); ++r)
    if (E->peer_ipc[r] && E->peer_home[r]) cudaIpcCloseMemHandle(E->peer_home[r]);
  if (E->home) cudaFree(E->home);
  if (E->host) {
    if (E->host_is_shm) {
      cudaHostUnregister(E->host);
      munmap(E->host, E->host_bytes);
    } else {
      cudaFreeHost(E->host);
    }
  }
  for (int i = 0; i < 2; ++i) {
    if (E->stage[i]) cudaFree(E->stage[i]);
    if (E->ev_stage[i]) cudaEventDestroy(E->ev_stage[i]);
  }
  if (E->sc) cudaStreamDestroy(E->sc);
  if (E->sx) cudaStreamDestroy(E->sx);
  if (E->sdec) cudaStreamDestroy(E->sdec);
  delete E;
}
}  // namespace

extern "C" {

int mspq_engine_create(const mspq_model_desc* md, const mspq_engine_opts* op, mspq_engine** out) {
  return guarded([&] {
    *out = nullptr;
    const auto& m = *md;
    if (m.L < 1 || m.E < 1 || m.K < 1 || m.K > m.E || m.E > 1024 || m.L * m.E > 8192)
      fail(MSPQ_ERR_SHAPE_VIOLATION, "need 1 <= K <= E <= 1024, L*E <= 8192");
    if (m.d % 256 || m.f % 256 || m.V < 1 || m.P < 2) fail(MSPQ_ERR_SHAPE_VIOLATION, "need d, f multiples of 256");
    if (op->kmax < 1 || op->kmax > 32) fail(MSPQ_ERR_K_OUT_OF_RANGE, "kmax must be in [1, 32]");
    mspq_engine* E = new mspq_engine();
    try {
      E->m = m;
      E->o = *op;
      E->store_path = op->host_store_path ? op->host_store_path : "";
      E->o.host_store_path = nullptr;
      CUDA_OK(cudaSetDevice(op->device));
      int lo, hi;
      cudaDeviceGetStreamPriorityRange(&lo, &hi);
      // compute at the highest priority: the verify GEMMs' CTAs go ahead of the XC decodes of
      // prefetched experts that run beside them (the decodes have slack: the link is slower)
      CUDA_OK(cudaStreamCreateWithPriority(&E->sc, cudaStreamNonBlocking, hi));
      CUDA_OK(cudaStreamCreateWithPriority(&E->sx, cudaStreamNonBlocking, hi));
      E->S16 = mspq_bf16_blob_bytes(m.d, m.f);
      E->codec = op->expert_codec;
      if (E->codec < 0 || E->codec > 1) fail(MSPQ_ERR_INVALID_CONFIG, "expert_codec must be 0 (none) or 1 (xc)");
      E->n_tiles = (int)(E->S16 / 16384);
      E->Sreg = E->codec ? ((mspq_xc_max_blob_bytes(E->n_tiles) + 4095) / 4096) * 4096 : E->S16;
      if (E->codec) {
        CUDA_OK(cudaStreamCreateWithPriority(&E->sdec, cudaStreamNonBlocking, lo));
        for (int i = 0; i < 2; ++i) {
          CUDA_OK(cudaMalloc(&E->stage[i], (size_t)E->Sreg));
          CUDA_OK(cudaEventCreateWithFlags(&E->ev_stage[i], cudaEventDisableTiming));
        }
      }
      E->S4 = mspq_int4_blob_bytes(m.d, m.f);
      // window capacity: the decode's k+1 slots, and 32-token prefill windows with attention (the
      // widest K3 / K1 / attention launch; fewer prefill windows = fewer expert re-fetches)
      E->S = std::max(1, std::min(op->max_streams, 32));
      E->Tmax = std::max(op->kmax + 1, (m.H > 0 || E->S > 1) ? 32 : 0);
      E->n_payload = m.unique_experts > 0 ? std::min(m.unique_experts, m.L * m.E) : m.L * m.E;
      if (m.H > 0) {
        if (m.Hkv < 1 || m.H % m.Hkv || m.H / m.Hkv > 8 || (m.Dh != 64 && m.Dh != 128) || (m.H * m.Dh) % 128 ||
            ((m.H + 2 * m.Hkv) * m.Dh) % 128)
          fail(MSPQ_ERR_SHAPE_VIOLATION, "attention: need Hkv | H, H/Hkv <= 8, Dh in {64, 128}, H*Dh and (H+2Hkv)*Dh % 128");
        E->attn = true;
        E->Nq = m.H * m.Dh;
        E->Nkv = m.Hkv * m.Dh;
        E->Nqkv = E->Nq + 2 * E->Nkv;
      }
      make_weights(E);
      alloc_host_store(E);
      make_experts(E);
      make_workspaces(E);
      E->ev_gemm.resize(m.L);
      E->ev_w0.resize(m.L);
      E->ev_w1.resize(m.L);
      E->ev_row.resize(E->Tmax);
      E->ev_g0.resize(E->Tmax);
      E->ev_g1.resize(E->Tmax);
      E->ev_k0.resize(m.L);
      E->ev_ka1.resize(m.L);
      E->ev_rt.resize(m.L);
      E->layer_parts.assign(m.L, 0);
      for (auto v : {&E->ev_gemm, &E->ev_w0, &E->ev_w1, &E->ev_row, &E->ev_k0, &E->ev_g0, &E->ev_g1, &E->ev_ka1, &E->ev_rt})
        for (auto& ev : *v) CUDA_OK(cudaEventCreate(&ev));
      for (auto p : {&E->ev_c0, &E->ev_dend, &E->ev_end, &E->ev_t0}) CUDA_OK(cudaEventCreate(p));
      CUDA_OK(cudaStreamSynchronize(E->sc));
    } catch (...) {
      destroy(E);
      throw;
    }
    *out = E;
    return MSPQ_OK;
  });
}

int mspq_engine_destroy(mspq_engine* E) {
  return guarded([&] {
    destroy(E);
    return MSPQ_OK;
  });
}

int mspq_engine_configure(mspq_engine* E, const char* cfg) {
  return guarded([&] {
    configure(E, cfg);
    return MSPQ_OK;
  });
}

int mspq_generate(mspq_engine* E, const int32_t* prompt, int n, int max_new, char** report) {
  return guarded([&] {
    *report = dupstr(generate(E, prompt, n, max_new));
    return MSPQ_OK;
  });
}

int mspq_generate_batch(mspq_engine* E, const int32_t* prompts, const int32_t* lens, int n_streams, int max_new,
                        char** report) {
  return guarded([&] {
    *report = dupstr(generate_batch(E, prompts, lens, n_streams, max_new));
    return MSPQ_OK;
  });
}

int mspq_engine_info(mspq_engine* E, char** out) {
  return guarded([&] {
    json j;
    const auto& m = E->m;
    j["L"] = m.L;
    j["E"] = m.E;
    j["K"] = m.K;
    j["d"] = m.d;
    j["f"] = m.f;
    j["V"] = m.V;
    j["expert_bytes_bf16"] = E->S16;
    j["expert_bytes_int4"] = E->S4;
    j["host_store_bytes"] = E->host_bytes;
    j["expert_codec"] = E->codec ? "xc" : "none";
    j["expert_wire_bytes_mean"] = E->codec ? (double)E->xc_bytes_total / E->n_payload : (double)E->S16;
    j["n_payload"] = E->n_payload;
    j["slot_buffers"] = E->nbuf;
    j["slot_pool_bytes"] = (uint64_t)E->nbuf * E->S16;
    j["draft_resident_bytes"] = (uint64_t)m.L * m.E * E->S4;
    j["pcie_bw_measured"] = E->pcie_bw_measured;
    j["draft_step_s"] = E->draft_step_s;
    j["pcie_init_latency_measured"] = E->pcie_fixed.first;
    j["pcie_overhead_measured"] = E->pcie_fixed.second;
    json vs = json::array();
    for (auto& [w, t] : E->verify_measured) vs.push_back({w, t});
    j["verify_samples_measured"] = vs;
    j["home_bytes"] = E->home_bytes;
    j["home_bw_measured"] = E->home_bw_measured;
    j["peer_group"] = E->peer_G;
    if (E->configured) j["profile"] = E->cfg.profile.to_json();
    *out = dupstr(j.dump());
    return MSPQ_OK;
  });
}

int mspq_engine_read(mspq_engine* E, const char* name, void* dst, long long bytes) {
  return guarded([&] {
    const auto& m = E->m;
    std::string n = name;
    const void* src = nullptr;
    size_t avail = 0;
    bool from_host = false;
    auto two = [&](const std::string& rest, int& a, int& b) { return sscanf(rest.c_str(), "%d:%d", &a, &b) == 2; };
    if (n == "embed") src = E->embed, avail = (size_t)m.V * m.d * 2;
    else if (n == "lm") src = E->lm, avail = (size_t)m.V * m.d * 2;
    else if (n == "pos") src = E->pos, avail = (size_t)m.P * m.d * 2;
    else if (n == "gamma:final") src = E->gfinal, avail = (size_t)m.d * 2;
    else if (n.rfind("gamma:", 0) == 0) src = E->gamma + (size_t)atoi(n.c_str() + 6) * m.d, avail = (size_t)m.d * 2;
    else if (n.rfind("router:", 0) == 0) src = E->router + (size_t)atoi(n.c_str() + 7) * m.E * m.d, avail = (size_t)m.E * m.d * 2;
    else if (n.rfind("draft:", 0) == 0) {
      int l, e;
      if (!two(n.substr(6), l, e)) fail(MSPQ_ERR_INVALID_CONFIG, n);
      src = E->draft4 + ((size_t)l * m.E + e) * E->S4;
      avail = E->S4;
    } else if (n.rfind("expert:", 0) == 0) {
      int l, e;
      if (!two(n.substr(7), l, e)) fail(MSPQ_ERR_INVALID_CONFIG, n);
      const unsigned char* hb = E->host_blob(E->payload(l * m.E + e));
      if (E->codec) {  // decode the stored blob back into the bf16 tile images
        if ((size_t)bytes > (size_t)E->S16) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "read beyond tensor");
        void *dblob, *dimg;
        const uint64_t wb = E->wire_bytes(E->payload(l * m.E + e));
        CUDA_OK(cudaMalloc(&dblob, wb));
        CUDA_OK(cudaMalloc(&dimg, E->S16));
        CUDA_OK(cudaMemcpy(dblob, hb, wb, cudaMemcpyHostToDevice));
        const int st = mspq_xc_decode(dblob, 0, E->n_tiles, dimg, 0, nullptr);
        cudaError_t ce = cudaDeviceSynchronize();
        if (ce == cudaSuccess && st == 0) ce = cudaMemcpy(dst, dimg, bytes, cudaMemcpyDeviceToHost);
        cudaFree(dblob);
        cudaFree(dimg);
        if (st) fail(st, mspq_last_error());
        if (ce != cudaSuccess) fail(MSPQ_ERR_CUDA, cudaGetErrorString(ce));
        return MSPQ_OK;
      }
      src = hb;
      avail = E->S16;
      from_host = true;
    } else if (n.rfind("kcache:", 0) == 0 || n.rfind("vcache:", 0) == 0) {
      const int l = atoi(n.c_str() + 7);
      if (!E->attn || l < 0 || l >= m.L) fail(MSPQ_ERR_INVALID_CONFIG, n);
      src = (n[0] == 'k' ? E->kcache : E->vcache) + (size_t)l * E->kv_layer();
      avail = E->kv_layer() * 2;
    } else if (n.rfind("wqkv:", 0) == 0 || n.rfind("wo:", 0) == 0) {
      const int l = atoi(n.c_str() + (n[1] == 'q' ? 5 : 3));
      if (!E->attn || l < 0 || l >= m.L) fail(MSPQ_ERR_INVALID_CONFIG, n);
      const size_t nq = (size_t)E->Nqkv * m.d * 2;
      src = E->wattn + (size_t)l * E->wattn_layer + (n[1] == 'q' ? 0 : nq);
      avail = n[1] == 'q' ? nq : (size_t)m.d * E->Nq * 2;
    } else if (n.rfind("gamma_attn:", 0) == 0) {
      const int l = atoi(n.c_str() + 11);
      if (!E->attn || l < 0 || l >= m.L) fail(MSPQ_ERR_INVALID_CONFIG, n);
      src = E->gamma_a + (size_t)l * m.d;
      avail = (size_t)m.d * 2;
    } else if (n.rfind("hmid_v:", 0) == 0 || n.rfind("hmid_d:", 0) == 0) {
      const auto& hist = n[5] == 'v' ? E->hmid_v_hist : E->hmid_d_hist;
      const size_t ci = (size_t)atoi(n.c_str() + 7);
      if (ci >= hist.size()) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "no residual capture for " + n + " (trace_level 3)");
      src = hist[ci].data();
      avail = hist[ci].size() * 4;
      from_host = true;
    } else if (n.rfind("hcap_v:", 0) == 0 || n.rfind("hcap_d:", 0) == 0) {
      const auto& hist = n[5] == 'v' ? E->hcap_v_hist : E->hcap_d_hist;
      const size_t ci = (size_t)atoi(n.c_str() + 7);
      if (ci >= hist.size()) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "no residual capture for " + n + " (trace_level 3)");
      src = hist[ci].data();
      avail = hist[ci].size() * 4;
      from_host = true;
    } else if (n.rfind("expert_blob:", 0) == 0) {
      int l, e;
      if (!two(n.substr(12), l, e)) fail(MSPQ_ERR_INVALID_CONFIG, n);
      src = E->host_blob(E->payload(l * m.E + e));
      avail = E->codec ? E->wire_bytes(E->payload(l * m.E + e)) : E->S16;
      from_host = true;
    } else
      fail(MSPQ_ERR_INVALID_CONFIG, "unknown tensor " + n);
    if ((size_t)bytes > avail) fail(MSPQ_ERR_RANGE_OUT_OF_BOUNDS, "read beyond tensor");
    if (from_host) memcpy(dst, src, bytes);
    else CUDA_OK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    return MSPQ_OK;
  });
}

int mspq_engine_home_create(mspq_engine* E, int group, int rank, void* ipc_out) {
  return guarded([&] {
    const auto& m = E->m;
    if (group < 1 || rank < 0 || rank >= group) fail(MSPQ_ERR_INVALID_CONFIG, "peer tier: need 0 <= rank < group");
    if (E->home) fail(MSPQ_ERR_INVALID_CONFIG, "peer tier: home region already created");
    CUDA_OK(cudaSetDevice(E->o.device));
    E->peer_G = group;
    E->peer_rank = rank;
    E->home_per_layer = (m.E + group - 1) / group;
    E->home_bytes = (size_t)m.L * E->home_per_layer * (size_t)E->S16;
    CUDA_OK(cudaMalloc(&E->home, E->home_bytes));
    E->peer_home.assign(group, nullptr);
    E->peer_ipc.assign(group, 0);
    // fill: every expert homed here, from the host store (XC blobs decoded on the GPU)
    unsigned char* blob = nullptr;
    if (E->codec) CUDA_OK(cudaMalloc(&blob, (size_t)E->Sreg));
    for (int l = 0; l < m.L; ++l)
      for (int e = rank; e < m.E; e += group) {
        const int key = l * m.E + e;
        unsigned char* dst = E->home + ((size_t)l * E->home_per_layer + e / group) * (size_t)E->S16;
        const unsigned char* hb = E->host_blob(E->payload(key));
        if (E->codec) {
          CUDA_OK(cudaMemcpyAsync(blob, hb, E->wire_bytes(E->payload(key)), cudaMemcpyHostToDevice, E->sc));
          CAPI_OK(mspq_xc_decode(blob, 0, E->n_tiles, dst, 0, E->sc));
        } else {
          CUDA_OK(cudaMemcpyAsync(dst, hb, E->S16, cudaMemcpyHostToDevice, E->sc));
        }
      }
    CUDA_OK(cudaStreamSynchronize(E->sc));
    if (blob) cudaFree(blob);
    E->peer_home[rank] = E->home;
    if (ipc_out) {
      cudaIpcMemHandle_t h;
      CUDA_OK(cudaIpcGetMemHandle(&h, E->home));
      memcpy(ipc_out, &h, sizeof(h));
    }
    return MSPQ_OK;
  });
}

int mspq_engine_peer_attach_ipc(mspq_engine* E, int peer_rank, const void* handle) {
  return guarded([&] {
    if (E->peer_G <= 0) fail(MSPQ_ERR_INVALID_CONFIG, "peer tier: create the home region first");
    if (peer_rank < 0 || peer_rank >= E->peer_G || peer_rank == E->peer_rank)
      fail(MSPQ_ERR_INVALID_CONFIG, "peer tier: bad peer rank");
    if (E->peer_home[peer_rank]) fail(MSPQ_ERR_INVALID_CONFIG, "peer tier: peer already attached");
    CUDA_OK(cudaSetDevice(E->o.device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    CUDA_OK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    E->peer_home[peer_rank] = (unsigned char*)p;
    E->peer_ipc[peer_rank] = 1;
    return MSPQ_OK;
  });
}

int mspq_engine_peer_attach(mspq_engine* E, int peer_rank, mspq_engine* P) {
  return guarded([&] {
    if (E->peer_G <= 0 || !P || P->peer_G != E->peer_G || P->peer_rank != peer_rank || !P->home)
      fail(MSPQ_ERR_INVALID_CONFIG, "peer tier: peer has no home region of this group / rank");
    if (peer_rank == E->peer_rank) fail(MSPQ_ERR_INVALID_CONFIG, "peer tier: bad peer rank");
    if (P->o.device != E->o.device) {
      int ok = 0;
      CUDA_OK(cudaDeviceCanAccessPeer(&ok, E->o.device, P->o.device));
      if (!ok) fail(MSPQ_ERR_CUDA, "peer tier: no peer access between the two GPUs");
      CUDA_OK(cudaSetDevice(E->o.device));
      const cudaError_t pe = cudaDeviceEnablePeerAccess(P->o.device, 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CUDA_OK(pe);
      cudaGetLastError();
    }
    E->peer_home[peer_rank] = P->home;
    return MSPQ_OK;
  });
}

}  // extern "C"
