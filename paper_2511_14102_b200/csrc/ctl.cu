// K4: the expert-cache control plane on the device (one warp per launch).
//
// Restates the reference scheduler/simulator rules (file:line into /root/reference/proj):
//   CacheState                      scheduler.cpp:76-138  -> res[] (key -> HBM buffer), stamp[]
//                                                            (LRU recency), lsize[], total
//   plan_prefetch                   scheduler.cpp:173-254 -> plan_rows (token-major, full ELB)
//                                                            and the causal row-by-row variant
//   select_victim_lookahead         scheduler.cpp:256-274 -> belady_victim (warp argmax)
//   policy_step                     scheduler.cpp:276-312 -> policy_step
//   prefetch_insert / the cycle     sim.cpp:152-295       -> k_ctl_replay_cycle (token-major,
//                                                            bit-exact with run_simulation)
//   live engine                     DESIGN.md §4          -> k_ctl_begin_cycle / k_ctl_plan_row /
//                                                            k_ctl_verify_layer (layer-major)
// Keys are l*E + e, so integer order == (layer, expert) order.  All 32 lanes run the same
// control flow on the same (volatile) state; lane 0 performs every mutation followed by
// __syncwarp(); scans over keys are split across lanes and reduced with exact tie-breaks.
// Every cache insertion allocates a physical HBM buffer from a free stack; evicted buffers are
// parked on a pending list until the end of the launch (the verify GEMM of this step may still
// read them) -- the host orders copies after the last reader.
#include <climits>

#include "common.cuh"
#include "ctl.h"

namespace mspq {

namespace {

MSPQ_D int lane_id() { return threadIdx.x & 31; }

struct ElbView {
  const int32_t* ids;   // row r, layer l, slot j at ids[(r*L + l)*K + j]
  const float* gf;      // fp32 gates (live) or nullptr
  const double* gd;     // fp64 gates (replay) or nullptr
  int k;                // rows available
};

struct Ctx {
  CtlDev C;
  ElbView elb;
  int* gb = nullptr;    // verify step: first-request buffer per expert of step_layer (smem)
  int step_layer = -1;
  bool emit = true;     // copy requests (live engine); replay runs the control plane only
};

MSPQ_D volatile int* V(int* p) { return (volatile int*)p; }

MSPQ_D int get(const Ctx& x, int slot) { return V(x.C.scal)[slot]; }
MSPQ_D void put(const Ctx& x, int slot, int v) {
  if (lane_id() == 0) V(x.C.scal)[slot] = v;
  __syncwarp();
}
MSPQ_D void add(const Ctx& x, int slot, int v) {
  if (lane_id() == 0) V(x.C.scal)[slot] = V(x.C.scal)[slot] + v;
  __syncwarp();
}

MSPQ_D bool contains(const Ctx& x, int key) { return V(x.C.res)[key] >= 0; }

MSPQ_D void touch(const Ctx& x, int key) {
  if (lane_id() == 0) {
    volatile unsigned long long* clk = (volatile unsigned long long*)x.C.clock;
    unsigned long long c = *clk + 1;
    *clk = c;
    ((volatile unsigned long long*)x.C.stamp)[key] = c;
  }
  __syncwarp();
}

MSPQ_D bool needs_eviction(const Ctx& x, int layer) {
  if (x.C.mode == CTL_GLOBAL) return get(x, S_TOTAL) >= x.C.cap_global;
  return V(x.C.lsize)[layer] >= x.C.cap[layer];
}

MSPQ_D int key_lo(const Ctx& x, int layer) { return layer >= 0 ? layer * x.C.E : 0; }
MSPQ_D int key_hi(const Ctx& x, int layer) { return layer >= 0 ? (layer + 1) * x.C.E : x.C.L * x.C.E; }

// least-recently-used resident key (smallest stamp), restricted to `layer` when >= 0
MSPQ_D int lru_victim(const Ctx& x, int layer) {
  unsigned long long best = ULLONG_MAX;
  int bk = -1;
  for (int key = key_lo(x, layer) + lane_id(); key < key_hi(x, layer); key += 32)
    if (contains(x, key)) {
      unsigned long long s = ((volatile unsigned long long*)x.C.stamp)[key];
      if (s < best) {
        best = s;
        bk = key;
      }
    }
  for (int off = 16; off >= 1; off >>= 1) {
    unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, off);
    int ok = __shfl_xor_sync(0xffffffffu, bk, off);
    if (ob < best || (ob == best && ok >= 0 && (bk < 0 || ok < bk))) {
      best = ob;
      bk = ok;
    }
  }
  return bk;
}

// ELB next use of key at or after `now` among the first `visible` rows (scheduler.cpp:33-39)
MSPQ_D int next_use(const Ctx& x, int key, int now, int visible) {
  const int L = x.C.L, K = x.C.K, E = x.C.E;
  const int l = key / E, e = key - l * E;
  const int end = min(visible, x.elb.k);
  for (int r = max(now, 0); r < end; ++r)
    for (int j = 0; j < K; ++j)
      if (x.elb.ids[((int64_t)r * L + l) * K + j] == e) return r;
  return INT_MAX;
}

// select_victim_lookahead: max next use, no use = +inf, tie -> larger key
MSPQ_D int belady_victim(const Ctx& x, int now, int visible, int layer) {
  int bu = -1, bk = -1;
  for (int key = key_lo(x, layer) + lane_id(); key < key_hi(x, layer); key += 32)
    if (contains(x, key)) {
      int u = next_use(x, key, now, visible);
      if (u > bu || (u == bu && key > bk)) {
        bu = u;
        bk = key;
      }
    }
  for (int off = 16; off >= 1; off >>= 1) {
    int ou = __shfl_xor_sync(0xffffffffu, bu, off);
    int ok = __shfl_xor_sync(0xffffffffu, bk, off);
    if (ou > bu || (ou == bu && ok > bk)) {
      bu = ou;
      bk = ok;
    }
  }
  return bk;
}

// Evicted buffers return to the free stack at once, except a buffer the current verify
// step's GEMM reads (first-request buffer of this layer), which is parked until the step ends.
MSPQ_D void erase(const Ctx& x, int key) {
  if (key < 0) return;  // nothing resident in the scope (capacity 0): nothing to evict
  if (lane_id() == 0) {
    volatile int* res = V(x.C.res);
    int buf = res[key];
    res[key] = -1;
    V(x.C.lsize)[key / x.C.E] -= 1;
    V(x.C.scal)[S_TOTAL] -= 1;
    const bool defer = x.gb && key / x.C.E == x.step_layer && ((volatile int*)x.gb)[key % x.C.E] == buf;
    if (buf >= 0) {
      if (defer) {
        int np = V(x.C.scal)[S_NPEND];
        V(x.C.pending)[np] = buf;
        V(x.C.scal)[S_NPEND] = np + 1;
      } else {
        int nf = V(x.C.scal)[S_NFREE];
        V(x.C.free_stack)[nf] = buf;
        V(x.C.scal)[S_NFREE] = nf + 1;
      }
    }
  }
  __syncwarp();
}

MSPQ_D void insert_key(const Ctx& x, int key) {
  if (lane_id() == 0) {
    volatile int* scal = V(x.C.scal);
    int nf = scal[S_NFREE];
    int buf = -1;
    if (nf > 0) {
      buf = V(x.C.free_stack)[nf - 1];
      scal[S_NFREE] = nf - 1;
    } else {
      scal[S_OVERFLOW] = 1;
    }
    V(x.C.res)[key] = buf;
    volatile unsigned long long* clk = (volatile unsigned long long*)x.C.clock;
    unsigned long long c = *clk + 1;
    *clk = c;
    ((volatile unsigned long long*)x.C.stamp)[key] = c;
    V(x.C.lsize)[key / x.C.E] += 1;
    scal[S_TOTAL] += 1;
  }
  __syncwarp();
}

MSPQ_D void log_event(const Ctx& x, int kind, int tag, int key, int hit, int victim) {
  if (lane_id() == 0) {
    volatile int* scal = V(x.C.scal);
    int n = scal[S_NLOG];
    if (x.C.log && n < x.C.log_cap) {
      volatile int* ev = V(x.C.log) + (int64_t)n * 6;
      ev[0] = kind;
      ev[1] = tag;
      ev[2] = key;
      ev[3] = hit;
      ev[4] = victim;
      ev[5] = V(x.C.res)[key];
    }
    scal[S_NLOG] = n + 1;
  }
  __syncwarp();
}

MSPQ_D void copy_request(const Ctx& x, int key, int kind) {
  if (!x.emit) return;
  if (lane_id() == 0) {
    volatile int* scal = V(x.C.scal);
    int n = scal[S_NREQ];
    if (n < x.C.req_cap) {
      int* rq = x.C.req_dev + (int64_t)n * 3;  // device staging; copied to mapped memory at exit
      rq[0] = key;
      rq[1] = V(x.C.res)[key];
      rq[2] = kind;
    } else {
      scal[S_OVERFLOW] = 2;
    }
    scal[S_NREQ] = n + 1;
  }
  __syncwarp();
}

// sim.cpp:158-177 prefetch_insert; returns true when a transfer is needed.
MSPQ_D bool prefetch_insert(const Ctx& x, int key, bool belady, int now, int visible, int kind,
                            int tag) {
  if (contains(x, key)) {
    if (!belady) touch(x, key);
    return false;
  }
  const int layer = key / x.C.E;
  const int vl = x.C.mode == CTL_PER_LAYER ? layer : -1;
  int victim = -1;
  if (needs_eviction(x, layer)) {
    victim = belady ? belady_victim(x, now, visible, vl) : lru_victim(x, vl);
    erase(x, victim);
  }
  insert_key(x, key);
  add(x, S_FETCHED, 1);
  log_event(x, kind, tag, key, 0, victim);
  copy_request(x, key, kind);
  return true;
}

// scheduler.cpp:276-312 policy_step; returns hit.
MSPQ_D bool policy_step(const Ctx& x, int key, int now, int tag) {
  const bool hit = contains(x, key);
  const int layer = key / x.C.E;
  const int vl = x.C.mode == CTL_PER_LAYER ? layer : -1;
  int victim = -1;
  const int pol = x.C.policy;
  if (pol == POL_LRU || pol == POL_SP_SOONER || pol == POL_SP_LATER) {
    if (hit) {
      touch(x, key);
    } else {
      if (needs_eviction(x, layer)) {
        victim = lru_victim(x, vl);
        erase(x, victim);
      }
      insert_key(x, key);
    }
  } else {
    if (!hit) {
      if (needs_eviction(x, layer)) {
        victim = belady_victim(x, now, INT_MAX, vl);
        erase(x, victim);
      }
      insert_key(x, key);
    }
  }
  log_event(x, EV_DEMAND, tag, key, hit ? 1 : 0, victim);
  if (!hit) {
    add(x, S_FETCHED, 1);
    add(x, S_DEMAND, 1);
    copy_request(x, key, EV_DEMAND);
  }
  return hit;
}

// The host reads the mapped counters only after the launch's event has completed, which makes
// the kernel's writes visible, so no system-scope fence is needed here (it cost ~2 us per launch).
MSPQ_D void publish(const Ctx& x) {
  __syncwarp();
  if (x.C.hstat)
    for (int i = lane_id(); i < S_COUNT; i += 32) ((volatile int*)x.C.hstat)[i] = V(x.C.scal)[i];
  __syncwarp();
}

MSPQ_D void release_pending(const Ctx& x) {
  if (lane_id() == 0) {
    volatile int* scal = V(x.C.scal);
    int np = scal[S_NPEND], nf = scal[S_NFREE];
    for (int i = 0; i < np; ++i) V(x.C.free_stack)[nf + i] = V(x.C.pending)[i];
    scal[S_NFREE] = nf + np;
    scal[S_NPEND] = 0;
  }
  __syncwarp();
}

// ELB confidence: gate / sum(gates in the cell), 1.0 when no gates (scheduler.cpp:51-57)
MSPQ_D double conf_of(const Ctx& x, int r, int l, int j) {
  const int L = x.C.L, K = x.C.K;
  const int64_t base = ((int64_t)r * L + l) * K;
  if (!x.elb.gf && !x.elb.gd) return 1.0;
  double norm = 0.0;
  for (int q = 0; q < K; ++q) norm += x.elb.gd ? x.elb.gd[base + q] : (double)x.elb.gf[base + q];
  if (!(norm > 0.0)) return 1.0;
  const double g = x.elb.gd ? x.elb.gd[base + j] : (double)x.elb.gf[base + j];
  return g / norm;
}

// ---------------------------------------------------------------- the planner
// absorb one ELB row into the candidate table (scheduler.cpp:191-199); `snap` = residency
// at plan time.
MSPQ_D void absorb_row(const Ctx& x, int r, const unsigned char* snap_or_null) {
  const int L = x.C.L, K = x.C.K, E = x.C.E;
  for (int l = 0; l < L; ++l)
    for (int j = 0; j < K; ++j) {
      const int e = x.elb.ids[((int64_t)r * L + l) * K + j];
      const int key = l * E + e;
      const bool res = snap_or_null ? snap_or_null[key] != 0 : contains(x, key);
      if (res || ((volatile unsigned char*)x.C.sched)[key]) continue;
      const double c = conf_of(x, r, l, j);
      if (lane_id() == 0) {
        volatile int* cf = V(x.C.cand_first);
        volatile double* cc = (volatile double*)x.C.cand_conf;
        if (cf[key] < 0) {
          cf[key] = r;
          cc[key] = c;
        } else if (c > cc[key]) {
          cc[key] = c;
        }
      }
      __syncwarp();
    }
}

// best remaining Phase-II candidate: priority conf*(k-first)/k desc, first asc, key asc
MSPQ_D int best_candidate(const Ctx& x, int k) {
  double bp = -1.0;
  int bf = INT_MAX, bk = -1;
  const int n = x.C.L * x.C.E;
  for (int key = lane_id(); key < n; key += 32) {
    const int f = ((volatile int*)x.C.cand_first)[key];
    if (f < 0) continue;
    const double p = ((volatile double*)x.C.cand_conf)[key] * (double)(k - f) / (double)k;
    if (bk < 0 || p > bp || (p == bp && (f < bf || (f == bf && key < bk)))) {
      bp = p;
      bf = f;
      bk = key;
    }
  }
  for (int off = 16; off >= 1; off >>= 1) {
    double op = __shfl_xor_sync(0xffffffffu, bp, off);
    int of = __shfl_xor_sync(0xffffffffu, bf, off);
    int ok = __shfl_xor_sync(0xffffffffu, bk, off);
    if (ok >= 0 && (bk < 0 || op > bp || (op == bp && (of < bf || (of == bf && ok < bk))))) {
      bp = op;
      bf = of;
      bk = ok;
    }
  }
  return bk;
}

MSPQ_D void mark_scheduled(const Ctx& x, int key) {
  if (lane_id() == 0) {
    ((volatile unsigned char*)x.C.sched)[key] = 1;
    V(x.C.cand_first)[key] = -1;
  }
  __syncwarp();
}

MSPQ_D void plan_item(const Ctx& x, int row, int key, int phase) {
  if (lane_id() == 0) {
    volatile int* scal = V(x.C.scal);
    int n = scal[S_NPLAN];
    if (n < x.C.plan_cap) {
      V(x.C.plan)[n * 3 + 0] = row;
      V(x.C.plan)[n * 3 + 1] = key;
      V(x.C.plan)[n * 3 + 2] = phase;
    }
    scal[S_NPLAN] = n + 1;
  }
  __syncwarp();
}

// Phase II for row i: take up to `budget` best candidates (scheduler.cpp:208-227).
template <class F>
MSPQ_D void phase2_select(const Ctx& x, int i, int k, F&& on_item) {
  for (int n = 0; n < x.C.budget; ++n) {
    const int key = best_candidate(x, k);
    if (key < 0) break;
    mark_scheduled(x, key);
    plan_item(x, i, key, 2);
    on_item(key);
  }
}

// Phase III: every remaining candidate by (first_use, key) (scheduler.cpp:229-241)
template <class F>
MSPQ_D void phase3_flush(const Ctx& x, int i, int k, F&& on_item) {
  const int n = x.C.L * x.C.E;
  for (int f = 0; f < k; ++f)
    for (int base = 0; base < n; base += 32) {
      const int key = base + lane_id();
      const bool m = key < n && ((volatile int*)x.C.cand_first)[key] == f;
      unsigned bal = __ballot_sync(0xffffffffu, m);
      while (bal) {
        const int b = __ffs(bal) - 1;
        bal &= bal - 1;
        const int kk = base + b;
        mark_scheduled(x, kk);
        plan_item(x, i, kk, 3);
        on_item(kk);
      }
    }
}

MSPQ_D void clear_planner(const Ctx& x) {
  const int n = x.C.L * x.C.E;
  for (int key = lane_id(); key < n; key += 32) {
    V(x.C.cand_first)[key] = -1;
    ((volatile unsigned char*)x.C.sched)[key] = 0;
    ((volatile unsigned char*)x.C.snap)[key] = contains(x, key) ? 1 : 0;
  }
  __syncwarp();
}

MSPQ_D void t12(int k, double f1, double f2, int& t1, int& t2) {
  t1 = (int)floor(f1 * k + 1e-9);
  t2 = (int)floor(f2 * k + 1e-9);
}

// sorted copy of a cell's experts as keys (required sets are std::set-ordered)
MSPQ_D int sorted_keys(const int32_t* ids, int K, int l, int E, int* out) {
  int n = 0;
  for (int j = 0; j < K; ++j) {
    int key = l * E + ids[j];
    bool dup = false;
    for (int q = 0; q < n; ++q) dup |= out[q] == key;
    if (dup) continue;
    int p = n++;
    while (p > 0 && out[p - 1] > key) {
      out[p] = out[p - 1];
      --p;
    }
    out[p] = key;
  }
  return n;
}

}  // namespace

// =============================================================== live engine
MSPQ_D void body_begin_cycle(CtlDev C, int k) {
  Ctx x{C, {C.elb_ids, C.elb_gates, nullptr, k}};
  int t1, t2;
  t12(k, C.f1, C.f2, t1, t2);
  put(x, S_K, k);
  put(x, S_T1, t1);
  put(x, S_T2, t2);
  for (int s : {S_NREQ, S_NLOG, S_NPLAN, S_FETCHED, S_DEMAND, S_JIT, S_OVERFLOW}) put(x, s, 0);
  clear_planner(x);
  publish(x);
}

// After draft row i: Phase II selection / Phase III flush with immediate (causal) inserts.
MSPQ_D void body_plan_row(CtlDev C, int i) {
  const int k = V(C.scal)[S_K];
  Ctx x{C, {C.elb_ids, C.elb_gates, nullptr, k}};
  put(x, S_NREQ, 0);
  if (C.policy != POL_SPECULATIVE || k == 0) {
    publish(x);
    return;
  }
  const int t1 = get(x, S_T1), t2 = get(x, S_T2);
  absorb_row(x, i, C.snap);
  auto ins = [&](int key) {
    prefetch_insert(x, key, true, 0, i + 1, EV_PLAN2 + 0, i);
  };
  auto ins3 = [&](int key) {
    if (!contains(x, key)) prefetch_insert(x, key, true, 0, i + 1, EV_PLAN3, i);
  };
  if (i >= t1 && i < t2) {
    if (C.budget > 0) phase2_select(x, i, k, ins);
  } else if (i >= t2) {
    phase3_flush(x, i, k, ins3);
  }
  if (i == k - 1 && t2 >= k) phase3_flush(x, i, k, ins3);
  release_pending(x);
  publish(x);
}

// Verify layer l over nslots window slots (slot s < k has ELB row s; slot k is unpredicted).
// tgt[s*K + j] = target expert ids.  Emits the per-expert first-request buffer table.
MSPQ_D void body_verify_layer(CtlDev C, int l, int nslots, const int32_t* __restrict__ tgt,
                                   int32_t* __restrict__ gbuf_out) {
  const int k = V(C.scal)[S_K];
  Ctx x{C, {C.elb_ids, C.elb_gates, nullptr, k}};
  const int E = C.E, K = C.K, L = C.L;
  __shared__ int gbuf[1024];
  // the layer's targets come from K1 in global memory; one warp-wide load instead of lane 0's
  // serial reads
  __shared__ int tgt_sm[1024];
  if (nslots * K <= 1024) {
    for (int i = lane_id(); i < nslots * K; i += 32) tgt_sm[i] = tgt[i];
    __syncwarp();
    tgt = tgt_sm;
  }
  x.gb = gbuf;
  x.step_layer = l;
  put(x, S_NREQ, 0);
  for (int e = lane_id(); e < E; e += 32) gbuf[e] = -2;
  __syncwarp();
  // coverage of the layer's required union before this step mutates anything
  {
    int hits = 0, size = 0;
    if (lane_id() == 0) {
      unsigned char seen[1024];
      for (int e = 0; e < E; ++e) seen[e] = 0;
      for (int s = 0; s < nslots; ++s)
        for (int j = 0; j < K; ++j) {
          int e = tgt[s * K + j];
          if (!seen[e]) {
            seen[e] = 1;
            ++size;
            hits += contains(x, l * E + e) ? 1 : 0;
          }
        }
      C.cov[l * 2 + 0] = hits;
      C.cov[l * 2 + 1] = size;
    }
    __syncwarp();
  }
  const int pol = C.policy;
  const bool sooner = pol == POL_SP_SOONER && L == 1;
  const bool later = pol == POL_SP_LATER || (pol == POL_SP_SOONER && L > 1);
  auto jit_cell = [&](int row) {
    for (int j = 0; j < K; ++j) {
      const int key = l * E + C.elb_ids[((int64_t)row * L + l) * K + j];
      if (prefetch_insert(x, key, false, row, INT_MAX, EV_JIT, row)) add(x, S_JIT, 1);
    }
  };
  if (sooner && nslots > 0 && k > 0) jit_cell(0);
  for (int s = 0; s < nslots; ++s) {
    const int row = s < k ? s : -1;
    if (later && row >= 0) jit_cell(row);
    if (sooner && s + 1 < nslots && s + 1 < k) jit_cell(s + 1);
    if (pol == POL_SPECULATIVE && row >= 0) {
      for (int j = 0; j < K; ++j) {
        const int key = l * E + C.elb_ids[((int64_t)row * L + l) * K + j];
        if (!contains(x, key) && prefetch_insert(x, key, true, row, INT_MAX, EV_REFILL, row))
          add(x, S_JIT, 1);
      }
    }
    int keys[64];
    const int n = sorted_keys(tgt + s * K, K, l, E, keys);
    int hits = 0;
    for (int q = 0; q < n; ++q) hits += contains(x, keys[q]) ? 1 : 0;
    if (lane_id() == 0) {
      C.step[(l * nslots + s) * 2 + 0] = hits;
      C.step[(l * nslots + s) * 2 + 1] = n;
    }
    for (int q = 0; q < n; ++q) {
      policy_step(x, keys[q], s, s);
      const int e = keys[q] - l * E;
      if (lane_id() == 0 && gbuf[e] == -2) gbuf[e] = V(C.res)[keys[q]];
      __syncwarp();
    }
  }
  // first-request buffer of every expert of this layer (-2 = not required): the grouped-GEMM
  // schedule (k_build_schedule) reads it; the host waits on exactly these buffers' copies.
  for (int e = lane_id(); e < E; e += 32) {
    gbuf_out[e] = gbuf[e];
    if (C.hsched) ((volatile int*)C.hsched)[1 + e] = gbuf[e];
  }
  if (lane_id() == 0 && C.hsched) ((volatile int*)C.hsched)[0] = E;
  __syncwarp();
  release_pending(x);
  publish(x);
}

// =============================================================== replay (token-major, exact)
// One speculative cycle of Engine::run (sim.cpp:118-295) over trace positions [pos, pos+k):
// plan + phase-2 inserts, coverage, the token-major slot loop.  Modeled times are NOT
// computed here; the host restates the lane arithmetic from the emitted counts.
MSPQ_D void body_replay_cycle(CtlDev C, ReplayTrace tr, int pos, int k_eff, int head_pos,
                                   ReplayOut out) {
  const int L = C.L, K = C.K, E = C.E;
  const int64_t rs = (int64_t)L * K;
  // the cycle's ELB rows are read by every Belady next-use scan: keep them in shared memory when
  // they fit (the serial global-memory scans dominated the replay kernel)
  __shared__ int elb_sm[4096];
  const int32_t* elb_src = tr.draft + pos * rs;
  if ((int64_t)k_eff * rs <= 4096) {
    for (int i = lane_id(); i < k_eff * rs; i += 32) elb_sm[i] = elb_src[i];
    __syncwarp();
    elb_src = elb_sm;
  }
  Ctx x{C, {elb_src, nullptr, tr.gates ? tr.gates + pos * rs : nullptr, k_eff}};
  x.emit = false;
  for (int s : {S_NREQ, S_NLOG, S_NPLAN, S_FETCHED, S_DEMAND, S_JIT, S_OVERFLOW}) put(x, s, 0);
  __shared__ unsigned char required[8192];
  for (int key = lane_id(); key < L * E; key += 32) required[key] = 0;
  __syncwarp();
  const int nwin = (head_pos >= 0 ? 1 : 0) + k_eff;
  auto win_pos = [&](int w) { return head_pos >= 0 ? (w == 0 ? head_pos : pos + w - 1) : pos + w; };
  auto win_row = [&](int w) { return head_pos >= 0 ? w - 1 : w; };
  for (int i = lane_id(); i < nwin * L * K; i += 32) {  // idempotent marks: lane-parallel
    const int w = i / (L * K), r = i - w * (L * K), l = r / K;
    required[l * E + tr.target[(int64_t)win_pos(w) * rs + r]] = 1;
  }
  __syncwarp();

  // ---- plan_prefetch over the full ELB against the cache as it is now
  int nflush = 0;
  if (C.policy == POL_SPECULATIVE && k_eff > 0) {
    clear_planner(x);  // snap = residency now
    int t1, t2;
    t12(k_eff, C.f1, C.f2, t1, t2);
    auto noop = [&](int) {};
    bool flushed = false;
    for (int i = 0; i < k_eff; ++i) {
      if (i < t1) {
        absorb_row(x, i, nullptr);
        continue;
      }
      if (i < t2) {
        absorb_row(x, i, nullptr);
        if (C.budget > 0) phase2_select(x, i, k_eff, noop);
        continue;
      }
      for (int r = 0; r < k_eff; ++r) absorb_row(x, r, nullptr);
      phase3_flush(x, i, k_eff, noop);
      flushed = true;
      break;
    }
    if (!flushed && t2 >= k_eff) {
      for (int r = 0; r < k_eff; ++r) absorb_row(x, r, nullptr);
      phase3_flush(x, k_eff - 1, k_eff, noop);
    }
    // apply: batches by issue row (sim.cpp:185-210)
    const int np = get(x, S_NPLAN);
    int nb = 0;
    int i = 0;
    while (i < np) {
      const int issue = C.plan[i * 3 + 0];
      int count = 0, has_req = 0;
      while (i < np && C.plan[i * 3 + 0] == issue) {
        const int key = C.plan[i * 3 + 1], phase = C.plan[i * 3 + 2];
        if (phase == 3) {
          if (!contains(x, key)) {
            if (lane_id() == 0) out.flush_keys[nflush] = key;
            ++nflush;
            ++count;
            has_req |= required[key];
          }
        } else if (prefetch_insert(x, key, true, 0, INT_MAX, EV_PLAN2, issue)) {
          ++count;
          has_req |= required[key];
        }
        ++i;
      }
      if (count > 0) {
        if (lane_id() == 0) {
          out.batches[nb * 3 + 0] = issue;
          out.batches[nb * 3 + 1] = count;
          out.batches[nb * 3 + 2] = has_req;
        }
        ++nb;
      }
    }
    if (lane_id() == 0) out.counts[R_NBATCH] = nb;
  } else if (lane_id() == 0) {
    out.counts[R_NBATCH] = 0;
  }
  __syncwarp();

  // ---- coverage at verification start (sim.cpp:212-224)
  if (lane_id() == 0)
    for (int l = 0; l < L; ++l) {
      unsigned char seen[1024];
      for (int e = 0; e < E; ++e) seen[e] = 0;
      int hits = 0, size = 0;
      for (int w = 0; w < nwin; ++w)
        for (int j = 0; j < K; ++j) {
          const int e = tr.target[(int64_t)win_pos(w) * rs + l * K + j];
          if (!seen[e]) {
            seen[e] = 1;
            ++size;
            hits += contains(x, l * E + e) ? 1 : 0;
          }
        }
      out.cov[l * 2 + 0] = hits;
      out.cov[l * 2 + 1] = size;
    }
  __syncwarp();

  // ---- token-major slots (sim.cpp:229-295)
  const int pol = C.policy;
  const bool sooner = pol == POL_SP_SOONER, later = pol == POL_SP_LATER;
  const int nslots = nwin * L;
  auto slot_row = [&](int s) { return win_row(s / L); };
  auto slot_layer = [&](int s) { return s % L; };
  auto add_jit = [&](int row, int key) {
    if (lane_id() == 0) {
      out.jit_rows[row * 2 + 0] += 1;
      out.jit_rows[row * 2 + 1] |= required[key];
    }
    __syncwarp();
  };
  if (lane_id() == 0)
    for (int r = 0; r < k_eff; ++r) out.jit_rows[r * 2 + 0] = out.jit_rows[r * 2 + 1] = 0;
  __syncwarp();
  auto jit_cell = [&](int row, int layer) {
    for (int j = 0; j < K; ++j) {
      const int key = layer * E + x.elb.ids[((int64_t)row * L + layer) * K + j];
      if (prefetch_insert(x, key, false, row, INT_MAX, EV_JIT, row)) add_jit(row, key);
    }
  };
  if (sooner && nslots > 0 && slot_row(0) >= 0) jit_cell(slot_row(0), slot_layer(0));
  bool flush_applied = nflush == 0;
  for (int s = 0; s < nslots; ++s) {
    const int row = slot_row(s), l = slot_layer(s), w = s / L;
    if (!flush_applied && row >= 0) {
      for (int q = 0; q < nflush; ++q) prefetch_insert(x, out.flush_keys[q], true, 0, INT_MAX, EV_PLAN3, -1);
      flush_applied = true;
    }
    if (later && row >= 0) jit_cell(row, l);
    if (sooner && s + 1 < nslots && slot_row(s + 1) >= 0) jit_cell(slot_row(s + 1), slot_layer(s + 1));
    if (pol == POL_SPECULATIVE && row >= 0 && l == 0) {
      for (int ll = 0; ll < L; ++ll)
        for (int j = 0; j < K; ++j) {
          const int key = ll * E + x.elb.ids[((int64_t)row * L + ll) * K + j];
          if (!contains(x, key) && prefetch_insert(x, key, true, row, INT_MAX, EV_REFILL, row))
            add_jit(row, key);
        }
    }
    int keys[64];
    const int n = sorted_keys(tr.target + (int64_t)win_pos(w) * rs + l * K, K, l, E, keys);
    int hits = 0;
    for (int q = 0; q < n; ++q) hits += contains(x, keys[q]) ? 1 : 0;
    if (lane_id() == 0) {
      out.step[s * 2 + 0] = hits;
      out.step[s * 2 + 1] = n;
    }
    __syncwarp();
    for (int q = 0; q < n; ++q) policy_step(x, keys[q], max(row, 0), w);
  }
  if (lane_id() == 0) {
    out.counts[R_FETCHED] = V(C.scal)[S_FETCHED];
    out.counts[R_DEMAND] = V(C.scal)[S_DEMAND];
    out.counts[R_NPLAN] = V(C.scal)[S_NPLAN];
    out.counts[R_NLOG] = V(C.scal)[S_NLOG];
    out.counts[R_OVERFLOW] = V(C.scal)[S_OVERFLOW];
  }
  __syncwarp();
  release_pending(x);
  publish(x);
}

// ---------------------------------------------------------------- shared-memory staging
// The whole cache/planner state (and the live ELB ids) is copied into shared memory by the
// CTA's 256 threads, warp 0 runs the control logic at smem latency, and the mutable state is
// written back.  Falls back to global memory when the state does not fit (stage_bytes == 0).
MSPQ_HD size_t al16(size_t b) { return (b + 15) & ~(size_t)15; }
MSPQ_HD size_t stage_bytes_of(int L, int E, int K, int nbuf, int kmax, bool elb) {
  const size_t n = (size_t)L * E;
  return al16(n * 4) + al16(n * 8) + 16 + al16(L * 4) + al16(S_COUNT * 4) + 2 * al16((size_t)(nbuf + 1) * 4) +
         2 * al16(n) + al16(n * 4) + al16(n * 8) + al16(L * 4) + (elb ? al16((size_t)kmax * L * K * 4) : 0);
}

// State copies between global memory and the shared-memory stage use 16-byte vectors. Both sides
// are padded to 16 bytes (global arrays to 256), so rounding the byte count up is safe.
// Several arrays in one pass: every thread issues up to 8 independent 16-byte loads before its
// stores, so the whole stage costs ~2 memory round trips instead of one or more per array (the
// per-array loop spent ~8 us in and ~6 us out of a ~32 us verify-layer launch).
struct StageSeg {
  void* d;
  const void* s;
  int n16;
};
template <int NS>
MSPQ_D void cp_multi(const StageSeg (&sg)[NS], int ns) {
  int total = 0;
  for (int i = 0; i < ns; ++i) total += sg[i].n16;
  for (int base = threadIdx.x; base < total; base += 8 * (int)blockDim.x) {
    uint4 v[8];
    uint4* dp[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      int idx = base + u * (int)blockDim.x;
      dp[u] = nullptr;
      if (idx < total) {
        int i = 0;
        while (idx >= sg[i].n16) idx -= sg[i++].n16;
        v[u] = reinterpret_cast<const uint4*>(sg[i].s)[idx];
        dp[u] = reinterpret_cast<uint4*>(sg[i].d) + idx;
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (dp[u]) *dp[u] = v[u];
  }
}
template <class T>
MSPQ_D StageSeg seg(T* d, const T* s, size_t cnt) {
  return StageSeg{(void*)d, (const void*)s, (int)((cnt * sizeof(T) + 15) / 16)};
}

MSPQ_D void stage(const CtlDev& G, CtlDev& S, unsigned char* sm, bool in, bool elb) {
  const size_t n = (size_t)G.L * G.E;
  unsigned char* p = sm;
  auto take = [&](size_t b) {
    unsigned char* q = p;
    p += al16(b);
    return q;
  };
  S.res = (int*)take(n * 4);
  S.stamp = (unsigned long long*)take(n * 8);
  S.clock = (unsigned long long*)take(16);
  S.lsize = (int*)take(G.L * 4);
  S.scal = (int*)take(S_COUNT * 4);
  S.free_stack = (int*)take((size_t)(G.nbuf + 1) * 4);
  S.pending = (int*)take((size_t)(G.nbuf + 1) * 4);
  S.snap = (unsigned char*)take(n);
  S.sched = (unsigned char*)take(n);
  S.cand_first = (int*)take(n * 4);
  S.cand_conf = (double*)take(n * 8);
  S.cap = (int*)take(G.L * 4);
  if (elb) S.elb_ids = (int32_t*)take((size_t)G.kmax * G.L * G.K * 4);
  if (in) {
    const StageSeg sg[13] = {seg(S.res, G.res, n),          seg(S.stamp, G.stamp, n),
                             seg(S.clock, G.clock, 1),      seg(S.lsize, G.lsize, G.L),
                             seg(S.scal, G.scal, S_COUNT),  seg(S.free_stack, G.free_stack, G.nbuf),
                             seg(S.pending, G.pending, G.nbuf), seg(S.snap, G.snap, n),
                             seg(S.sched, G.sched, n),      seg(S.cand_first, G.cand_first, n),
                             seg(S.cand_conf, G.cand_conf, n), seg(S.cap, G.cap, G.L),
                             seg(S.elb_ids, G.elb_ids, elb ? (size_t)G.kmax * G.L * G.K : 0)};
    cp_multi(sg, 13);
  } else {
    const StageSeg sg[11] = {seg(G.res, S.res, n),          seg(G.stamp, S.stamp, n),
                             seg(G.clock, S.clock, 1),      seg(G.lsize, S.lsize, G.L),
                             seg(G.scal, S.scal, S_COUNT),  seg(G.free_stack, S.free_stack, G.nbuf),
                             seg(G.pending, S.pending, G.nbuf), seg(G.snap, S.snap, n),
                             seg(G.sched, S.sched, n),      seg(G.cand_first, S.cand_first, n),
                             seg(G.cand_conf, S.cand_conf, n)};
    cp_multi(sg, 11);
  }
}

// copy requests are accumulated in device memory and written to the host-mapped queue in one
// coalesced pass at kernel exit (the host reads them after the launch's event)
MSPQ_D void flush_requests(const CtlDev& G, const CtlDev& S) {
  const int n = min(((volatile int*)S.scal)[S_NREQ], G.req_cap);
  const int4* src = reinterpret_cast<const int4*>(G.req_dev);
  volatile int* dst = (volatile int*)G.req;
  for (int i = threadIdx.x; i < n * 3; i += blockDim.x) dst[i] = G.req_dev[i];
  (void)src;
}

// ------------------------------------------------------------------ whole-trace replay
// The governor in IEEE double with explicit round-to-nearest ops (no FMA contraction), the same
// operation sequence as engine.cpp / perfmodel.cpp, so select_k picks the host's k bit for bit.
MSPQ_D double gv_k_accept(const double* p, int k) {  // perfmodel.cpp:85-97
  double sum = 0.0, prefix = 1.0;
  for (int i = 0; i < k; ++i) {
    prefix = __dmul_rn(prefix, p[i]);
    sum = __dadd_rn(sum, prefix);
  }
  return sum;
}
MSPQ_D double gv_t_verify(const GovDev& g, double window) {  // perfmodel.cpp:112-123
  int hi = 1;
  while (hi + 1 < g.nvs && g.vs_x[hi] < window) ++hi;
  const double x0 = g.vs_x[hi - 1], y0 = g.vs_y[hi - 1], x1 = g.vs_x[hi], y1 = g.vs_y[hi];
  const double t = __ddiv_rn(__dsub_rn(window, x0), __dsub_rn(x1, x0));
  return __dadd_rn(y0, __dmul_rn(t, __dsub_rn(y1, y0)));
}
MSPQ_D double gv_t_cycle(const GovDev& g, int k, int n) {  // perfmodel.cpp:99-128
  const double td = __dadd_rn(g.draft_base, __dmul_rn((double)k, g.draft_tok));
  const double tp = n == 0 ? 0.0 : __dadd_rn(g.overhead, __ddiv_rn(__dmul_rn((double)n, g.expert_bytes), g.pcie_bw));
  return __dadd_rn(__dadd_rn(fmax(td, g.init_lat), tp), gv_t_verify(g, (double)(k + 1)));
}
MSPQ_D int gv_select_k(const GovDev& g, const double* p, double gg) {  // perfmodel.cpp:166-183
  const int hi = min(g.k_max, g.k_slo);
  int best_k = g.k_min;
  double best = -1.0;
  for (int k = g.k_min; k <= hi; ++k) {
    const int est = (int)llround(__dmul_rn(gg, (double)k));
    const double v = __ddiv_rn(gv_k_accept(p, k), gv_t_cycle(g, k, est));
    if (v > best) {
      best = v;
      best_k = k;
    }
  }
  return best_k;
}

MSPQ_D void body_replay_all(CtlDev C, ReplayTrace tr, const unsigned char* acc, int n, GovDev gv, ReplayAllOut o) {
  __shared__ double p[64];
  __shared__ int k_sh;
  const int lane = lane_id();
  for (int i = lane; i < gv.kcap; i += 32) p[i] = gv.initial_accept;
  double gg = (double)C.L * (double)C.K;
  int pos = 0, head_pos = -1, ci = 0;
  __syncwarp();
  while (pos < n) {
    const int rem = n - pos;
    if (lane == 0) k_sh = gv.use_gov ? gv_select_k(gv, p, gg) : gv.fixed_k;
    __syncwarp();
    const int k_eff = min(k_sh, rem);
    int* sl = o.slices + (size_t)ci * o.stride;
    ReplayOut oc{sl, sl + o.o_batch, sl + o.o_jit, sl + o.o_cov, sl + o.o_step, o.flush_keys};
    body_replay_cycle(C, tr, pos, k_eff, head_pos, oc);
    __syncwarp();
    const int fetched = ((volatile int*)sl)[R_FETCHED];
    int accepted = 0;
    while (accepted < k_eff && acc[pos + accepted]) ++accepted;
    const int consumed = min(accepted + 1, rem);
    const int bonus = consumed - min(accepted, consumed);
    if (lane == 0) {
      o.k_eff[ci] = k_eff;
      // EMA over the outcomes up to and including the first rejection (perfmodel.cpp:206-217)
      for (int i = 0; i < k_eff && i < gv.kcap; ++i) {
        const bool ok = acc[pos + i] != 0;
        p[i] = __dadd_rn(__dmul_rn(__dsub_rn(1.0, gv.alpha), p[i]), __dmul_rn(gv.alpha, ok ? 1.0 : 0.0));
        if (!ok) break;
      }
    }
    gg = __ddiv_rn((double)fetched, (double)k_eff);
    head_pos = bonus > 0 ? pos + accepted : -1;
    pos += consumed;
    ++ci;
    __syncwarp();
  }
  if (lane == 0) *o.n_cycles = ci;
}

// STAGED is a template parameter so the state pointers' address space (shared vs global) is
// known at compile time inside the control logic.
#define CTL_KERNEL(NAME, BODY, ELB, PARAMS, ARGS)                   \
  template <bool STAGED>                                            \
  __global__ void __launch_bounds__(256) NAME PARAMS {              \
    pdl_enter(); /* launched with launch_pdl (kernels.h) */         \
    extern __shared__ __align__(16) unsigned char ctl_sm[];         \
    CtlDev S = C;                                                   \
    if constexpr (STAGED) {                                         \
      stage(C, S, ctl_sm, true, ELB);                               \
      __syncthreads();                                              \
    }                                                               \
    if (threadIdx.x < 32) BODY ARGS;                                \
    __syncthreads();                                                \
    flush_requests(C, S);                                           \
    if constexpr (STAGED) stage(C, S, ctl_sm, false, ELB);          \
  }

CTL_KERNEL(k_ctl_begin_cycle, body_begin_cycle, true, (CtlDev C, int k), (S, k))
CTL_KERNEL(k_ctl_plan_row, body_plan_row, true, (CtlDev C, int i), (S, i))
CTL_KERNEL(k_ctl_verify_layer, body_verify_layer, true,
           (CtlDev C, int l, int nslots, const int32_t* tgt, int32_t* gbuf), (S, l, nslots, tgt, gbuf))
CTL_KERNEL(k_ctl_replay_cycle, body_replay_cycle, false,
           (CtlDev C, ReplayTrace tr, int pos, int k_eff, int head_pos, ReplayOut o), (S, tr, pos, k_eff, head_pos, o))

CTL_KERNEL(k_ctl_replay_all, body_replay_all, false,
           (CtlDev C, ReplayTrace tr, const unsigned char* acc, int n, GovDev gv, ReplayAllOut o),
           (S, tr, acc, n, gv, o))

size_t ctl_stage_bytes(const CtlDev& C, bool elb) {
  const size_t b = stage_bytes_of(C.L, C.E, C.K, C.nbuf, C.kmax, elb);
  return b + 16 * 1024 <= 227 * 1024 ? b : 0;  // leave room for the kernels' static smem
}

__global__ void k_ctl_reset(CtlDev C, int nbuf) {
  const int n = C.L * C.E;
  for (int key = lane_id(); key < n; key += 32) {
    C.res[key] = -1;
    C.stamp[key] = 0;
    C.cand_first[key] = -1;
    C.sched[key] = 0;
    C.snap[key] = 0;
  }
  for (int l = lane_id(); l < C.L; l += 32) C.lsize[l] = 0;
  for (int b = lane_id(); b < nbuf; b += 32) C.free_stack[b] = nbuf - 1 - b;
  __syncwarp();
  if (lane_id() == 0) {
    for (int s = 0; s < S_COUNT; ++s) C.scal[s] = 0;
    C.scal[S_NFREE] = nbuf;
    *C.clock = 0;
  }
}

cudaError_t ctl_reset(const CtlDev& C, int nbuf, cudaStream_t st) {
  k_ctl_reset<<<1, 32, 0, st>>>(C, nbuf);
  return cudaGetLastError();
}
template <class K>
static size_t prep(K kern, const CtlDev& C, bool elb) {
  const size_t b = ctl_stage_bytes(C, elb);
  // one constant limit (the largest stage ctl_stage_bytes admits): replays of different configs run
  // concurrently from several host threads (replay_many), and a per-launch size could be lowered by
  // another thread between its set and this launch
  if (b > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 211 * 1024);
  return b;
}
#define CTL_LAUNCH(KERN, ELB, ...)                                                          \
  do {                                                                                      \
    cudaError_t e_ = C.stage ? launch_pdl(KERN<true>, dim3(1), dim3(256), prep(KERN<true>, C, ELB), \
                                          st, __VA_ARGS__)                                  \
                             : launch_pdl(KERN<false>, dim3(1), dim3(32), 0, st, __VA_ARGS__);     \
    if (e_ != cudaSuccess) return e_;                                                       \
  } while (0)
cudaError_t ctl_begin_cycle(const CtlDev& C, int k, cudaStream_t st) {
  CTL_LAUNCH(k_ctl_begin_cycle, true, C, k);
  return cudaGetLastError();
}
cudaError_t ctl_plan_row(const CtlDev& C, int i, cudaStream_t st) {
  CTL_LAUNCH(k_ctl_plan_row, true, C, i);
  return cudaGetLastError();
}
cudaError_t ctl_verify_layer(const CtlDev& C, int l, int nslots, const int32_t* tgt, int32_t* gbuf,
                             cudaStream_t st) {
  CTL_LAUNCH(k_ctl_verify_layer, true, C, l, nslots, tgt, gbuf);
  return cudaGetLastError();
}
cudaError_t ctl_replay_cycle(const CtlDev& C, const ReplayTrace& tr, int pos, int k_eff,
                             int head_pos, const ReplayOut& o, cudaStream_t st) {
  CTL_LAUNCH(k_ctl_replay_cycle, false, C, tr, pos, k_eff, head_pos, o);
  return cudaGetLastError();
}

cudaError_t ctl_replay_all(const CtlDev& C, const ReplayTrace& tr, const unsigned char* acc, int n,
                           const GovDev& gv, const ReplayAllOut& o, cudaStream_t st) {
  CTL_LAUNCH(k_ctl_replay_all, false, C, tr, acc, n, gv, o);
  return cudaGetLastError();
}

}  // namespace mspq
