// Device cache-controller interface (K4).  See ctl.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace mspq {

enum CtlMode : int { CTL_PER_LAYER = 0, CTL_GLOBAL = 1 };
// Policy ordinals follow moespeq::Policy (scheduler.hpp:95-101)
enum CtlPolicy : int { POL_LRU = 0, POL_LOOKAHEAD = 1, POL_SP_SOONER = 2, POL_SP_LATER = 3, POL_SPECULATIVE = 4 };
// event kinds in the hit/miss log
enum CtlEvent : int { EV_DEMAND = 0, EV_PLAN2 = 1, EV_PLAN3 = 2, EV_JIT = 3, EV_REFILL = 4 };
// device scalar slots
enum CtlScalar : int {
  S_TOTAL = 0, S_NFREE, S_NPEND, S_K, S_T1, S_T2, S_NREQ, S_NLOG, S_NPLAN, S_FETCHED, S_DEMAND,
  S_JIT, S_OVERFLOW, S_COUNT
};
// replay per-cycle count slots
enum ReplayCount : int { R_NBATCH = 0, R_FETCHED, R_DEMAND, R_NPLAN, R_NLOG, R_OVERFLOW, R_COUNT };

struct CtlDev {
  int L, E, K, mode, policy, cap_global, budget;
  int nbuf, kmax, stage;       // stage = run launches on a shared-memory copy of the state
  double f1, f2;
  int* cap;                    // [L] per-layer capacities (entropy-weighted override allowed)
  int* res;                    // [L*E] buffer id or -1
  unsigned long long* stamp;   // [L*E] LRU recency
  unsigned long long* clock;   // [1]
  int* lsize;                  // [L]
  int* scal;                   // [S_COUNT]
  int* free_stack;             // [nbuf]
  int* pending;                // [nbuf]
  unsigned char* snap;         // [L*E] residency at plan time
  unsigned char* sched;        // [L*E] already scheduled this cycle
  int* cand_first;             // [L*E] first ELB row predicting the key, -1 = not a candidate
  double* cand_conf;           // [L*E] best confidence seen
  int32_t* elb_ids;            // [kmax][L][K] live ELB (written by the draft router)
  float* elb_gates;            // [kmax][L][K]
  int* req;                    // [req_cap][3] copy requests (key, buffer, kind), host-mapped
  int* req_dev;                // [req_cap][3] device-side accumulation of the same
  int req_cap;
  int* log;                    // [log_cap][6] (kind, tag, key, hit, victim, buffer)
  int log_cap;
  int* plan;                   // [plan_cap][3] (row, key, phase)
  int plan_cap;
  int* cov;                    // [L][2] live: (hits, size) of each layer's required union
  int* step;                   // [L][nslots][2] live: per (layer, slot) step coverage counts
  int* hstat;                  // [S_COUNT] mapped pinned host mirror of scal (written at exit)
  int* hsched;                 // [1+E] mapped: E, then first-request buffer per expert (-2 unused)
};

struct ReplayTrace {
  const int32_t* target;  // [n][L][K]
  const int32_t* draft;   // [n][L][K]
  const double* gates;    // [n][L][K] or nullptr
};

struct ReplayOut {
  int* counts;      // [R_COUNT]
  int* batches;     // [kmax][3] (issue row, count, has_required)
  int* jit_rows;    // [kmax][2] (count, has_required)
  int* cov;         // [L][2]
  int* step;        // [(kmax+1)*L][2]
  int* flush_keys;  // [L*E]
};

// Whole-trace replay in one launch (k_ctl_replay_all): the Amortization-Roofline governor runs on
// the device between cycles (perfmodel.cpp:85-217 in IEEE double, no contraction, bit-identical to
// the host's), so no per-cycle host round trip.  Per-cycle outputs go to slices of `stride` ints
// laid out like one ReplayOut (counts | batches | jit_rows | cov | step) at slot ci.
struct GovDev {
  int use_gov, fixed_k, k_min, k_max, k_slo, kcap;
  double alpha, initial_accept;
  double pcie_bw, init_lat, overhead, expert_bytes, draft_base, draft_tok;
  int nvs;
  double vs_x[16], vs_y[16];
};
struct ReplayAllOut {
  int* slices;     // [max_cycles][stride]
  int stride;      // ints per cycle slice
  int o_batch, o_jit, o_cov, o_step;  // offsets inside a slice
  int* k_eff;      // [max_cycles]
  int* n_cycles;   // [1]
  int* flush_keys; // [L*E] scratch
};
cudaError_t ctl_replay_all(const CtlDev& C, const ReplayTrace& tr, const unsigned char* acc, int n,
                           const GovDev& gv, const ReplayAllOut& o, cudaStream_t st);

size_t ctl_stage_bytes(const CtlDev& C, bool elb);
cudaError_t ctl_reset(const CtlDev& C, int nbuf, cudaStream_t st);
cudaError_t ctl_begin_cycle(const CtlDev& C, int k, cudaStream_t st);
cudaError_t ctl_plan_row(const CtlDev& C, int i, cudaStream_t st);
cudaError_t ctl_verify_layer(const CtlDev& C, int l, int nslots, const int32_t* tgt, int32_t* gbuf,
                             cudaStream_t st);
cudaError_t ctl_replay_cycle(const CtlDev& C, const ReplayTrace& tr, int pos, int k_eff,
                             int head_pos, const ReplayOut& o, cudaStream_t st);

}  // namespace mspq
