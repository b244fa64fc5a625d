"""TEST INFRASTRUCTURE ONLY — independent Python restatement of the reference control plane.

Follows, rule by rule (file:line into /root/reference/proj):
  ExpertLookaheadBuffer / build_elb / next_use      scheduler.cpp:9-63
  CacheState (PerLayer / Global, per-layer caps)    scheduler.cpp:76-138
  plan_prefetch (3 phases)                          scheduler.cpp:173-254
  select_victim_lookahead (Belady, tie -> larger)   scheduler.cpp:256-274
  policy_step (5 policies)                          scheduler.cpp:276-312
  step_coverage                                     scheduler.cpp:314-320
  reorder_verification                              scheduler.cpp:339-357
  perfmodel (k_accept, t_*, select_k, TTFT, EMA)    perfmodel.cpp:85-217
  Engine::run (the cycle loop, modeled two lanes)   sim.cpp:98-432, entropy caps sim.cpp:26-43

`simulate(trace, cfg)` reproduces run_simulation's report (pinned against oracle/_ref).
`simulate(..., order="layer")` is the layer-major restatement (identical integers in PerLayer
mode).  `live_cycle(...)` is the causal, layer-major rule set the device engine
follows in live decoding: it is this file — not the reference — that pins the
engine's live hit/miss sequence.

Every cache mutation is appended to an event log: (kind, slot_or_row, layer, expert, hit,
victim) so hit/miss *sequences* can be compared, not only aggregates.
"""
from __future__ import annotations

import math
from collections import OrderedDict

INT_MAX = 2**31 - 1
POLICIES = ["lru", "lookahead", "sp-sooner", "sp-later", "speculative"]


# ----------------------------------------------------------------------------- perfmodel
def default_profile():
    # perfmodel.hpp:15-30 defaults
    return dict(pcie_bandwidth=16e9, pcie_init_latency=20e-3, pcie_overhead=2e-3,
                expert_size_bytes=25_000_000, draft_base=5e-3, draft_per_token=3e-3,
                verify_samples=[(1.0, 10e-3), (5.0, 20e-3), (9.0, 40e-3), (17.0, 75e-3)],
                token_bytes=1.0)


def profile_from_json(j):
    p = default_profile()
    m = {"pcie_bandwidth_bytes_per_s": "pcie_bandwidth", "pcie_init_latency_s": "pcie_init_latency",
         "pcie_overhead_s": "pcie_overhead", "expert_size_bytes": "expert_size_bytes",
         "draft_base_s": "draft_base", "draft_per_token_s": "draft_per_token",
         "token_bytes": "token_bytes"}
    for k, v in j.items():
        if k == "verify_samples":
            p["verify_samples"] = [(float(a), float(b)) for a, b in v]
        elif k in m:
            p[m[k]] = v
        else:
            raise ValueError("unknown profile field: " + k)
    return p


def k_accept(p, k):  # perfmodel.cpp:85-97
    if k < 0 or k > len(p):
        raise ValueError("KOutOfRange")
    s, prefix = 0.0, 1.0
    for i in range(k):
        prefix *= p[i]
        s += prefix
    return s


def t_draft(prof, k):  # perfmodel.cpp:99-102
    return prof["draft_base"] + float(k) * prof["draft_per_token"]


def t_pcie_new(prof, n):  # perfmodel.cpp:104-110
    if n == 0:
        return 0.0
    return prof["pcie_overhead"] + float(n) * float(prof["expert_size_bytes"]) / prof["pcie_bandwidth"]


def t_verify(prof, window):  # perfmodel.cpp:112-123
    s = prof["verify_samples"]
    hi = 1
    while hi + 1 < len(s) and s[hi][0] < window:
        hi += 1
    x0, y0 = s[hi - 1]
    x1, y1 = s[hi]
    t = (window - x0) / (x1 - x0)
    return y0 + t * (y1 - y0)


def t_cycle(prof, k, n):  # perfmodel.cpp:125-128
    return max(t_draft(prof, k), prof["pcie_init_latency"]) + t_pcie_new(prof, n) + t_verify(prof, float(k + 1))


def select_k(prof, p, k_min, k_max, k_slo, est):  # perfmodel.cpp:166-183
    hi = min(k_max, k_slo)
    best_k, best = k_min, -1.0
    for k in range(k_min, hi + 1):
        v = k_accept(p, k) / t_cycle(prof, k, est(k))
        if v > best:
            best, best_k = v, k
    return best_k


def k_slo_from_ttft(prof, budget, est, k_min, k_max):  # perfmodel.cpp:185-204
    lat = lambda k: t_cycle(prof, k, est(k))
    if budget < lat(k_min):
        raise ValueError("InfeasibleBudget")
    lo, hi = k_min, k_max
    while lo < hi:
        mid = lo + (hi - lo + 1) // 2
        if lat(mid) <= budget:
            lo = mid
        else:
            hi = mid - 1
    return lo


def update_acceptance(p, alpha, outcomes):  # perfmodel.cpp:206-217
    q = list(p)
    for i, o in enumerate(outcomes):
        q[i] = (1.0 - alpha) * q[i] + alpha * (1.0 if o else 0.0)
        if not o:
            break
    return q


def llround(x):
    # std::llround: half away from zero
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


# ----------------------------------------------------------------------------- ELB
class ELB:
    """k x L grid of [(expert, confidence)] cells (scheduler.cpp:9-63)."""

    def __init__(self, rows):
        self.rows = rows  # rows[r][l] = [(expert, conf), ...]

    @staticmethod
    def build(draft_sets_rows, gates_rows=None):
        # scheduler.cpp:41-63: conf = gate / sum(gates of the cell); 1.0 when no gates or sum == 0
        rows = []
        for r, ds in enumerate(draft_sets_rows):
            g = gates_rows[r] if gates_rows is not None else None
            row = []
            for l, experts in enumerate(ds):
                cell = []
                norm = 0.0
                if g:
                    for v in g[l]:
                        norm += v
                for s, e in enumerate(experts):
                    conf = 1.0
                    if g and norm > 0.0:
                        conf = g[l][s] / norm
                    cell.append((e, conf))
                row.append(cell)
            rows.append(row)
        return ELB(rows)

    @property
    def filled(self):
        return len(self.rows)

    def next_use(self, key, now, visible=None):
        # scheduler.cpp:33-39, restricted to the first `visible` rows in causal (live) mode
        l, e = key
        end = self.filled if visible is None else min(visible, self.filled)
        for i in range(max(now, 0), end):
            for ent in self.rows[i][l]:
                if ent[0] == e:
                    return i
        return None


# ----------------------------------------------------------------------------- cache
class Cache:
    """CacheState (scheduler.cpp:76-138); recency OrderedDict front = least recent."""

    def __init__(self, mode, capacity, per_layer_caps=None):
        self.mode = mode
        self.capacity = capacity
        self.caps = per_layer_caps
        self.recency = OrderedDict()
        self.layer_sizes = {}

    def capacity_for(self, layer):
        if self.mode == "global":
            return self.capacity
        if self.caps and 0 <= layer < len(self.caps):
            return self.caps[layer]
        return self.capacity

    def contains(self, key):
        return key in self.recency

    def touch(self, key):
        if key in self.recency:
            self.recency.move_to_end(key)

    def insert(self, key):
        if self.contains(key):
            self.touch(key)
            return
        if self.needs_eviction(key[0]):
            raise RuntimeError("insert would exceed capacity")
        self.recency[key] = True
        self.layer_sizes[key[0]] = self.layer_sizes.get(key[0], 0) + 1

    def erase(self, key):
        if key in self.recency:
            del self.recency[key]
            self.layer_sizes[key[0]] -= 1

    def needs_eviction(self, layer):
        if self.mode == "global":
            return len(self.recency) >= self.capacity
        return self.layer_sizes.get(layer, 0) >= self.capacity_for(layer)

    def lru_victim(self, layer=-1):
        for key in self.recency:
            if layer < 0 or key[0] == layer:
                return key
        return None

    def resident_sorted(self):
        return sorted(self.recency.keys())


def select_victim_lookahead(cache, elb, now, layer_filter=-1, visible=None):
    # scheduler.cpp:256-274
    found, victim, victim_use = False, None, -1
    for key in cache.resident_sorted():
        if layer_filter >= 0 and key[0] != layer_filter:
            continue
        u = elb.next_use(key, now, visible)
        use_at = INT_MAX if u is None else u
        if not found or use_at > victim_use or (use_at == victim_use and key > victim):
            found, victim, victim_use = True, key, use_at
    if not found:
        raise RuntimeError("EmptyCache")
    return victim


def policy_step(policy, cache, key, elb, now, log=None, tag=None):
    # scheduler.cpp:276-312
    hit = cache.contains(key)
    victim_layer = key[0] if cache.mode == "per_layer" else -1
    evicted = None
    if policy in ("lru", "sp-sooner", "sp-later"):
        if hit:
            cache.touch(key)
        else:
            if cache.needs_eviction(key[0]):
                evicted = cache.lru_victim(victim_layer)
                cache.erase(evicted)
            cache.insert(key)
    else:
        if not hit:
            if cache.needs_eviction(key[0]):
                evicted = select_victim_lookahead(cache, elb, now, victim_layer)
                cache.erase(evicted)
            cache.insert(key)
    if log is not None:
        log.append(("demand", tag, key[0], key[1], hit, evicted))
    return hit


# ----------------------------------------------------------------------------- planner
def _t12(k, f1, f2):
    # scheduler.cpp:181-182: floor with a 1e-9 nudge
    return int(math.floor(f1 * k + 1e-9)), int(math.floor(f2 * k + 1e-9))


def plan_prefetch(elb, contains, budget, f1=0.25, f2=0.75):
    """scheduler.cpp:173-254.  `contains(key)` = residency at plan time."""
    k = elb.filled
    items = []
    if k == 0:
        return items
    t1, t2 = _t12(k, f1, f2)
    cands = {}  # key -> [conf, first_use]
    scheduled = set()

    def absorb(row):
        for l, cell in enumerate(elb.rows[row]):
            for e, conf in cell:
                key = (l, e)
                if contains(key) or key in scheduled:
                    continue
                if key not in cands:
                    cands[key] = [conf, row]
                else:
                    cands[key][0] = max(cands[key][0], conf)

    def flush_sorted():
        return sorted(cands.items(), key=lambda kv: (kv[1][1], kv[0]))

    for i in range(k):
        if i < t1:
            absorb(i)
            continue
        if i < t2:
            absorb(i)
            if budget <= 0:
                continue
            pool = sorted(cands.items(),
                          key=lambda kv: (-(kv[1][0] * float(k - kv[1][1]) / k), kv[1][1], kv[0]))
            for key, _ in pool[:min(budget, len(pool))]:
                items.append((i, key, 2))
                scheduled.add(key)
                del cands[key]
            continue
        for row in range(k):
            absorb(row)
        for key, _ in flush_sorted():
            items.append((i, key, 3))
            scheduled.add(key)
        cands.clear()
        break
    if t2 >= k and k > 0:
        for row in range(k):
            absorb(row)
        for key, _ in flush_sorted():
            items.append((k - 1, key, 3))
    return items


class CausalPlanner:
    """Row-by-row execution of plan_prefetch for a live engine: row i may only see ELB rows
    <= i.  Candidates are filtered against the residency snapshot taken at cycle start (as the
    reference's plan_prefetch sees a const cache).  Phase-II selections are identical to the
    reference's; Phase-III items come out in the identical (first_use, key) order, but keys
    first predicted in a row r > t2 are issued after row r instead of after row t2."""

    def __init__(self, k, budget, f1, f2, snapshot):
        self.k, self.budget = k, budget
        self.t1, self.t2 = _t12(k, f1, f2)
        self.snap = snapshot
        self.cands = {}
        self.scheduled = set()

    def _absorb(self, elb, row):
        for l, cell in enumerate(elb.rows[row]):
            for e, conf in cell:
                key = (l, e)
                if key in self.snap or key in self.scheduled:
                    continue
                if key not in self.cands:
                    self.cands[key] = [conf, row]
                else:
                    self.cands[key][0] = max(self.cands[key][0], conf)

    def row(self, elb, i):
        k, out = self.k, []
        self._absorb(elb, i)
        if self.t1 <= i < self.t2:
            if self.budget > 0:
                pool = sorted(self.cands.items(),
                              key=lambda kv: (-(kv[1][0] * float(k - kv[1][1]) / k), kv[1][1], kv[0]))
                for key, _ in pool[:min(self.budget, len(pool))]:
                    out.append((i, key, 2))
                    self.scheduled.add(key)
                    del self.cands[key]
        elif i >= self.t2:
            out += self._flush(i)
        # a phase boundary at or past the window end flushes at the last row (scheduler.cpp:243-252)
        if i == k - 1 and self.t2 >= k:
            out += self._flush(i)
        return out

    def _flush(self, i):
        out = []
        for key, _ in sorted(self.cands.items(), key=lambda kv: (kv[1][1], kv[0])):
            out.append((i, key, 3))
            self.scheduled.add(key)
        self.cands.clear()
        return out


def reorder_verification(window_tokens, routing):
    # scheduler.cpp:339-357
    plan = []
    for l, per_tok in enumerate(routing):
        groups = {}
        for i, experts in enumerate(per_tok):
            for e in experts:
                groups.setdefault(e, []).append(window_tokens[i])
        plan.append([{"expert": e, "tokens": groups[e]} for e in sorted(groups)])
    return plan


# ----------------------------------------------------------------------------- trace helpers
def parse_trace(text):
    import json
    lines = [ln for ln in text.splitlines() if ln.strip()]
    head = json.loads(lines[0])
    sh = head["shape"]
    shape = dict(L=sh["L"], N=sh["N"], top_k=sh["top_k"], shared=sh["shared"],
                 expert_bytes=sh["expert_bytes"])
    toks = []
    for ln in lines[1:]:
        r = json.loads(ln)
        L = shape["L"]
        tgt = [None] * L
        dr = [None] * L
        for l, es in r["target"]:
            tgt[l] = list(es)
        for l, es in r["draft"]:
            dr[l] = list(es)
        gates = None
        if "gates" in r:
            gates = [None] * L
            for l, gs in r["gates"]:
                gates[l] = list(gs)
        toks.append(dict(target=tgt, draft=dr, gates=gates, acc=bool(r["acc"])))
    return shape, toks


def layer_entropy(toks, layer, N):
    counts = [0] * N
    total = 0
    for t in toks:
        for e in t["target"][layer]:
            counts[e] += 1
            total += 1
    h = 0.0
    for c in counts:
        if c:
            p = c / total
            h -= p * math.log2(p)
    return h


def entropy_caps(shape, toks, base):
    # sim.cpp:26-43
    L = shape["L"]
    h = [layer_entropy(toks, l, shape["N"]) for l in range(L)]
    mean = 0.0
    for v in h:
        mean += v
    mean /= float(L)
    caps = [base] * L
    if mean <= 0.0:
        return caps
    for l in range(L):
        scaled = float(base) * h[l] / mean
        caps[l] = max(shape["top_k"], llround(scaled))
    return caps


# ----------------------------------------------------------------------------- config
def sim_config(cfg: dict):
    """Reference run-config schema (run_config.hpp:30-50) -> flat dict with defaults
    (sim.hpp:15-34)."""
    c = dict(policy="speculative", capacity_mode="per_layer", cache_capacity=8,
             entropy_weighted_capacity=False, fixed_k=4, use_governor=False, k_min=1, k_max=16,
             k_slo=16, ttft_budget=0.0, f1=0.25, f2=0.75, prefetch_budget=2, rollback=0.0,
             ema_alpha=0.1, initial_accept=0.8, collect_plans=False, profile=default_profile())
    for k, v in cfg.items():
        if k == "k":
            if v == "governor":
                c["use_governor"] = True
            else:
                c["use_governor"], c["fixed_k"] = False, int(v)
        elif k == "governor":
            c["k_min"] = v.get("k_min", 1)
            c["k_max"] = v.get("k_max", 16)
            c["k_slo"] = v.get("k_slo", 16)
            c["ttft_budget"] = v.get("ttft_budget_s", 0.0)
        elif k == "phases":
            c["f1"], c["f2"] = v.get("f1", 0.25), v.get("f2", 0.75)
        elif k == "rollback_s":
            c["rollback"] = v
        elif k == "profile":
            c["profile"] = profile_from_json(v)
        elif k in ("policy", "capacity_mode", "cache_capacity", "entropy_weighted_capacity",
                   "prefetch_budget", "ema_alpha", "initial_accept", "collect_plans", "seed",
                   "estimator", "verify_overlap", "log", "prefetch_defer"):
            c[k] = v
        else:
            raise ValueError("unknown config key " + k)
    return c


# ----------------------------------------------------------------------------- the cycle loop
def simulate(trace_text, cfg_json, order="token", log=None):
    """Engine::run (sim.cpp:98-432).  order='token' is the reference's slot order;
    order='layer' processes each layer's slots contiguously with the flush / staged refill /
    single-prefetch insertions split per layer (valid for PerLayer caches).  Returns a dict in
    SimReport::to_json's schema (sim.cpp:468-510)."""
    shape, toks = parse_trace(trace_text)
    c = sim_config(cfg_json)
    prof = dict(c["profile"])
    if shape["expert_bytes"] > 0:  # sim.cpp:54-55
        prof["expert_size_bytes"] = shape["expert_bytes"]
    L = shape["L"]
    n = len(toks)
    if n == 0:
        return dict(total_tokens=0, total_time_s=0.0, tpot_s=0.0, ttft_s=0.0, mean_coverage=0.0,
                    mean_step_coverage=0.0, mean_accepted=0.0, stall_time_s=0.0,
                    total_new_experts=0, cycles=[])
    caps = None
    if c["capacity_mode"] == "per_layer" and c["entropy_weighted_capacity"]:
        caps = entropy_caps(shape, toks, c["cache_capacity"])
    cache = Cache(c["capacity_mode"], c["cache_capacity"], caps)
    k_cap = max(c["k_max"] if c["use_governor"] else c["fixed_k"], 1)
    accept = [c["initial_accept"]] * k_cap
    g = float(L) * float(shape["top_k"])
    est = lambda gg: (lambda k: int(llround(gg * float(k))))
    k_slo = c["k_slo"]
    if c["use_governor"] and c["ttft_budget"] > 0.0:
        k_slo = min(k_slo, k_slo_from_ttft(prof, c["ttft_budget"], est(g), c["k_min"], c["k_max"]))
    policy = c["policy"]
    report = dict(stall_time_s=0.0, total_new_experts=0, cycles=[])
    now_t, pos, ci = 0.0, 0, 0
    step_cov_total, step_total, layer_cov_total, layer_cov_count, acc_total = 0.0, 0, 0.0, 0, 0
    head_pos = -1
    channel_free = 0.0
    while pos < n:
        rem = n - pos
        kk = c["fixed_k"] if not c["use_governor"] else select_k(prof, accept, c["k_min"], c["k_max"], k_slo, est(g))
        k_eff = min(kk, rem)
        t0 = now_t
        rec = dict(cycle=ci, k=k_eff, start_s=t0, segments=[])
        win_toks = toks[pos:pos + k_eff]
        elb = ELB.build([t["draft"] for t in win_toks],
                        [t["gates"] for t in win_toks] if win_toks and win_toks[0]["gates"] else None)
        draft_dur = t_draft(prof, k_eff)
        draft_end = t0 + draft_dur
        rec["segments"].append(("compute", "draft", t0, draft_dur))
        draft_done_at = lambda row: t0 + prof["draft_base"] + float(row + 1) * prof["draft_per_token"]
        window = ([(head_pos, -1)] if head_pos >= 0 else []) + [(pos + i, i) for i in range(k_eff)]
        required_union = set()
        for vpos, _ in window:
            for l in range(L):
                for e in toks[vpos]["target"][l]:
                    required_union.add((l, e))
        st = dict(fetched=0)
        batches = []

        def victim_layer(key):
            return key[0] if cache.mode == "per_layer" else -1

        def prefetch_insert(key, belady, now_row, kind, tag):
            # sim.cpp:158-177
            if cache.contains(key):
                if not belady:
                    cache.touch(key)
                return False
            ev = None
            if cache.needs_eviction(key[0]):
                if belady:
                    ev = select_victim_lookahead(cache, elb, now_row, victim_layer(key))
                else:
                    ev = cache.lru_victim(victim_layer(key))
                cache.erase(ev)
            cache.insert(key)
            st["fetched"] += 1
            if log is not None:
                log.append((kind, tag, key[0], key[1], False, ev))
            return True

        plan = []
        flush_keys = []
        if policy == "speculative":
            plan = plan_prefetch(elb, cache.contains, c["prefetch_budget"], c["f1"], c["f2"])
            i = 0
            while i < len(plan):
                issue = plan[i][0]
                b = dict(issue_time=draft_done_at(issue), count=0, has_required=False)
                while i < len(plan) and plan[i][0] == issue:
                    key, phase = plan[i][1], plan[i][2]
                    if phase == 3:
                        if not cache.contains(key):
                            flush_keys.append(key)
                            b["count"] += 1
                            if key in required_union:
                                b["has_required"] = True
                    elif prefetch_insert(key, True, 0, "plan2", issue):
                        b["count"] += 1
                        if key in required_union:
                            b["has_required"] = True
                    i += 1
                if b["count"] > 0:
                    batches.append(b)
        # coverage at verification start (sim.cpp:212-224)
        cov = []
        for l in range(L):
            req = set()
            for vpos, _ in window:
                for e in toks[vpos]["target"][l]:
                    req.add((l, e))
            v = sum(1 for key in req if cache.contains(key)) / float(len(req))
            cov.append(v)
            layer_cov_total += v
            layer_cov_count += 1
        rec["coverage"] = cov
        if order == "token" or L == 1:
            slots = [(vpos, row, l) for vpos, row in window for l in range(L)]
        else:
            slots = [(vpos, row, l) for l in range(L) for vpos, row in window]
        step_cov = {}
        demand = 0
        row_batches = {}

        def jit_cell(row, layer):
            for e, _ in elb.rows[row][layer]:
                key = (layer, e)
                if prefetch_insert(key, False, row, "jit", row):
                    b = row_batches.setdefault(row, dict(count=0, has_required=False))
                    b["count"] += 1
                    if key in required_union:
                        b["has_required"] = True

        sooner, later = policy == "sp-sooner", policy == "sp-later"
        lm = order == "layer" and L > 1
        if lm and sooner:
            # per layer, "one layer ahead" (token-major) == "at the slot" when L >= 2
            sooner, later = False, True
        if not lm:
            if sooner and slots and slots[0][1] >= 0:
                jit_cell(slots[0][1], slots[0][2])
            flush_applied = len(flush_keys) == 0
        else:
            flushed_layers = set()
        for s, (vpos, row, l) in enumerate(slots):
            if not lm:
                if not flush_applied and row >= 0:
                    for key in flush_keys:
                        prefetch_insert(key, True, 0, "flush", -1)
                    flush_applied = True
            else:
                if row >= 0 and l not in flushed_layers:
                    flushed_layers.add(l)
                    for key in flush_keys:
                        if key[0] == l:
                            prefetch_insert(key, True, 0, "flush", -1)
            if later and row >= 0:
                jit_cell(row, l)
            if sooner and s + 1 < len(slots) and slots[s + 1][1] >= 0:
                jit_cell(slots[s + 1][1], slots[s + 1][2])
            if policy == "speculative" and row >= 0:
                refill_layers = [l] if lm else range(L)
                if lm or l == 0:
                    for ll in refill_layers:
                        for e, _ in elb.rows[row][ll]:
                            key = (ll, e)
                            if not cache.contains(key) and prefetch_insert(key, True, row, "refill", row):
                                b = row_batches.setdefault(row, dict(count=0, has_required=False))
                                b["count"] += 1
                                if key in required_union:
                                    b["has_required"] = True
            now_row = max(row, 0)
            req = sorted({(l, e) for e in toks[vpos]["target"][l]})
            step_cov[(vpos, row, l)] = sum(1 for key in req if cache.contains(key)) / float(len(req))
            for key in req:
                was = cache.contains(key)
                policy_step(policy, cache, key, elb, now_row, log, (vpos, row))
                if not was:
                    st["fetched"] += 1
                    demand += 1
        # step coverage mean in the reference's (token-major) summation order
        step_cov_sum = 0.0
        for vpos, row in window:
            for l in range(L):
                step_cov_sum += step_cov[(vpos, row, l)]
        step_count = len(slots)
        jit_batches = [row_batches[r] for r in sorted(row_batches) if row_batches[r]["count"] > 0]
        # I/O lane (sim.cpp:302-347)
        any_req = demand > 0 or any(b["has_required"] for b in batches) or any(
            b["has_required"] for b in jit_batches)
        p0 = draft_end
        channel = max(t0, channel_free)
        if any_req:
            init_start = channel
            channel = init_start + prof["pcie_init_latency"]
            rec["segments"].append(("io", "io_init", init_start, prof["pcie_init_latency"]))
            p0 = max(draft_end, channel)
        required_drain = p0
        S, B = float(prof["expert_size_bytes"]), prof["pcie_bandwidth"]
        for b in batches:
            b["start"] = max(b["issue_time"], channel)
            dur = prof["pcie_overhead"] + float(b["count"]) * S / B
            b["end"] = b["start"] + dur
            channel = b["end"]
            rec["segments"].append(("io", "io_new", b["start"], dur))
            if b["has_required"]:
                required_drain = max(required_drain, b["end"])
        for b in jit_batches:
            b["start"] = max(p0, channel)
            dur = prof["pcie_overhead"] + float(b["count"]) * S / B
            b["end"] = b["start"] + dur
            channel = b["end"]
            rec["segments"].append(("io", "io_new", b["start"], dur))
            if b["has_required"]:
                required_drain = max(required_drain, b["end"])
        sync_dur = t_pcie_new(prof, demand)
        io_wait = max(0.0, required_drain - p0)
        if demand > 0:
            io_wait = max(io_wait, channel - p0)
        if sync_dur > 0.0:
            rec["segments"].append(("io", "io_new", p0 + io_wait, sync_dur))
            channel = max(channel, p0 + io_wait + sync_dur)
        channel_free = channel
        verify_start = p0 + io_wait + sync_dur
        verify_dur = t_verify(prof, float(k_eff + 1))
        rec["segments"].append(("compute", "verify", verify_start, verify_dur))
        cycle_end = verify_start + verify_dur
        accepted = 0
        while accepted < k_eff and toks[pos + accepted]["acc"]:
            accepted += 1
        if accepted < k_eff and c["rollback"] > 0.0:
            rec["segments"].append(("compute", "rollback", cycle_end, c["rollback"]))
            cycle_end += c["rollback"]
        consumed = min(accepted + 1, rem)
        bonus = consumed - min(accepted, consumed)
        rec["accepted"] = consumed - bonus
        rec["bonus"] = bonus
        head_pos = pos + accepted if bonus > 0 else -1
        rec["step_coverage"] = step_cov_sum / step_count if step_count > 0 else 0.0
        rec["steps"] = step_count
        rec["new_experts"] = st["fetched"]
        rec["bytes"] = st["fetched"] * prof["expert_size_bytes"]
        rec["io_wait_s"] = io_wait
        rec["sync_fetch_s"] = sync_dur
        rec["sync_count"] = demand
        rec["span_s"] = cycle_end - t0
        if c["collect_plans"]:
            rec["prefetch_plan"] = [dict(issue_after_token=it[0], layer=it[1][0], expert=it[1][1],
                                         phase=it[2]) for it in plan]
            wpos = [vp for vp, _ in window]
            routing = [[toks[vp]["target"][l] for vp, _ in window] for l in range(L)]
            rec["execution_plan"] = [dict(layer=l, groups=grp) for l, grp in
                                     enumerate(reorder_verification(wpos, routing))]
        outcomes = []
        for i in range(k_eff):
            ok = toks[pos + i]["acc"]
            outcomes.append(ok)
            if not ok:
                break
        outcomes = outcomes[:len(accept)]
        accept = update_acceptance(accept, c["ema_alpha"], outcomes)
        g = float(st["fetched"]) / float(k_eff)
        report["stall_time_s"] += verify_start - draft_end
        step_cov_total += step_cov_sum
        step_total += step_count
        acc_total += rec["accepted"]
        report["total_new_experts"] += st["fetched"]
        report["cycles"].append(rec)
        now_t = cycle_end
        pos += consumed
        ci += 1
    report["total_tokens"] = pos
    report["total_time_s"] = now_t
    report["tpot_s"] = now_t / pos if pos else 0.0
    report["ttft_s"] = report["cycles"][0]["span_s"] if report["cycles"] else 0.0
    report["mean_coverage"] = layer_cov_total / layer_cov_count if layer_cov_count else 0.0
    report["mean_step_coverage"] = step_cov_total / step_total if step_total else 0.0
    report["mean_accepted"] = acc_total / len(report["cycles"]) if report["cycles"] else 0.0
    return report


# ----------------------------------------------------------------------------- live (causal) cycle
def live_cycle(cache, elb, targets, cfg, log=None, ids_visible_causal=True):
    """One live-engine cycle.  `elb` has k rows = the draft's routing for window
    slots 0..k-1 (slot 0 = the previous bonus token); `targets[s][l]` = the target model's
    top-k for window slot s in 0..k (slot k = last drafted token, unpredicted).

    Draft phase: CausalPlanner row by row; phase-2 and phase-3 keys are inserted right away
    (Belady now=0 over the rows drafted so far).  Verify phase: layer-major; for each layer:
    coverage, then per slot: single-prefetch JIT cells, staged refill (speculative), step
    coverage, demand policy_step in ascending expert order with now = rows verified so far.
    Returns dict of per-cycle integers; appends events to `log`."""
    L = len(targets[0])
    k = elb.filled
    policy = cfg["policy"]
    out = dict(fetched=0, demand=0, plan_items=[], coverage_hits=[], coverage_size=[],
               step_hits=[], step_size=[], jit=0, refetch=0)
    # refetch: an insertion in verify layer l of a key the layer already requested (evicted after
    # its first request): the engine serves it from the first-request buffer, still parked
    # (live.cpp issue_copies, refetch_from_hbm; ctl.cu erase)
    demanded = [None]

    def victim_layer(key):
        return key[0] if cache.mode == "per_layer" else -1

    def ins(key, belady, now_row, visible, kind, tag, touch=False):
        if cache.contains(key):
            if not belady:
                cache.touch(key)
            return False
        ev = None
        if cache.needs_eviction(key[0]):
            if belady:
                ev = select_victim_lookahead(cache, elb, now_row, victim_layer(key), visible)
            else:
                ev = cache.lru_victim(victim_layer(key))
            cache.erase(ev)
        cache.insert(key)
        out["fetched"] += 1
        if demanded[0] is not None and key in demanded[0]:
            out["refetch"] += 1
        if log is not None:
            log.append((kind, tag, key[0], key[1], False, ev))
        return True

    if policy == "speculative" and k > 0:
        planner = CausalPlanner(k, cfg["prefetch_budget"], cfg["f1"], cfg["f2"], set(cache.recency))
        for i in range(k):
            items = planner.row(elb, i)
            for (row, key, phase) in items:
                out["plan_items"].append((row, key, phase))
                ins(key, True, 0, i + 1 if ids_visible_causal else None, "plan%d" % phase, row)
    nslots = len(targets)
    for l in range(L):
        demanded[0] = set()
        req_l = sorted({(l, e) for s in range(nslots) for e in targets[s][l]})
        out["coverage_hits"].append(sum(1 for key in req_l if cache.contains(key)))
        out["coverage_size"].append(len(req_l))
        row_of = lambda s: s if s < k else -1
        # sp-sooner is "one layer ahead"; per layer that is sp-later unless L == 1 (one slot ahead)
        sooner = policy == "sp-sooner" and L == 1
        later = policy == "sp-later" or (policy == "sp-sooner" and L > 1)
        if sooner and nslots and row_of(0) >= 0:
            for e, _ in elb.rows[0][l]:
                if ins((l, e), False, 0, None, "jit", 0):
                    out["jit"] += 1
        for s in range(nslots):
            row = row_of(s)
            if later and row >= 0:
                for e, _ in elb.rows[row][l]:
                    if ins((l, e), False, row, None, "jit", row):
                        out["jit"] += 1
            if sooner and s + 1 < nslots and row_of(s + 1) >= 0:
                for e, _ in elb.rows[s + 1][l]:
                    if ins((l, e), False, s + 1, None, "jit", s + 1):
                        out["jit"] += 1
            if policy == "speculative" and row >= 0:
                for e, _ in elb.rows[row][l]:
                    key = (l, e)
                    if not cache.contains(key) and ins(key, True, row, None, "refill", row):
                        out["jit"] += 1
            now_row = s  # rows already verified before this slot (head: 0; unpredicted tail: k)
            req = sorted({(l, e) for e in targets[s][l]})
            out["step_hits"].append(sum(1 for key in req if cache.contains(key)))
            out["step_size"].append(len(req))
            for key in req:
                was = cache.contains(key)
                policy_step(policy, cache, key, elb, now_row, log, (s, row))
                if not was:
                    out["fetched"] += 1
                    out["demand"] += 1
                    if key in demanded[0]:
                        out["refetch"] += 1
                demanded[0].add(key)
    return out


# ----------------------------------------------------------------------------- live governor
ELB_BETA = 1.0 / 32.0  # per drafted row decay of the elb estimator's routing frequencies


def elb_raw(freq, resident, L, E, k):
    """The live engine's "elb" |E_new(k)| estimate before calibration (live.cpp
    `elb_raw`): per layer, each non-resident expert e is fetched if any of the k+1 window tokens
    routes to it, probability 1-(1-p[l,e])^(k+1); summed in (layer, expert) order."""
    s = 0.0
    for i in range(L * E):
        if (i // E, i % E) not in resident:
            s += 1.0 - math.pow(1.0 - freq[i], float(k + 1))
    return s


def elb_estimate(freq, resident, calib, L, E, k):
    """Calibrated estimate: llround(calib[k] * raw), calib[k] = EMA (weight 1/4) of fetched / raw
    over the cycles run at k."""
    return llround(calib[k] * elb_raw(freq, resident, L, E, k))


def elb_update(freq, elb_rows, L, E):
    """Per drafted row r, per layer: p <- (1-beta) p + beta [e in the row's top-K]."""
    for row in elb_rows:
        for l in range(L):
            for e in range(E):
                freq[l * E + e] *= 1.0 - ELB_BETA
            for e in row[l]:
                freq[l * E + e] += ELB_BETA


def live_governor_ks(report, cfg_json, L, E, K, estimator="linear", kmax=16):
    """The k sequence the live engine's governor must pick (live.cpp generate; sim.cpp:118-120,
    394-404) given the run's own outcomes: select_k over the report's (re-fitted) profile, the EMA
    acceptance fed with each cycle's accepted prefix, and either the reference's linear g*k
    estimator (g = fetched/k of the last cycle, starting at L*K) or the elb estimator over this
    oracle's own cache replay (live_cycle) and the cycle's ELB rows.  Returns per cycle the
    expected k, its estimate, the unclamped select_k and the governor inputs (p, g, est table)."""
    c = sim_config(cfg_json)
    prof = profile_from_json(report["profile"])
    kcap = max(c["k_max"] if c["use_governor"] else c["fixed_k"], 1)
    accept = [c["initial_accept"]] * kcap
    g = float(L) * float(K)
    freq = [float(K) / E] * (L * E)
    calib = [1.0] * (kmax + 1)
    cache = Cache(c["capacity_mode"], c["cache_capacity"])
    resident = set()
    rem = report["total_tokens"]
    out = []
    for cyc in report["cycles"]:
        if estimator == "elb":
            est = lambda kk: elb_estimate(freq, resident, calib, L, E, kk)  # noqa: E731
        else:
            est = lambda kk, gg=g: llround(gg * float(kk))  # noqa: E731
        kk = select_k(prof, accept, c["k_min"], c["k_max"], c["k_slo"], est) if c["use_governor"] else c["fixed_k"]
        k = max(1, min(kk, rem, kmax))
        out.append(dict(k=k, est=est(k), select_k=kk, p=list(accept), g=g,
                        table=[est(j) for j in range(c["k_max"] + 1)]))
        raw = elb_raw(freq, resident, L, E, k) if estimator == "elb" else 0.0
        refetch_on = cfg_json.get("refetch_from_hbm", True)
        kc = cyc["k"]
        acc = cyc["accepted"]
        outcomes = []
        for i in range(kc):
            outcomes.append(i < acc)
            if i >= acc:
                break
        accept = update_acceptance(accept, c["ema_alpha"], outcomes[:len(accept)])
        g = float(cyc["new_experts"]) / float(kc)
        if estimator == "elb":
            lc = live_cycle(cache, ELB.build(cyc["elb"], cyc["elb_gates"]), cyc["target"], c)
            # calibrated on the fetches that crossed the link (in-layer refetches come from HBM)
            moved = float(cyc["new_experts"]) - (float(lc["refetch"]) if refetch_on else 0.0)
            if raw > 0.0:
                calib[k] = (1.0 - 0.25) * calib[k] + 0.25 * (moved / raw)
            elb_update(freq, cyc["elb"], L, E)
            resident = set(cache.recency)
        rem -= acc + cyc["bonus"]
    return out
