"""CPU suite: the oracle is pinned before it is trusted.

  * the Python control-plane restatement reproduces the reference's run_simulation
    (oracle/_ref, compiled from /root/reference sources) bit-exactly on random configs and on
    the committed golden fixtures;
  * reference golden vectors / known-answer tests (tests/*.cpp, acceptance_main.cpp);
  * the causal (live) planner emits the reference's item sequence;
  * model-oracle properties (parity unpinned by the reference: no model exists there)."""
import json
import math
import os
import random

import numpy as np
import pytest

from helpers import diff
from oracle import control_plane as cp
from oracle import model as om

HERE = os.path.dirname(os.path.abspath(__file__))


def _norm(rep):
    for c in rep["cycles"]:
        c["segments"] = [(s["lane"], s["label"], s["start_s"], s["duration_s"]) for s in c["segments"]]
    return rep


def test_restatement_matches_golden_fixtures():
    cases = json.load(open(os.path.join(HERE, "golden", "replay_cases.json")))
    for case in cases[:-1]:
        got = cp.simulate(case["trace"], case["config"])
        assert diff(got, _norm(json.loads(json.dumps(case["report"])))) is None


def test_restatement_matches_reference_random(ref):
    rng = random.Random(11)
    for trial in range(120):
        L, N = rng.randint(1, 4), rng.randint(3, 12)
        K = rng.randint(1, min(3, N - 1))
        soft = 0.468 if K >= 2 else 0.0
        tr = ref.generate_trace(L, N, K, rng.randint(5, 60), 0.441, soft, 1 - 0.441 - soft,
                                rng.choice([0.5, 0.8]), rng.choice([0, 1, 2]), rng.randint(0, 1 << 30))
        cfg = {"policy": cp.POLICIES[trial % 5], "capacity_mode": rng.choice(["per_layer", "global"]),
               "cache_capacity": K + rng.randint(0, N), "prefetch_budget": rng.randint(0, 3),
               "collect_plans": True, "k": rng.choice([rng.randint(1, 8), "governor"])}
        want = _norm(ref.run_simulation(tr, cfg))
        assert diff(cp.simulate(tr, cfg), want) is None, (trial, cfg)
        if cfg["capacity_mode"] == "per_layer" and not (cfg["policy"] == "sp-sooner" and L == 1):
            lm = cp.simulate(tr, cfg, order="layer")  # layer-major == token-major
            for x, y in zip(lm["cycles"], want["cycles"]):
                for k in ("k", "accepted", "bonus", "new_experts", "sync_count", "coverage", "span_s"):
                    assert x[k] == y[k]


def test_reference_known_answers():
    # perfmodel (test_perfmodel.cpp:97-171, acceptance_main.cpp:166-176)
    p = cp.default_profile()
    assert cp.t_draft(p, 8) == pytest.approx(0.029, abs=1e-15)
    assert cp.t_pcie_new(p, 10) == pytest.approx(0.017625, abs=1e-15)
    assert cp.t_pcie_new(p, 0) == 0.0
    assert cp.t_cycle(p, 8, 10) == pytest.approx(0.086625, abs=1e-15)
    q = dict(p, verify_samples=[(1.0, 10e-3), (5.0, 20e-3)])
    assert cp.t_verify(q, 3.0) == pytest.approx(15e-3)
    assert cp.t_verify(q, 9.0) == pytest.approx(30e-3)
    assert cp.k_accept([0.9] * 16, 16) == pytest.approx(7.332281830033343, rel=1e-14)
    assert cp.update_acceptance([0.9], 0.1, [True])[0] == pytest.approx(0.91)
    assert cp.update_acceptance([0.5] * 3, 0.1, [True, False, True]) == pytest.approx([0.55, 0.45, 0.5])
    # scheduler (test_scheduler.cpp)
    c = cp.Cache("global", 3)
    hits = sum(cp.policy_step("lru", c, (0, r), None, 0) for r in [0, 1, 2, 0, 1, 2])
    assert hits == 3
    elb = cp.ELB.build([[[0]], [[1]], [[0]], [[2]]])
    c = cp.Cache("per_layer", 2)
    c.insert((0, 1))
    c.insert((0, 0))
    assert cp.select_victim_lookahead(c, elb, 2) == (0, 1)
    assert cp.select_victim_lookahead(c, elb, 1) == (0, 0)
    elb = cp.ELB.build([[[9], [9]]])
    c = cp.Cache("global", 4)
    for k in [(0, 2), (1, 5), (0, 4)]:
        c.insert(k)
    assert cp.select_victim_lookahead(c, elb, 0) == (1, 5)
    # gate-priority phase-2 case (test_scheduler.cpp:220-237)
    elb = cp.ELB.build([[[4, 9]], [[7]], [[8]], [[6]]], [[[0.9, 0.1]], [[1.0]], [[1.0]], [[1.0]]])
    plan = cp.plan_prefetch(elb, lambda k: False, 1, 0.25, 0.75)
    assert plan[0][1:] == ((0, 4), 2)
    # flush at window end (test_scheduler.cpp:261-271)
    elb = cp.ELB.build([[[1]], [[2]]])
    plan = cp.plan_prefetch(elb, lambda k: False, 0, 1.0, 1.0)
    assert [(i, ph) for i, _, ph in plan] == [(1, 3), (1, 3)]
    # Belady offline optimum on {0,1,2,0,1} with capacity 2 -> 4 misses
    rows = [[[r]] for r in [0, 1, 2, 0, 1]]
    elb = cp.ELB.build(rows)
    c = cp.Cache("global", 2)
    misses = 0
    for i, r in enumerate([0, 1, 2, 0, 1]):
        if c.contains((0, r)):
            continue
        misses += 1
        if c.needs_eviction(0):
            c.erase(cp.select_victim_lookahead(c, elb, i))
        c.insert((0, r))
    assert misses == 4


def test_reference_sim_known_answer(ref):
    # test_sim.cpp:94-110: 9 all-accepted tokens at k=4 -> cycles (4,+1), (4,+0)
    tr = ref.generate_trace(1, 4, 1, 9, 1.0, 0.0, 0.0, 1.0, 0.0, 1, expert_bytes=1000)
    r = cp.simulate(tr, {"policy": "lru", "cache_capacity": 4, "k": 4})
    assert [(c["accepted"], c["bonus"]) for c in r["cycles"]] == [(4, 1), (4, 0)]


def test_causal_planner_emits_reference_sequence():
    rng = random.Random(1)
    for _ in range(1500):
        L, E = rng.randint(1, 3), rng.randint(2, 8)
        K, k = rng.randint(1, min(2, E)), rng.randint(1, 9)
        rows = [[sorted(rng.sample(range(E), K)) for _ in range(L)] for _ in range(k)]
        gates = [[[rng.random() for _ in range(K)] for _ in range(L)] for _ in range(k)] if rng.random() < .5 else None
        elb = cp.ELB.build(rows, gates)
        res = {(l, e) for l in range(L) for e in range(E) if rng.random() < 0.3}
        f1 = rng.choice([0, 0.25, 0.5, 1.0])
        f2 = max(f1, rng.choice([0.5, 0.75, 1.0]))
        b = rng.randint(0, 3)
        want = cp.plan_prefetch(elb, lambda key: key in res, b, f1, f2)
        pl = cp.CausalPlanner(k, b, f1, f2, res)
        got = [it for i in range(k) for it in pl.row(elb, i)]
        assert [(x[1], x[2]) for x in got] == [(x[1], x[2]) for x in want]
        assert all(g[0] >= w[0] for g, w in zip(got, want))


def test_model_oracle_properties():
    # det_exp close to exp; counter RNG deterministic and in range; INT4 error bound
    for x in np.linspace(-80, 80, 401, dtype=np.float32):
        v = om.lib().orc_det_exp(float(x))
        assert abs(v - math.exp(float(x))) <= 4e-7 * math.exp(float(x))
    u1 = om.uniform(5, 123, 10000)
    assert np.array_equal(u1, om.uniform(5, 123, 10000))
    assert np.array_equal(u1[100:200], om.uniform(5, 123, 100, start=100))
    assert u1.min() > -1 and u1.max() < 1 and abs(u1.mean()) < 0.03
    w = om.gen(1, 77, 64, 256, 0.1)
    q, s = om.quantize(w)
    err = np.abs(om.dequantize(q, s) - om.bf16_to_f32(w))
    sc = np.repeat(om.bf16_to_f32(s), 128, axis=1)
    # sym zero=8: levels (q-8)*s span [-8s, 7s]; +amax clips to 7s = amax - amax/15 (~0.5 s)
    assert (err <= 0.55 * sc + 1e-8).all()
    assert q.max() <= 15


def test_oracle_speculative_decode_is_lossless():
    """Greedy speculative decoding commits exactly the target's greedy sequence."""
    m = om.Model(om.ModelDesc(**om.CONFIGS["tiny"]))
    prompt = [1, 2, 3, 4, 9]
    om.prefill(m, prompt)  # shared-KV attention: the prompt's rows 0..3
    greedy, tok = [], 9
    for p in range(4, 4 + 24):
        tok, _, _ = m.forward(tok, p, draft=False)
        greedy.append(tok)
    for ks in ([1], [3], [6, 2, 4]):
        cyc = om.speculative_decode(m, 9, 4, ks, 24, prompt=prompt)
        assert [t for c in cyc for t in c["committed"]] == greedy


def test_c_weight_generator_equals_numpy_definition():
    """orc_gen_bf16 (speed) == gen_np (the numpy restatement of the counter-hash generator)."""
    from oracle import model as om
    for seed, tensor, rows, cols, scale in [(1234, om.t_expert(3, 7, 1), 64, 96, 0.0379),
                                            (9, om.T_LM, 5, 4096, 1.0), (77, om.t_router(0), 16, 256, 0.25)]:
        assert np.array_equal(om.gen(seed, tensor, rows, cols, scale), om.gen_np(seed, tensor, rows, cols, scale))


def test_fast_oracle_rows_match_numpy_definition():
    """decode_ref.c (the multi-threaded full-size oracle) generates and INT4-round-trips weight
    rows bit-identically to model.py's gen/quantize/dequantize."""
    import ctypes
    d = om.ModelDesc(L=2, E=4, K=2, d=256, f=384, V=64, seed=77)
    key = om.tensor_key(d.seed, om.t_expert(1, 3, 0))
    ref_w = om.gen(d.seed, om.t_expert(1, 3, 0), d.f, d.d, d.a_up())
    q, s = om.quantize(ref_w)
    deq = om.dequantize(q, s)
    row = np.empty(d.d, dtype=np.float32)
    for r in (0, 5, d.f - 1):
        om.lib().orc_weight_row(key, r * d.d, d.d, ctypes.c_float(d.a_up()), 0, om._p(row))
        assert np.array_equal(row, om.bf16_to_f32(ref_w[r]))
        om.lib().orc_weight_row(key, r * d.d, d.d, ctypes.c_float(d.a_up()), 1, om._p(row))
        assert np.array_equal(row, deq[r])
    # an all-zero group keeps a unit scale and dequantises to zero (model.py sf_safe)
    z = np.zeros((1, 128), dtype=np.uint16)
    qz, sz = om.quantize(z)
    assert np.all(om.dequantize(qz, sz) == 0) and om.bf16_to_f32(sz)[0, 0] == 1.0


def test_fast_oracle_decode_equals_numpy_oracle():
    """Fast (C, double accumulation) and numpy (fp32 BLAS) oracles agree on the expert FFN to
    fp32 rounding and decode the same tokens and routing on the tiny model."""
    d = om.ModelDesc(**om.CONFIGS["tiny"])
    slow, fast = om.Model(d, fast=False), om.Model(d, fast=True)
    rng = np.random.default_rng(3)
    xn = om.f32_to_bf16(rng.standard_normal((3, d.d)).astype(np.float32))
    for draft in (False, True):
        yf = fast.ffn_batch(xn, 2, 5, draft)
        ys = np.stack([slow.ffn(xn[i], 2, 5, draft)[0] for i in range(3)])
        assert np.abs(yf - ys).max() <= 1e-5 * np.abs(ys).max()
    a = om.speculative_decode(slow, 7, 3, [3, 2, 4], 12, prompt=[5, 6, 8, 7])
    b = om.speculative_decode(fast, 7, 3, [3, 2, 4], 12, prompt=[5, 6, 8, 7])
    for x, y in zip(a, b):
        assert x["committed"] == y["committed"] and x["draft"] == y["draft"]
        assert [[r[0].tolist() for r in s] for s in x["target"]] == [[r[0].tolist() for r in s] for s in y["target"]]
