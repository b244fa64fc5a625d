"""Replay parity: the device control plane (K4, k_ctl_replay_cycle) driven by the product's
host loop must reproduce the reference's run_simulation report BIT-EXACTLY -- integers,
per-layer coverage, step coverage, plans, modeled segments and totals."""
import json
import os
import random

import pytest

from helpers import diff

HERE = os.path.dirname(os.path.abspath(__file__))
pytestmark = pytest.mark.gpu


def _load():
    with open(os.path.join(HERE, "golden", "replay_cases.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("idx", range(41))
def test_replay_matches_reference_golden(cuda, idx):
    import paper_2511_14102_b200 as m
    case = _load()[idx]
    got = m.run_simulation(case["trace"], case["config"])
    d = diff(got, case["report"])
    assert d is None, (case["config"], d)


def test_replay_random_against_live_reference(cuda, ref):
    import paper_2511_14102_b200 as m
    rng = random.Random(2024)
    pol = ["lru", "lookahead", "sp-sooner", "sp-later", "speculative"]
    for trial in range(60):
        L, N = rng.randint(1, 6), rng.randint(2, 24)
        K = rng.randint(1, min(4, N - 1)) if N > 1 else 1
        soft = 0.468 if K >= 2 else 0.0
        mis = 1 - 0.441 - soft if K < N else 0.0
        tr = ref.generate_trace(L, N, K, rng.randint(1, 90), 1 - soft - mis, soft, mis,
                                rng.random(), rng.choice([0.0, 0.5, 1.5]), rng.randint(0, 10**9))
        cfg = {"policy": pol[trial % 5], "capacity_mode": rng.choice(["per_layer", "global"]),
               "cache_capacity": K + rng.randint(0, N), "prefetch_budget": rng.randint(0, 4),
               "collect_plans": True, "k": rng.randint(1, 10)}
        if rng.random() < 0.4:
            cfg["k"] = "governor"
        want = ref.run_simulation(tr, cfg)
        got = m.run_simulation(tr, cfg)
        d = diff(got, want)
        assert d is None, (trial, cfg, d)


def test_replay_errors_map_to_reference_codes(cuda, ref):
    import paper_2511_14102_b200 as m
    tr = ref.generate_trace(2, 8, 2, 10, seed=1)
    with pytest.raises(m.MspqError) as e:
        m.run_simulation(tr, {"cache_capacity": 1})  # below top_k -> InvalidConfig
    assert e.value.name == "InvalidConfig"
    with pytest.raises(m.MspqError) as e:
        m.run_simulation(tr, {"policy": "mru"})
    assert e.value.name == "UnknownPolicy"
    with pytest.raises(m.MspqError) as e:
        m.run_simulation("", {})
    assert e.value.name == "EmptyTrace"


def test_replay_event_log_matches_python_oracle(cuda, ref):
    """Hit/miss SEQUENCE parity (not only aggregates): the device's per-event log equals the
    Python restatement's log (oracle/control_plane.py, itself pinned to the reference)."""
    import paper_2511_14102_b200 as m
    from oracle import control_plane as cp
    rng = random.Random(5)
    kinds = {0: "demand", 1: "plan2", 2: "flush", 3: "jit", 4: "refill"}
    for trial in range(25):
        L, N, K = rng.randint(1, 4), rng.randint(4, 12), 2
        tr = ref.generate_trace(L, N, K, rng.randint(10, 60), seed=rng.randint(0, 10**6))
        cfg = {"policy": ["lru", "lookahead", "sp-sooner", "sp-later", "speculative"][trial % 5],
               "capacity_mode": rng.choice(["per_layer", "global"]),
               "cache_capacity": K + rng.randint(0, 4), "k": rng.randint(1, 6)}
        log = []
        cp.simulate(tr, cfg, log=log)
        got = m.run_simulation(tr, dict(cfg, log=True))
        dev = [ev for cyc in got["log"] for ev in cyc]
        want = [(k, l, e, int(h), -1 if v is None else v[0], -1 if v is None else v[1])
                for (k, tag, l, e, h, v) in log]
        gotn = [(kinds[ev[0]], ev[2], ev[3], ev[4], ev[5], ev[6]) for ev in dev]
        assert gotn == want, trial


def test_replay_one_launch_path_against_reference(cuda, ref):
    """Without logs / plans the whole trace replays in ONE launch with the governor on the device
    (mspq_cache_replay_all): every report stays bit-exact with the reference run_simulation,
    governor-chosen k included (the host re-derives each k and fails on a mismatch)."""
    import paper_2511_14102_b200 as m
    rng = random.Random(77)
    pol = ["lru", "lookahead", "sp-sooner", "sp-later", "speculative"]
    for trial in range(60):
        L, N = rng.randint(1, 8), rng.randint(2, 32)
        K = rng.randint(1, min(4, N - 1))
        soft = 0.468 if K >= 2 else 0.0
        tr = ref.generate_trace(L, N, K, rng.randint(1, 300), 0.441, soft, 1 - 0.441 - soft, rng.random(),
                                rng.choice([0.0, 1.0, 2.0]), rng.randint(0, 10**9), expert_bytes=rng.choice([25_000_000, 157_286_400]))
        cfg = {"policy": pol[trial % 5], "capacity_mode": rng.choice(["per_layer", "global"]),
               "cache_capacity": K + rng.randint(0, N), "prefetch_budget": rng.randint(0, 4),
               "k": rng.randint(1, 12)}
        if rng.random() < 0.7:
            cfg["k"] = "governor"
            cfg["governor"] = {"k_min": 1, "k_max": rng.choice([8, 16]), "k_slo": 16}
        want = ref.run_simulation(tr, cfg)
        got = m.run_simulation(tr, cfg)
        assert diff(got, want) is None, (trial, cfg, diff(got, want))
