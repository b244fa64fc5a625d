"""Control-plane replay throughput: the reference's run_simulation on the host CPU (oracle/_ref,
1 thread) vs the device controller (mspq_replay) on the same synthetic trace and config, per
BASELINE model shape.  Reports µs per committed token and checks the reports are identical.
usage: python tools/replay_bench.py [--tokens 2000]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_14102_b200 as m  # noqa: E402
from oracle import ref  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tokens", type=int, default=2000)
ap.add_argument("--out", default="gpurun_out/replay_bench.jsonl")
a = ap.parse_args()
rows = []
for name, (L, E, K), cap in [("tiny", (4, 8, 2), 4), ("mixtral", (32, 8, 2), 2), ("phi", (32, 16, 2), 4),
                              ("qwen3", (48, 128, 8), 32)]:
    sh = m.MODEL_SHAPES[name]
    tr = ref.generate_trace(L, E, K, a.tokens, seed=1, expert_bytes=3 * sh["d"] * sh["f"] * 2)
    for policy in ["lru", "speculative"]:
        cfg = {"policy": policy, "cache_capacity": cap, "k": "governor",
               "governor": {"k_min": 1, "k_max": 16, "k_slo": 16}}
        t0 = time.perf_counter()
        want = ref.run_simulation(tr, cfg)
        t_ref = time.perf_counter() - t0
        m.run_simulation(tr, cfg)  # warm
        t0 = time.perf_counter()
        got = m.run_simulation(tr, cfg)
        t_dev = time.perf_counter() - t0
        n = want["total_tokens"]
        row = dict(model=name, policy=policy, cap=cap, tokens=n, cycles=len(want["cycles"]),
                   ref_cpu_us_per_token=t_ref / n * 1e6, device_us_per_token=t_dev / n * 1e6,
                   speedup=t_ref / t_dev, identical=json.dumps(got, sort_keys=True) == json.dumps(want, sort_keys=True))
        rows.append(row)
        print(json.dumps(row), flush=True)
# compare_policies (sim.cpp:539-574): the reference loops run_simulation over (policy, capacity)
# serially; the device replays the configs concurrently (replay_many).  Rows must match exactly.
POLS = ["lru", "lookahead", "sp-sooner", "sp-later", "speculative"]
for name, (L, E, K), caps in [("phi", (32, 16, 2), [4, 8, 12]), ("qwen3", (48, 128, 8), [16, 32, 64])]:
    sh = m.MODEL_SHAPES[name]
    tr = ref.generate_trace(L, E, K, a.tokens, seed=1, expert_bytes=3 * sh["d"] * sh["f"] * 2)
    cfg = {"k": "governor", "governor": {"k_min": 1, "k_max": 16, "k_slo": 16}}
    t0 = time.perf_counter()
    want = ref.compare_policies(tr, cfg, POLS, caps)  # the reference's own compare_policies (oracle/_ref)
    t_ref = time.perf_counter() - t0
    m.compare_policies(tr, cfg, POLS, caps)  # warm
    t0 = time.perf_counter()
    got = m.compare_policies(tr, cfg, POLS, caps)
    t_dev = time.perf_counter() - t0
    row = dict(model=name, api="compare_policies", configs=len(POLS) * len(caps), tokens=a.tokens,
               ref_cpu_s=t_ref, device_s=t_dev, speedup=t_ref / t_dev,
               identical=json.dumps(got, sort_keys=True) == json.dumps(want, sort_keys=True))
    rows.append(row)
    print(json.dumps(row), flush=True)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    for r in rows:
        f.write(json.dumps(r) + "\n")
