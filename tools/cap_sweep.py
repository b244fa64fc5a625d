"""Phi-shaped live decode across per-layer cache caps (SURVEY.md §6.4 / BASELINE.md §5): decode
tokens/s, exposed-H2D fraction, fetched experts per token, mean k, PCIe-roofline fraction.
usage: python tools/cap_sweep.py [--caps 4,8,12,14,16] [--tokens 32] [--steps 2] [--k governor[,1,2,4..]]
       [--estimator linear|elb]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_14102_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="phi")
ap.add_argument("--caps", default="4,8,12,14,16")
ap.add_argument("--tokens", type=int, default=32)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--k", default="governor")
ap.add_argument("--policy", default="speculative")
ap.add_argument("--estimator", default="")
ap.add_argument("--out", default="gpurun_out/cap_sweep.jsonl")
a = ap.parse_args()
cfg = m.ModelConfig.named(a.model)
t0 = time.time()
eng = m.Engine(cfg, kmax=16, trace_level=0)
print("engine", time.time() - t0, eng.info(), flush=True)
rows = []
import random
rng = random.Random(5)
for cap, kk in [(int(c), kk) for c in a.caps.split(",") for kk in a.k.split(",")]:
    conf = {"policy": a.policy, "cache_capacity": cap}
    conf.update({"k": "governor", "governor": {"k_min": 1, "k_max": 16, "k_slo": 16}} if kk == "governor" else {"k": int(kk)})
    if a.estimator:
        conf["estimator"] = a.estimator
    eng.configure(conf)
    for _ in range(a.warmup):
        eng.generate([rng.randrange(cfg.V) for _ in range(8)], a.tokens)
    reps = [eng.generate([rng.randrange(cfg.V) for _ in range(8)], a.tokens) for _ in range(a.steps)]
    tok = sum(r["total_tokens"] for r in reps)
    dev = sum(r["total_time_s"] for r in reps)
    stall = sum(r["stall_time_s"] for r in reps)
    h2d = sum(r["h2d_bytes"] for r in reps)
    cyc = [c for r in reps for c in r["cycles"]]
    info = eng.info()
    row = dict(cap=cap, k=kk, estimator=a.estimator or "linear", cap_frac=cap / cfg.E, tokens_per_s=tok / dev, exposed_h2d_frac=stall / dev,
               exposed_h2d_ms_per_token=stall / tok * 1e3, fetched_per_token=sum(r["total_new_experts"] for r in reps) / tok,
               mean_k=sum(c["k"] for c in cyc) / len(cyc), accept=sum(c["accepted"] for c in cyc) / sum(c["k"] for c in cyc),
               pcie_roofline_frac=(h2d / info["pcie_bw_measured"]) / dev, mean_coverage=sum(r["mean_coverage"] for r in reps) / len(reps),
               draft_step_ms=sum(r["kernels"]["draft_time_s"] for r in reps) / max(1, sum(r["kernels"]["draft_steps"] for r in reps)) * 1e3,
               k3_GBps=sum(r["kernels"]["k3_weight_bytes"] for r in reps) / max(1e-9, sum(r["kernels"]["k3_time_s"] for r in reps)) / 1e9)
    rows.append(row)
    print(json.dumps(row), flush=True)
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    for r in rows:
        f.write(json.dumps(r) + "\n")
eng.close()
