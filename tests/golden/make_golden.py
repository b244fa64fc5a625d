"""Generates tests/golden/replay_cases.json by running the UNMODIFIED reference control plane
(oracle/_ref/libmoespeq_ref.so, built from /root/reference by oracle/Makefile).  Run here (the
reference tree is not on the GPU box); the fixture is committed."""
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

POL = ["lru", "lookahead", "sp-sooner", "sp-later", "speculative"]


def cases(seed=7, n=40):
    rng = random.Random(seed)
    out = []
    while len(out) < n:
        L = rng.randint(1, 4)
        N = rng.randint(3, 16)
        K = rng.randint(1, min(3, N - 1))
        soft = 0.468 if K >= 2 else 0.0
        toks = rng.randint(5, 70)
        tr = ref.generate_trace(L, N, K, toks, 0.441, soft, 1 - 0.441 - soft, rng.choice([0.5, 0.8, 1.0]),
                                rng.choice([0.0, 1.0, 2.0]), rng.randint(0, 1 << 30),
                                expert_bytes=rng.randint(10**5, 10**8))
        cfg = {"policy": POL[len(out) % 5], "capacity_mode": rng.choice(["per_layer", "global"]),
               "cache_capacity": K + rng.randint(0, N), "prefetch_budget": rng.randint(0, 3),
               "collect_plans": True, "rollback_s": rng.choice([0.0, 1e-3])}
        if rng.random() < 0.5:
            cfg["k"] = rng.randint(1, 8)
        else:
            cfg["k"] = "governor"
            cfg["governor"] = {"k_min": 1, "k_max": rng.randint(2, 12), "k_slo": 16,
                               "ttft_budget_s": rng.choice([0.0, 0.3])}
        if cfg["capacity_mode"] == "per_layer" and rng.random() < 0.3:
            cfg["entropy_weighted_capacity"] = True
        if rng.random() < 0.3:
            cfg["phases"] = {"f1": rng.choice([0, 0.25, 0.5]), "f2": rng.choice([0.5, 0.75, 1.0])}
        try:
            rep = ref.run_simulation(tr, cfg)
        except ref.RefError:
            continue
        out.append({"trace": tr, "config": cfg, "report": rep})
    return out


if __name__ == "__main__":
    data = cases()
    # one larger case at a model shape (Phi-like L=32,N=16,top2; expert bytes of Phi bf16)
    tr = ref.generate_trace(32, 16, 2, 300, seed=11, expert_bytes=157286400)
    cfg = {"policy": "speculative", "cache_capacity": 4, "k": "governor",
           "governor": {"k_min": 1, "k_max": 16, "k_slo": 16}, "collect_plans": True}
    data.append({"trace": tr, "config": cfg, "report": ref.run_simulation(tr, cfg)})
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "replay_cases.json")
    with open(path, "w") as f:
        json.dump(data, f)
    print(path, len(data), os.path.getsize(path))
