"""Prefill cost of a 128-token prompt at the bench config: windows, fetches, time per window.
usage: python tools/prefill_probe.py [--cap 4] [--prompt-len 128]"""
import argparse
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_14102_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cap", type=int, default=4)
ap.add_argument("--prompt-len", type=int, default=128)
a = ap.parse_args()
cfg = m.ModelConfig.named("phi")
eng = m.Engine(cfg, kmax=16, trace_level=0)
eng.configure({"policy": "speculative", "cache_capacity": a.cap, "k": "governor",
               "governor": {"k_min": 1, "k_max": 16, "k_slo": 16}})
rng = random.Random(3)
for rep_i in range(2):
    prompt = [rng.randrange(cfg.V) for _ in range(a.prompt_len)]
    t0 = time.perf_counter()
    r = eng.generate(prompt, 8)
    wall = time.perf_counter() - t0
    pf = r["prefill"]
    print(json.dumps({"wall_s": wall, "prefill_s": pf["time_s"], "prefill_expert_copies": pf["expert_copies"],
                      "prefill_h2d_GB": pf["h2d_bytes"] / 1e9, "windows": pf["windows"],
                      "decode_s": r["total_time_s"], "decode_tokens": r["total_tokens"]}))
eng.close()
