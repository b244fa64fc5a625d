"""Export a live decode of the bench configuration (BASELINE config 3: Phi shape, per-layer cap
4/16, speculative policy, governor) as a reference JSONL trace (to_reference_trace), with the
B200-fitted HardwareProfile of the run in the header's meta.  bench.py --impl reference replays it
through the reference's run_simulation, so the reference arm runs on the routing this engine
produced (same_config).  Needs a GPU.
usage: python tools/export_live_trace.py [--tokens 256] [--out tests/golden/live_trace_phi_cap4.jsonl]"""
import argparse
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_14102_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="phi")
ap.add_argument("--cap", type=int, default=4)
ap.add_argument("--tokens", type=int, default=256)
ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "live_trace_phi_cap4.jsonl"))
a = ap.parse_args()
cfg = m.ModelConfig.named(a.model)
eng = m.Engine(cfg, kmax=16, trace_level=1)
conf = {"policy": "speculative", "cache_capacity": a.cap, "k": "governor",
        "governor": {"k_min": 1, "k_max": 16, "k_slo": 16}}
eng.configure(conf)
rng = random.Random(1000)  # bench.py prompts(): 128 random ids, seed 1000 (rank 0)
prompt = [rng.randrange(cfg.V) for _ in range(128)]
rep = eng.generate(prompt, a.tokens)
eng.close()
meta = {"policy": conf["policy"], "cache_capacity": str(a.cap), "profile": json.dumps(rep["profile"]),
        "live_tokens_per_s": "%.6f" % (rep["total_tokens"] / rep["total_time_s"]),
        "model": a.model, "prompt_seed": "1000"}
text = m.to_reference_trace(rep, cfg, meta)
with open(a.out, "w") as f:
    f.write(text)
print(a.out, len(text.splitlines()) - 1, "positions,", rep["total_tokens"] / rep["total_time_s"], "tok/s live")
