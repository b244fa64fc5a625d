"""Small Phi-shaped decode for ncu: warm up, then profile one generate() call.
usage: ncu --profile-from-start off ... python tools/profile_run.py [--tokens N] [--unique U]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_14102_b200 as m  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="phi")
ap.add_argument("--tokens", type=int, default=4)
ap.add_argument("--unique", type=int, default=16)
ap.add_argument("--cap", type=int, default=4)
ap.add_argument("--k", default="4")
ap.add_argument("--prompt-len", type=int, default=3, help="prompt tokens (attention context)")
a = ap.parse_args()
cfg = m.ModelConfig.named(a.model, unique_experts=a.unique)
eng = m.Engine(cfg, kmax=16, trace_level=0)
conf = {"policy": "speculative", "cache_capacity": a.cap, "k": int(a.k)}
eng.configure(conf)
eng.generate([1, 2, 3], 8)
torch.cuda.synchronize()
torch.cuda.profiler.start()
prompt = [(5 + 7 * i) % cfg.V for i in range(a.prompt_len)]
r = eng.generate(prompt, a.tokens)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("tokens", r["tokens"], "cycles", len(r["cycles"]), "k3", r["kernels"])
eng.close()
