"""One Phi-shaped replay (run_simulation on the device controller) for the ncu launch list."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2511_14102_b200 as m
from oracle import ref
name = sys.argv[1] if len(sys.argv) > 1 else "phi"
policy = sys.argv[2] if len(sys.argv) > 2 else "speculative"
sh = m.MODEL_SHAPES[name]
cap = {"tiny": 4, "mixtral": 2, "phi": 4, "qwen3": 32}[name]
tr = ref.generate_trace(sh["L"], sh["E"], sh["K"], 400, seed=1, expert_bytes=3 * sh["d"] * sh["f"] * 2)
cfg = {"policy": policy, "cache_capacity": cap, "k": "governor", "governor": {"k_min": 1, "k_max": 16, "k_slo": 16}}
m.run_simulation(tr, cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
t0 = time.perf_counter()
r = m.run_simulation(tr, cfg)
dt = time.perf_counter() - t0
torch.cuda.profiler.stop()
print("cycles", len(r["cycles"]), "tokens", r["total_tokens"], "wall us/token", dt / r["total_tokens"] * 1e6)
