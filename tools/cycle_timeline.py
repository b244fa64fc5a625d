"""Where the PCIe link sits idle in a Phi-shaped capped-cache decode: per cycle, the union of the
copy batches' busy intervals against the cycle span, and per verify layer the chain from the
controller's decision to the GEMM's end.  Usage: python tools/cycle_timeline.py [tokens] [cap]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2511_14102_b200 as m

tokens = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = m.ModelConfig.named("phi")
eng = m.Engine(cfg, kmax=16, trace_level=1, expert_codec=os.environ.get("CODEC", "xc"))
eng.configure({"policy": "speculative", "cache_capacity": cap, "k": "governor",
               "governor": {"k_min": 1, "k_max": 16, "k_slo": 16}})
rng = np.random.default_rng(7)
eng.generate([int(x) for x in rng.integers(0, cfg.V, 8)], 4)  # warm-up
rep = eng.generate([int(x) for x in rng.integers(0, cfg.V, 8)], tokens)
for c in rep["cycles"][:4]:
    t0, span = c["start_s"], c["span_s"]
    io = sorted((s["start_s"], s["start_s"] + s["duration_s"]) for s in c["segments"] if s["lane"] == "io")
    busy, cur = 0.0, None
    for a, b in io:
        if cur and a <= cur[1]:
            cur[1] = max(cur[1], b)
        else:
            if cur: busy += cur[1] - cur[0]
            cur = [a, b]
    if cur: busy += cur[1] - cur[0]
    dr = [s for s in c["segments"] if s["label"] == "draft"][0]
    print(f"cycle {c['cycle']} k={c['k']} span {span * 1e3:.2f} ms, draft {dr['duration_s'] * 1e3:.2f} ms, "
          f"copies busy {busy * 1e3:.2f} ms ({busy / span:.3f}), fetched {c['new_experts']}, batches {len(io)}")
    lt = np.array(c["layer_times"]) - t0
    ends = [b for _, b in io]
    for l, (w0, k0, ge, rt) in enumerate(lt):
        prev = lt[l - 1][2] if l else dr["start_s"] + dr["duration_s"] - t0
        print(f"  L{l:2d} ctl-done {w0 * 1e3:8.3f}  (+{(w0 - prev) * 1e6:6.0f} us after prev GEMM: "
              f"route {(rt - prev) * 1e6:4.0f}, ctl {(w0 - rt) * 1e6:4.0f})  "
              f"gemm start {k0 * 1e3:8.3f}  gemm {(ge - k0) * 1e6:6.0f} us")
    print("  io batches (ms):", [(round((a - t0) * 1e3, 2), round((b - t0) * 1e3, 2)) for a, b in io])
