"""Batched multi-stream decode vs one stream at a time (mspq_generate_batch).

For each (streams B, draft length k): B random 128-token prompts decoded together for --tokens
new tokens each through Engine.generate_batch (lru controller, one shared verify pass per cycle),
against the same B prompts decoded one after another through Engine.generate (same policy and k).
Prints one JSON line per point: aggregate decode tok/s on the device clock (prefill excluded on
both sides), experts fetched per token, exposed H2D fraction.

    python tools/batch_bench.py --model phi --cap 4 --streams 1,2,4,8 --k 1,2,3
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="phi")
    ap.add_argument("--cap", type=int, default=4)
    ap.add_argument("--streams", default="1,2,4,8")
    ap.add_argument("--k", default="1,2,3")
    ap.add_argument("--tokens", type=int, default=64)
    ap.add_argument("--solo", action="store_true", help="also time the streams one after another")
    a = ap.parse_args()
    import numpy as np
    import torch

    import paper_2511_14102_b200 as m
    torch.cuda.set_device(0)
    cfg = m.ModelConfig.named(a.model)
    Bs = [int(x) for x in a.streams.split(",")]
    eng = m.Engine(cfg, kmax=16, trace_level=0, max_streams=max(Bs))
    rng = np.random.default_rng(11)
    prompts = [rng.integers(0, cfg.V, 128).tolist() for _ in range(max(Bs))]
    for k in [int(x) for x in a.k.split(",")]:
        for B in Bs:
            if B * (k + 1) > 32:
                continue
            conf = {"policy": "lru", "cache_capacity": a.cap, "k": k}
            eng.configure(conf)
            eng.generate_batch(prompts[:B], 8)  # warm
            eng.configure(conf)
            r = eng.generate_batch(prompts[:B], a.tokens)
            line = {"model": a.model, "cap": a.cap, "k": k, "streams": B,
                    "batch_tok_s": r["total_tokens"] / r["total_time_s"],
                    "batch_fetch_per_tok": r["total_new_experts"] / r["total_tokens"],
                    "batch_exposed_h2d_frac": r["stall_time_s"] / r["total_time_s"],
                    "cycles": len(r["cycles"]),
                    "accept_per_cycle": sum(sum(c["accepted"]) for c in r["cycles"]) / max(1, len(r["cycles"]))}
            if a.solo:
                eng.configure(conf)
                tok = t = f = 0
                for p in prompts[:B]:
                    s = eng.generate(p, a.tokens)
                    tok += s["total_tokens"]
                    t += s["total_time_s"]
                    f += s["total_new_experts"]
                line.update(solo_tok_s=tok / t, solo_fetch_per_tok=f / tok, speedup=line["batch_tok_s"] / (tok / t))
            print(json.dumps(line), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
