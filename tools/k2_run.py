"""Phi-shaped draft FFN (K2, INT4 tcgen05) for one token, engine split choice (W13 S=1, W2 S=4):
time gather+W13+finalize+W2 with CUDA events; under ncu this gives the per-kernel list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_14102_b200 import ops
d, f, E, K = 4096, 6400, 16, 2
s4 = ops.int4_blob_bytes(d, f)
blobs = torch.randint(0, 255, (E * s4,), dtype=torch.uint8, device="cuda")
ids = torch.tensor([[3, 7]], dtype=torch.int32, device="cuda")
s = ops.build_schedule(ids, E)
xn = torch.randint(-3000, 3000, (1, d), dtype=torch.int16, device="cuda")
sp1, sp2 = int(os.environ.get("SP1", 1)), int(os.environ.get("SP2", 2))
for _ in range(3):
    ops.moe_int4_tc(s, xn, blobs, s4, 0, E, d, f, split1=sp1, split2=sp2)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(20):
    ops.moe_int4_tc(s, xn, blobs, s4, 0, E, d, f, split1=sp1, split2=sp2)
ev1.record(); torch.cuda.synchronize()
us = ev0.elapsed_time(ev1) * 50
print(f"split {sp1}/{sp2}: {us:.1f} us per draft FFN layer (2 experts, {2 * s4 / 1e6:.1f} MB INT4) -> {2 * s4 / us / 1e3:.0f} GB/s")
