"""Expert codec throughput on one B200: GPU decode rate vs grid size, and the chunked
pinned-host -> staging -> decode pipeline vs a plain bf16 H2D copy of the same expert."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_14102_b200 import ops  # noqa: E402
from paper_2511_14102_b200._lib import lib  # noqa: E402

d, f = 4096, 6400
blob = ops.fill_expert(5, 1, 3, d, f, 1.0, 1.0)
tiles = torch.cat([ops.tile_bf16(blob[: 2 * f * d], 2 * f, d).view(-1), ops.tile_bf16(blob[2 * f * d:], d, f).view(-1)])
n = tiles.numel() // 8192
xb = ops.xc_encode(tiles)
S16 = tiles.numel() * 2
res = {"expert_bytes": S16, "blob_bytes": xb.numel(), "ratio": xb.numel() / S16}
dst = torch.empty_like(tiles)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for ctas in [8, 16, 32, 64, 148, 296, 592]:
    for _ in range(2):
        ops.xc_decode(xb, n, dst=dst, n_ctas=ctas)
    ev0.record()
    for _ in range(5):
        ops.xc_decode(xb, n, dst=dst, n_ctas=ctas)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 5
    res[f"decode_ms_{ctas}ctas"] = ms
    res[f"decode_GBps_out_{ctas}ctas"] = S16 / ms / 1e6
assert torch.equal(dst, tiles)
# pinned host copies
h_raw = torch.empty(S16, dtype=torch.uint8, pin_memory=True)
h_raw.copy_(tiles.view(torch.uint8).cpu())
h_xc = torch.empty(xb.numel(), dtype=torch.uint8, pin_memory=True)
h_xc.copy_(xb.cpu())
d_raw = torch.empty(S16, dtype=torch.uint8, device="cuda")
stg = torch.empty_like(xb)
for _ in range(2):
    d_raw.copy_(h_raw, non_blocking=True)
ev0.record()
for _ in range(5):
    d_raw.copy_(h_raw, non_blocking=True)
ev1.record()
torch.cuda.synchronize()
res["h2d_raw_ms"] = ev0.elapsed_time(ev1) / 5
res["h2d_raw_GBps"] = S16 / res["h2d_raw_ms"] / 1e6
ev0.record()
for _ in range(5):
    stg.copy_(h_xc, non_blocking=True)
ev1.record()
torch.cuda.synchronize()
res["h2d_blob_ms"] = ev0.elapsed_time(ev1) / 5
toff = xb[64:64 + 4 * (n + 1)].cpu().view(torch.int32).tolist()
cs = torch.cuda.Stream(priority=-1)
ds = torch.cuda.Stream(priority=-1)
for nc in [1, 2, 4, 8, 16]:
    for ctas in [16, 32, 64, 128]:
        evs = []
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(cs)
        ds.wait_event(start)
        for rep in range(4):
            for c in range(nc):
                t0, t1 = n * c // nc, n * (c + 1) // nc
                b0, b1 = (toff[t0] if c else 0), toff[t1]
                with torch.cuda.stream(cs):
                    stg[b0:b1].copy_(h_xc[b0:b1], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(cs)
                ds.wait_event(e)
                with torch.cuda.stream(ds):
                    ops.xc_decode(stg, n, t0, t1, dst=dst, n_ctas=ctas)
            de = torch.cuda.Event()
            de.record(ds)
            cs.wait_event(de)  # single staging buffer: next expert waits for this decode
        end.record(ds)
        torch.cuda.synchronize()
        ms = start.elapsed_time(end) / 4
        res[f"pipe_ms_nc{nc}_ctas{ctas}"] = ms
print(json.dumps(res, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/xc_bench.json", "w"), indent=1)
