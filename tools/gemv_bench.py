"""In-stream rate of the draft GEMV (mspq_moe_int4_gemv) at a model's shape: W13 + W2 of two experts
per call, rotating over E experts so the weights stream from HBM (not L2); CUDA events around 200
back-to-back calls.  usage: python tools/gemv_bench.py [--model phi] [--split2 2]"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2511_14102_b200 as m  # noqa: E402
from paper_2511_14102_b200._lib import check, lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="phi")
ap.add_argument("--split2", type=int, default=2)
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--tc", action="store_true", help="time the tcgen05 K2 (k_umma_int4p, tile-major blobs) instead")
ap.add_argument("--variant", type=int, default=0, help="GEMV tile/batch variant (mspq_debug_gemv_variant)")
a = ap.parse_args()
cfg = m.ModelConfig.named(a.model)
d, f, E, K = cfg.d, cfg.f, cfg.E, cfg.K
s4 = lib().mspq_int4_blob_bytes(d, f)
blobs = torch.randint(0, 255, (E * s4,), dtype=torch.uint8, device="cuda")
# scales: set every bf16 scale word to 1.0 so outputs stay finite
q13, s13, q2 = 2 * f * d // 2, 2 * f * (d // 128) * 2, d * f // 2
for e in range(E):
    o = e * s4
    blobs[o + q13:o + q13 + s13].view(torch.int16).fill_(0x3F80)
    blobs[o + q13 + s13 + q2:o + s4].view(torch.int16).fill_(0x3F80)
x = (torch.randn(d, device="cuda") * 0.5).to(torch.bfloat16)
act = torch.zeros(K * f, dtype=torch.int16, device="cuda")
y = torch.zeros(8 * K * d, dtype=torch.float32, device="cuda")
ng = torch.tensor([K], dtype=torch.int32, device="cuda")
pairs = [torch.tensor([(2 * i) % E, (2 * i + 1) % E], dtype=torch.int32, device="cuda") for i in range(E // 2)]
P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731


ws = torch.zeros(lib().mspq_moe_bf16_tc_ws_bytes(d, f, 1, K, K, 8), dtype=torch.uint8, device="cuda")
goff = torch.tensor(list(range(K + 1)), dtype=torch.int32, device="cuda")
etok = torch.zeros(K, dtype=torch.int32, device="cuda")
egrp = torch.tensor(list(range(K)), dtype=torch.int32, device="cuda")


def run(i):
    pr = pairs[i % len(pairs)]
    if a.tc:
        check(lib().mspq_moe_int4_tc(P(ng), P(pr), P(pr), P(goff), P(etok), P(egrp), P(x), P(blobs), s4, 0, E, d, f,
                                     1, K, K, 1, a.split2, P(ws), P(y), None))
    else:
        check(lib().mspq_moe_int4_gemv(P(ng), P(pr), P(x), P(blobs), s4, 0, E, d, f, K, a.split2, P(act), P(y), None))


check(lib().mspq_debug_gemv_variant(a.variant))
for i in range(20):
    run(i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(a.iters):
    run(i)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(f"{'tcgen05 K2' if a.tc else 'GEMV v%d' % a.variant} {a.model}: {ms * 1e3:.1f} us per layer (W13 + W2 of {K} experts, {K * s4 / 1e6:.1f} MB) = "
      f"{K * s4 / (ms * 1e-3) / 1e12:.2f} TB/s")
