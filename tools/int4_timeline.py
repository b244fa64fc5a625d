"""Run one Phi-shaped K2 (INT4 tcgen05) W13 launch and print the first CTA's per-role timeline."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_14102_b200 import ops, _lib
d, f, E, K = 4096, 6400, 16, 2
s4 = ops.int4_blob_bytes(d, f)
blobs = torch.randint(0, 255, (E * s4,), dtype=torch.uint8, device="cuda")
ids = torch.tensor([[3, 7]], dtype=torch.int32, device="cuda")
s = ops.build_schedule(ids, E)
xn = torch.randint(-3000, 3000, (1, d), dtype=torch.int16, device="cuda")
for split1 in (1, 2):
    for _ in range(3):
        ops.moe_int4_tc(s, xn, blobs, s4, 0, E, d, f, split1=split1, split2=1)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(10):
        ops.moe_int4_tc(s, xn, blobs, s4, 0, E, d, f, split1=split1, split2=1)
    ev1.record(); torch.cuda.synchronize()
    print("split1", split1, "total per call (gather+W13+finalize+W2) us", ev0.elapsed_time(ev1) * 100)
tl = (ctypes.c_longlong * 2048)()
_lib.check(_lib.lib().mspq_debug_timeline(tl, 2048))
t = np.array(tl[:2048], dtype=np.int64)
t0 = t[0]
def show(name, lo, n):
    v = t[lo:lo + n]
    v = v[v > 0]
    print(name, ((v - t0) / 1965).round(2).tolist()[:40])
show("producer stage issue (us)", 1, 40)
show("dequant got data kb", 256, 40)
show("dequant got slot kb", 1024, 40)
show("dequant done kb", 512, 40)
show("mma got kb", 768, 40)
show("epilogue got group", 1280, 40)
