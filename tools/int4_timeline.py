"""Per-role timeline of the first CTA of one Phi-shaped K2 (INT4 tcgen05) W13 launch (engine split
choice: W13 S=SP1 (default 1), W2 S=SP2 (default 4)), plus the per-call time of the draft FFN."""
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
sp1, sp2 = int(os.environ.get("SP1", 1)), int(os.environ.get("SP2", 4))
abl = int(os.environ.get("ABLATE", 0))  # diagnostics: 1 no MMA, 2 no TMEM store, 4 no dequant math
_lib.check(_lib.lib().mspq_debug_timeline((ctypes.c_longlong * 1)(), -100 - abl))
for _ in range(3):
    ops.moe_int4_tc(s, xn, blobs, s4, 0, E, d, f, split1=sp1, split2=sp2)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for _ in range(10):
    ops.moe_int4_tc(s, xn, blobs, s4, 0, E, d, f, split1=sp1, split2=sp2)
ev1.record(); torch.cuda.synchronize()
print(f"split {sp1}/{sp2}: gather+W13+finalize+W2 {ev0.elapsed_time(ev1) * 100:.1f} us per call")
tl = (ctypes.c_longlong * 2048)()
_lib.check(_lib.lib().mspq_debug_timeline(tl, -1))
from paper_2511_14102_b200._lib import check, lib as L
# arm, then run only up to the W13 launch: the recorder stays armed for W13 and W2 (the W2 launch
# overwrites CTA stamps), so time W13 on its own through a split2 the stamps can tell apart
ops.moe_int4_tc(s, xn, blobs, s4, 0, E, d, f, split1=sp1, split2=sp2)
torch.cuda.synchronize()
_lib.check(_lib.lib().mspq_debug_timeline(tl, 2048))
t = np.array(tl[:2048], dtype=np.int64)
t0 = t[0]
def show(name, lo, n):
    v = t[lo:lo + n]
    v = v[v > 0]
    print(name, ((v - t0) / 1965).round(2).tolist()[:40])
show("producer weight issue (us)", 1, 40)
show("dequant got data group", 256, 40)
show("dequant done group", 512, 40)
show("mma got group", 768, 40)
show("epilogue got group", 1280, 40)
st, en = t[1536:2048:2], t[1537:2048:2]
ok = (st > 0) & (en > 0)
st, en = st[ok], en[ok]
if len(st):
    b0 = st.min()
    print("W13 launch CTAs:", len(st), "start spread us", round((st.max() - b0) / 1e3, 2),
          "end min/median/max us", [round(x / 1e3, 2) for x in (np.min(en - b0), np.median(en - b0), np.max(en - b0))])
    order = np.argsort(en - b0)
    print("slowest CTAs (id, start, end us):", [(int(i), round((st[i] - b0) / 1e3, 2), round((en[i] - b0) / 1e3, 2)) for i in order[-6:]])
