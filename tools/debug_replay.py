"""Find the first divergence between the device replay and the oracle on one golden case."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_14102_b200 as m
from oracle import control_plane as cp
idx = int(sys.argv[1]) if len(sys.argv) > 1 else 31
case = json.load(open("tests/golden/replay_cases.json"))[idx]
cfg = dict(case["config"]); cfg["log"] = True
ref = case["report"]
for rep in range(3):
    got = m.run_simulation(case["trace"], cfg)
    print("rep", rep, "total", got["total_time_s"], "ref", ref["total_time_s"])
log = []
orc = cp.simulate(case["trace"], json.dumps(case["config"]), log=log)
print("oracle total", orc["total_time_s"])
gc = got.get("cycles", [])
rc = ref.get("cycles", [])
for i, (a, b) in enumerate(zip(gc, rc)):
    if a != b:
        print("first differing cycle", i)
        for k in a:
            if a.get(k) != b.get(k): print(" ", k, a.get(k), "|", b.get(k))
        break
gl = got.get("event_log") or got.get("log") or got.get("logs")
print("keys", list(got.keys()))
if gl is not None:
    dev = [tuple(ev[2:]) for cyc in gl for ev in cyc]
    orc_ev = [(e[2], e[3], int(e[4]), e[5][0] if e[5] else -1, e[5][1] if e[5] else -1) for e in log]
    print("n events dev", len(dev), "oracle", len(orc_ev))
    for j, (a, b) in enumerate(zip(dev, orc_ev)):
        if tuple(a) != tuple(b):
            print("first event mismatch at", j, "dev", a, "oracle", b)
            print("context dev", dev[max(0,j-5):j+3]); print("context orc", orc_ev[max(0,j-5):j+3]); print("raw orc", log[max(0,j-5):j+3])
            break
    else:
        print("event logs agree")
