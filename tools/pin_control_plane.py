import sys, random, json, time
sys.path.insert(0, '.')
from oracle import ref, control_plane as cp
def cmp(a, b, path=""):
    if isinstance(a, dict):
        for k in b:
            if k not in a: return f"{path}.{k} missing"
            r = cmp(a[k], b[k], path+"."+k)
            if r: return r
        return None
    if isinstance(a, list) or isinstance(a, tuple):
        if len(a) != len(b): return f"{path} len {len(a)} vs {len(b)}"
        for i,(x,y) in enumerate(zip(a,b)):
            r = cmp(x,y,f"{path}[{i}]")
            if r: return r
        return None
    if isinstance(b, float) or isinstance(a, float):
        if a != b: return f"{path}: {a!r} vs {b!r}"
        return None
    if a != b: return f"{path}: {a!r} vs {b!r}"
def norm_ref(r):
    for c in r["cycles"]:
        c["segments"] = [(s["lane"], s["label"], s["start_s"], s["duration_s"]) for s in c["segments"]]
    return r
rng = random.Random(int(sys.argv[1]) if len(sys.argv)>1 else 0)
bad = 0; t_ref=t_py=0
for trial in range(200):
    L = rng.randint(1,4); N = rng.randint(3,12); K = rng.randint(1, min(3, N-1))
    soft = 0.468 if K>=2 else 0.0
    tr = ref.generate_trace(L,N,K,rng.randint(5,80),0.441,soft,1-0.441-soft,rng.choice([0.5,0.8,1.0]),rng.choice([0,1,2]),rng.randint(0,1<<30), expert_bytes=rng.randint(1,10**8))
    pol = rng.choice(cp.POLICIES)
    mode = rng.choice(["per_layer","global"])
    cfg = {"policy":pol, "capacity_mode":mode, "cache_capacity": K + rng.randint(0, N), "prefetch_budget": rng.randint(0,3),
           "collect_plans": True, "rollback_s": rng.choice([0.0, 1e-3])}
    if rng.random() < 0.5: cfg["k"] = rng.randint(1,8)
    else: cfg["k"] = "governor"; cfg["governor"] = {"k_min":1,"k_max":rng.randint(1,12),"k_slo":16, "ttft_budget_s": rng.choice([0.0, 0.2])}
    if mode=="per_layer" and rng.random()<0.3: cfg["entropy_weighted_capacity"]=True
    if rng.random()<0.3: cfg["phases"]={"f1":rng.choice([0,0.25,0.5]),"f2":rng.choice([0.5,0.75,1.0])}
    try:
        t=time.time(); a = norm_ref(ref.run_simulation(tr, cfg)); t_ref+=time.time()-t
    except ref.RefError as e:
        continue
    t=time.time(); b = cp.simulate(tr, cfg); t_py+=time.time()-t
    r = cmp(b, a)
    if r: bad += 1; print(trial, pol, mode, cfg, r)
    if mode=="per_layer" and not (pol=="sp-sooner" and L==1):
        c = cp.simulate(tr, cfg, order="layer")
        for x,y in zip(c["cycles"], a["cycles"]):
            for key in ["k","accepted","bonus","new_experts","sync_count","coverage","io_wait_s","span_s"]:
                if x[key]!=y[key]: print("LM mismatch", trial, pol, key, x[key], y[key]); bad+=1; break
print("bad", bad, "t_ref", t_ref, "t_py", t_py)
