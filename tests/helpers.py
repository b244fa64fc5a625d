"""Shared test helpers."""


def diff(a, b, path="", tol=0.0):
    """First difference between two JSON-like trees (None if equal).  tol=0 => bit-exact."""
    if isinstance(b, dict):
        if not isinstance(a, dict):
            return f"{path}: type"
        for k in b:
            if k not in a:
                return f"{path}.{k} missing"
            r = diff(a[k], b[k], path + "." + k, tol)
            if r:
                return r
        return None
    if isinstance(b, (list, tuple)):
        if len(a) != len(b):
            return f"{path}: len {len(a)} vs {len(b)}"
        for i, (x, y) in enumerate(zip(a, b)):
            r = diff(x, y, f"{path}[{i}]", tol)
            if r:
                return r
        return None
    if isinstance(b, float) or isinstance(a, float):
        if tol == 0.0:
            return None if a == b else f"{path}: {a!r} vs {b!r}"
        return None if abs(a - b) <= tol * max(1.0, abs(b)) else f"{path}: {a!r} vs {b!r}"
    return None if a == b else f"{path}: {a!r} vs {b!r}"


KINDS = {0: "demand", 1: "plan2", 2: "plan3", 3: "jit", 4: "refill"}


def oracle_model(cfg, **kw):
    """CPU oracle of a paper_2511_14102_b200.ModelConfig (same weights, attention included)."""
    from oracle import model as om
    return om.Model(om.ModelDesc(**cfg.oracle_kwargs()), **kw)


def _events(log):
    return [(k, l, e, int(h), -1 if v is None else v[0], -1 if v is None else v[1]) for (k, tag, l, e, h, v) in log]


def device_events(log):
    return [(KINDS[ev[0]], ev[2], ev[3], ev[4], ev[5], ev[6]) for ev in log]


def check_control_plane(rep, conf):
    """Replay the run's decode cycles through oracle/control_plane.live_cycle on the run's own
    routing (the prefill streams experts outside the capped cache and leaves it alone); every
    cycle's device hit/miss event log must equal the restatement's.  Returns the oracle cache."""
    from oracle import control_plane as cp
    c = cp.sim_config(conf)
    cache = cp.Cache(c["capacity_mode"], c["cache_capacity"])
    for cyc in rep["cycles"]:
        log = []
        out = cp.live_cycle(cache, cp.ELB.build(cyc["elb"], cyc["elb_gates"]), cyc["target"], c, log)
        assert device_events(cyc["log"]) == _events(log), ("hit/miss log", cyc["cycle"])
        want = out["refetch"] if conf.get("refetch_from_hbm", True) else 0
        assert cyc["refetch_hbm"] == want, ("in-layer refetches", cyc["cycle"])
    return cache
