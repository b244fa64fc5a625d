"""K4 device controller in isolation (live rules), driven through the C-ABI with random ELBs and
target routings: every decision (event log, copy requests, buffer table) must equal the Python
restatement oracle/control_plane.live_cycle, with and without shared-memory staging."""
import ctypes
import random

import numpy as np
import pytest
import torch

from oracle import control_plane as cp

pytestmark = pytest.mark.gpu
KINDS = {0: "demand", 1: "plan2", 2: "plan3", 3: "jit", 4: "refill"}


def run_device(L, E, K, kmax, conf, cycles, staging):
    from paper_2511_14102_b200 import _lib
    lib = _lib.lib()
    c = cp.sim_config(conf)
    nbuf = (L * c["cache_capacity"] if c["capacity_mode"] == "per_layer" else c["cache_capacity"]) + E + 8
    h = ctypes.c_void_p()
    _lib.check(lib.mspq_cache_create(L, E, K, kmax, nbuf, 0, ctypes.byref(h)))
    caps = (ctypes.c_int * L)(*([c["cache_capacity"]] * L))
    s = torch.cuda.current_stream().cuda_stream
    pol = cp.POLICIES.index(c["policy"])
    mode = 0 if c["capacity_mode"] == "per_layer" else 1
    _lib.check(lib.mspq_cache_configure(h, mode, pol, caps, c["cache_capacity"], c["prefetch_budget"],
                                        c["f1"], c["f2"], s))
    _lib.check(lib.mspq_cache_set_staging(h, 1 if staging else 0))
    v = _lib.CacheView()
    _lib.check(lib.mspq_cache_view_get(h, ctypes.byref(v)))
    gbuf = torch.zeros(E, dtype=torch.int32, device="cuda")
    logs = []
    for (elb_ids, elb_gates, tgt) in cycles:
        k = elb_ids.shape[0]
        _lib.check(lib.mspq_cache_begin_cycle(h, k, s))
        ids_d = torch.from_numpy(elb_ids.reshape(-1).astype(np.int32)).cuda()
        g_d = torch.from_numpy(elb_gates.reshape(-1).astype(np.float32)).cuda()
        # the draft router normally writes these rows; here the test writes them
        _memcpy(v.elb_ids, ids_d.data_ptr(), ids_d.numel() * 4)
        _memcpy(v.elb_gates, g_d.data_ptr(), g_d.numel() * 4)
        for i in range(k):
            _lib.check(lib.mspq_cache_plan_row(h, i, s))
        tg = torch.from_numpy(tgt.astype(np.int32)).cuda()  # [L][T][K]
        T = tgt.shape[1]
        for l in range(L):
            _lib.check(lib.mspq_cache_verify_layer(h, l, T, tg[l].contiguous().data_ptr(), gbuf.data_ptr(), s))
        torch.cuda.synchronize()
        n = v.host_stat[7]
        raw = torch.empty(n * 6, dtype=torch.int32, device="cuda")
        _memcpy(raw.data_ptr(), v.log, n * 24)
        raw = raw.cpu().numpy().reshape(n, 6)
        logs.append([(KINDS[int(r[0])], int(r[2]) // E, int(r[2]) % E, int(r[3]),
                      -1 if r[4] < 0 else int(r[4]) // E, -1 if r[4] < 0 else int(r[4]) % E) for r in raw])
    lib.mspq_cache_destroy(h)
    return logs


def _memcpy(dst, src, nbytes):
    """device -> device copy between raw pointers (torch views, no ownership)"""
    torch.cuda.synchronize()
    _view(dst, nbytes).copy_(_view(src, nbytes))
    torch.cuda.synchronize()


def _view(ptr, nbytes):
    # wrap a raw device pointer as a uint8 tensor (no ownership)
    class Holder:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
    return torch.as_tensor(Holder(), device="cuda")


def run_oracle(L, E, K, conf, cycles):
    c = cp.sim_config(conf)
    cache = cp.Cache(c["capacity_mode"], c["cache_capacity"])
    logs = []
    for (elb_ids, elb_gates, tgt) in cycles:
        elb = cp.ELB.build(elb_ids.tolist(), elb_gates.tolist())
        targets = [[tgt[l][s].tolist() for l in range(L)] for s in range(tgt.shape[1])]
        log = []
        cp.live_cycle(cache, elb, targets, c, log)
        logs.append([(k, l, e, int(h), -1 if v is None else v[0], -1 if v is None else v[1])
                     for (k, tag, l, e, h, v) in log])
    return logs


@pytest.mark.parametrize("staging", [True, False])
@pytest.mark.parametrize("policy", cp.POLICIES)
def test_live_controller_matches_oracle(cuda, staging, policy):
    rng = np.random.default_rng(cp.POLICIES.index(policy) * 7 + staging)
    for trial in range(6):
        L, E, K = int(rng.integers(1, 5)), int(rng.integers(3, 20)), 2
        kmax = 8
        mode = ["per_layer", "global"][trial % 2]
        cap = int(rng.integers(K, E + 1)) if mode == "per_layer" else int(rng.integers(K, L * E + 1))
        conf = {"policy": policy, "capacity_mode": mode, "cache_capacity": cap,
                "prefetch_budget": int(rng.integers(0, 3)), "k": 4}
        cycles = []
        for _ in range(5):
            k = int(rng.integers(1, kmax + 1))
            elb_ids = np.stack([[rng.choice(E, K, replace=False) for _ in range(L)] for _ in range(k)])
            elb_g = rng.random((k, L, K)).astype(np.float32)
            tgt = np.stack([[rng.choice(E, K, replace=False) for _ in range(k + 1)] for _ in range(L)])
            cycles.append((elb_ids, elb_g, tgt))
        got = run_device(L, E, K, kmax, conf, cycles, staging)
        want = run_oracle(L, E, K, conf, cycles)
        for ci, (g, w) in enumerate(zip(got, want)):
            assert g == w, (policy, mode, staging, trial, ci)
