"""The C-ABI library loads and exports every symbol include/mspq_capi.h declares; host-side
(GPU-free) entry points behave: the governor restatement equals the reference's."""
import os
import random
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mspq_capi.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mspq_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    from __graft_entry__ import build
    build()
    from paper_2511_14102_b200 import _lib
    return _lib


def test_every_declared_symbol_is_exported(built):
    so = built.LIB_PATH
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mspq_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    assert set(built.EXPORTS) <= exported
    built.lib()  # loads, resolves every signature


def test_status_strings_follow_reference_error_codes(built):
    L = built.lib()
    names = ["OK", "MalformedRecord", "ShapeViolation", "EmptyTrace", "InvalidFidelity", "DegenerateShape",
             "LayerOutOfRange", "ShapeMismatch", "RangeOutOfBounds", "EmptyCache", "UnknownPolicy",
             "EmptyRequired", "IncompleteRouting", "KOutOfRange", "InsufficientSamples", "EmptyRange",
             "InfeasibleBudget", "InvalidConfig", "IoError"]  # errors.hpp:8-27 order
    for i, n in enumerate(names):
        assert L.mspq_status_string(i).decode() == n


def test_governor_matches_reference(built, ref):
    import paper_2511_14102_b200 as m
    rng = random.Random(3)
    for trial in range(150):
        samples, w = [], 1.0
        for _ in range(rng.randint(2, 5)):
            samples.append([w, rng.uniform(1e-3, 0.1)])
            w += rng.randint(1, 6)
        samples.sort()
        prof = {"pcie_bandwidth_bytes_per_s": rng.uniform(1e9, 6e10), "pcie_init_latency_s": rng.uniform(0, 0.03),
                "pcie_overhead_s": rng.uniform(0, 0.003), "expert_size_bytes": rng.randint(10**6, 4 * 10**8),
                "draft_base_s": rng.uniform(0, 0.01), "draft_per_token_s": rng.uniform(1e-4, 0.01),
                "verify_samples": samples}
        kmax = rng.randint(1, 16)
        req = {"profile": prof, "p": [rng.random() for _ in range(16)], "alpha": rng.random(),
               "k_min": 1, "k_max": kmax, "k_slo": rng.randint(1, 16), "g": rng.uniform(0, 40),
               "ttft_budget": rng.choice([0.0, rng.uniform(0.01, 1.0)]),
               "outcomes": [rng.random() < 0.7 for _ in range(rng.randint(0, 8))]}
        if req["k_slo"] < 1:
            continue
        try:
            want = ref.governor(req)
        except ref.RefError:
            with pytest.raises(m.MspqError):
                m.governor(req)
            continue
        got = m.governor(req)
        for k in ("select_k", "t_cycle", "k_accept", "t_verify", "updated_p"):
            assert got[k] == want[k], (trial, k)
        if "k_slo_ttft" in want:
            if isinstance(want["k_slo_ttft"], int):
                assert got["k_slo_ttft"] == want["k_slo_ttft"]
            else:
                assert str(got["k_slo_ttft"]).startswith("error")
