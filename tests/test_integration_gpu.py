"""INTEGRATION.md §2 is real code: integration/sim_b200.cpp (the reference-side binding a
maintainer adds) compiles against the reference headers (oracle/Makefile ->
oracle/_ref/sim_b200_check) and, on the GPU, its SimReport equals the reference's
run_simulation byte for byte on the golden replay cases."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "sim_b200_check")


def test_reference_side_binding_builds():
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference tree absent (the binary is built where it is)")
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8"])
    assert os.access(BIN, os.X_OK)


@pytest.mark.gpu
def test_reference_side_binding_reproduces_run_simulation(cuda, tmp_path):
    if not os.access(BIN, os.X_OK):
        pytest.skip("oracle/_ref/sim_b200_check not built")
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "replay_cases.json")))
    for i, case in enumerate(cases[:12]):
        tp, cp_ = tmp_path / f"t{i}.jsonl", tmp_path / f"c{i}.json"
        tp.write_text(case["trace"])
        cp_.write_text(json.dumps(case["config"]))
        r = subprocess.run([BIN, str(tp), str(cp_)], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0 and r.stdout.startswith("identical"), (i, r.stdout, r.stderr[-500:])
