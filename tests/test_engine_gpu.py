"""Live engine parity (generate()): the B200 decode loop vs the CPU oracle on the same
random-init weights and prompt.

  * expert-selection traces (draft ELB rows, target routing per window slot and layer): bit-exact
  * draft tokens, target argmax, accepted counts, committed tokens: bit-exact
  * cache hit/miss SEQUENCE: the device controller's event log == oracle/control_plane.live_cycle
    replayed on the engine's own routing (every policy, both capacity modes)
  * ELB gate scores: within 5e-3 absolute (hidden states differ at ~1e-4 relative: fp32 FFN
    accumulation order vs the oracle, and the bf16 rounding of the SiLU*up activation that it
    can flip by one ulp)
Near-ties are not masked: a mismatch fails the test."""
import numpy as np
import pytest

from helpers import check_control_plane
from oracle import control_plane as cp
from oracle import model as om

pytestmark = pytest.mark.gpu
KINDS = {0: "demand", 1: "plan2", 2: "plan3", 3: "jit", 4: "refill"}


def _engine(name="tiny", kmax=8, **kw):
    import paper_2511_14102_b200 as m
    cfg = m.ModelConfig.named(name, **kw)
    return m.Engine(cfg, kmax=kmax, trace_level=2), cfg


def _oracle_desc(cfg):
    return om.ModelDesc(**cfg.oracle_kwargs())


def _check_traces(rep, cyc_oracle):
    assert len(rep["cycles"]) == len(cyc_oracle)
    for c, o in zip(rep["cycles"], cyc_oracle):
        assert c["k"] == o["k"]
        assert c["draft_tokens"] == o["draft"]
        assert c["target_argmax"] == o["target_argmax"]
        assert c["accepted"] + c["bonus"] == len(o["committed"])
        assert c["tokens"] == o["committed"]
        for r in range(o["k"]):
            for l in range(len(o["elb"][r])):
                assert c["elb"][r][l] == o["elb"][r][l][0].tolist(), ("elb", r, l)
                assert np.allclose(c["elb_gates"][r][l], o["elb"][r][l][1], atol=5e-3)
        for s in range(o["k"] + 1):
            for l in range(len(o["target"][s])):
                assert c["target"][s][l] == o["target"][s][l][0].tolist(), ("target", s, l)


def _control_plane_log(rep, cfg_json, L, E):
    c = cp.sim_config(cfg_json)
    cache = cp.Cache(c["capacity_mode"], c["cache_capacity"])
    out = []
    for cyc in rep["cycles"]:
        elb = cp.ELB.build(cyc["elb"], cyc["elb_gates"])
        log = []
        cp.live_cycle(cache, elb, cyc["target"], c, log)
        out.append([(k, l, e, int(h), -1 if v is None else v[0], -1 if v is None else v[1])
                    for (k, tag, l, e, h, v) in log])
    return out


def test_generate_tiny_matches_oracle_end_to_end(cuda):
    eng, cfg = _engine()
    conf = {"policy": "speculative", "cache_capacity": 3, "k": 4}
    eng.configure(conf)
    prompt = [7, 100, 3, 250, 11]
    rep = eng.generate(prompt, 40)
    assert len(rep["tokens"]) == 40
    model = om.Model(_oracle_desc(cfg))
    ks = [c["k"] for c in rep["cycles"]]
    oc = om.speculative_decode(model, prompt[-1], len(prompt) - 1, ks, 40, prompt=prompt)
    _check_traces(rep, oc)
    want = _control_plane_log(rep, conf, cfg.L, cfg.E)
    for c, w in zip(rep["cycles"], want):
        got = [(KINDS[ev[0]], ev[2], ev[3], ev[4], ev[5], ev[6]) for ev in c["log"]]
        assert got == w
    eng.close()


@pytest.mark.parametrize("policy", ["lru", "lookahead", "sp-sooner", "sp-later", "speculative"])
@pytest.mark.parametrize("mode", ["per_layer", "global"])
def test_live_hit_miss_sequence_all_policies(cuda, policy, mode):
    eng, cfg = _engine()
    conf = {"policy": policy, "capacity_mode": mode, "cache_capacity": 3 if mode == "per_layer" else 9,
            "k": 5, "prefetch_budget": 1}
    eng.configure(conf)
    rep = eng.generate([1, 2, 3], 30)
    check_control_plane(rep, conf)  # + each cycle's in-layer refetch count (served from HBM)
    want = _control_plane_log(rep, conf, cfg.L, cfg.E)
    tot_fetched = 0
    for c, w in zip(rep["cycles"], want):
        got = [(KINDS[ev[0]], ev[2], ev[3], ev[4], ev[5], ev[6]) for ev in c["log"]]
        assert got == w, (policy, mode, c["cycle"])
        tot_fetched += c["new_experts"]
    # every fetched expert moved real bytes over PCIe
    assert rep["h2d_bytes_bf16"] == tot_fetched * cfg.expert_bytes_bf16()
    assert 0 < rep["h2d_bytes"] <= rep["h2d_bytes_bf16"] or tot_fetched == 0
    eng.close()


def test_generate_governor_and_rerun_determinism(cuda):
    eng, cfg = _engine()
    conf = {"policy": "speculative", "cache_capacity": 4, "k": "governor",
            "governor": {"k_min": 1, "k_max": 8, "k_slo": 8}}
    eng.configure(conf)
    r1 = eng.generate([42], 32)
    eng.configure(conf)
    r2 = eng.generate([42], 32)
    assert r1["tokens"] == r2["tokens"]  # greedy speculative decode is lossless: same text for any k
    for c in r1["cycles"]:
        assert 1 <= c["k"] <= 8
    # token stream equals plain greedy target decoding (the oracle's, k=1 cycles commit one draft)
    model = om.Model(_oracle_desc(cfg))
    oc = om.speculative_decode(model, 42, 0, [c["k"] for c in r1["cycles"]], 32, prompt=[42])
    assert r1["tokens"] == [t for o in oc for t in o["committed"]]
    eng.close()


def test_engine_weights_match_oracle_generator(cuda):
    eng, cfg = _engine()
    model = om.Model(_oracle_desc(cfg))
    d, f = cfg.d, cfg.f
    from test_kernels_gpu import untile
    raw = np.frombuffer(eng.read("expert:2:5", cfg.expert_bytes_bf16()), dtype=np.uint16)
    g, u, dn = model.expert(2, 5)
    w13 = untile(raw[:2 * f * d], 2 * f, d)  # host store keeps tile-major SW128 images
    assert np.array_equal(w13[0::2], g) and np.array_equal(w13[1::2], u)
    assert np.array_equal(untile(raw[2 * f * d:], d, f), dn)
    r = np.frombuffer(eng.read("router:1", cfg.E * d * 2), dtype=np.uint16).reshape(cfg.E, d)
    assert np.array_equal(r, model.router(1))
    eng.close()


def test_engine_rejects_bad_configs(cuda):
    import paper_2511_14102_b200 as m
    eng, cfg = _engine()
    with pytest.raises(m.MspqError) as e:
        eng.configure({"cache_capacity": 1})
    assert e.value.name == "InvalidConfig"
    with pytest.raises(m.MspqError) as e:
        eng.configure({"bogus": 1})
    assert e.value.name == "InvalidConfig"
    with pytest.raises(m.MspqError) as e:
        eng.configure({"k": 32})
    assert e.value.name == "KOutOfRange"
    eng.close()


def test_live_trace_replays_through_reference_tools(cuda, ref):
    """A live run exported as a reference JSONL trace parses and replays in the reference's own
    run_simulation, and the device replay of it is bit-exact with that."""
    import paper_2511_14102_b200 as m
    eng, cfg = _engine()
    eng.configure({"policy": "speculative", "cache_capacity": 3, "k": 4})
    rep = eng.generate([3, 1, 4, 1, 5], 48)
    eng.close()
    text = m.to_reference_trace(rep, cfg)
    lines = text.strip().splitlines()
    assert len(lines) > 10
    conf = {"policy": "speculative", "cache_capacity": 3, "k": 4, "collect_plans": True}
    want = ref.run_simulation(text, conf)
    got = m.run_simulation(text, conf)
    from helpers import diff
    assert diff(got, want) is None


def test_expert_codec_is_lossless_end_to_end(cuda):
    """The XC host store (compressed experts, GPU decode into the slot) changes only the bytes on
    the link: tokens, routing traces and the hit/miss log equal the raw-store engine's."""
    import paper_2511_14102_b200 as m
    cfg = m.ModelConfig.named("tiny")
    conf = {"policy": "speculative", "cache_capacity": 3, "k": 4}
    prompt = [7, 100, 3, 250, 11]
    reps = {}
    for codec in ["none", "xc"]:
        eng = m.Engine(cfg, kmax=8, trace_level=2, expert_codec=codec)
        eng.configure(conf)
        reps[codec] = eng.generate(prompt, 32)
        if codec == "xc":
            assert eng.read("expert_blob:1:2", 64)[:4] == b"XCB1"
        eng.close()
    a, b = reps["none"], reps["xc"]
    assert a["tokens"] == b["tokens"]
    for ca, cb in zip(a["cycles"], b["cycles"]):
        for key in ["k", "draft_tokens", "target_argmax", "target", "elb", "log", "new_experts"]:
            assert ca[key] == cb[key], key
    # the raw store moves every fetch's bf16 bytes except the in-layer refetches (served from HBM)
    assert b["h2d_bytes_bf16"] - a["refetch_hbm"] * cfg.expert_bytes_bf16() == a["h2d_bytes"]
    assert a["refetch_hbm"] == b["refetch_hbm"]
    assert b["total_new_experts"] > 0 and b["h2d_bytes"] < 0.72 * a["h2d_bytes"]


@pytest.mark.parametrize("name,cap,k", [("phi", 4, 3), ("qwen3", 32, 2), ("mixtral", 2, 2)])
def test_generate_full_width_shapes_match_oracle(cuda, name, cap, k):
    """BASELINE model widths (Phi-3.5-MoE: E=16 top-2 d=4096 ffn=6400 V=32064; Qwen3-30B-A3B:
    E=128 top-8 d=2048 ffn=768 V=151936; Mixtral-8x7B: E=8 top-2 d=4096 ffn=14336 V=32000) on 2
    layers, capped cache, XC host store: every routing
    trace, draft token, target argmax and committed token equals the CPU oracle's, and the
    hit/miss log equals the control-plane restatement's."""
    eng, cfg = _engine(name, L=2)
    conf = {"policy": "speculative", "cache_capacity": cap, "k": k}
    eng.configure(conf)
    prompt = [11, 200, 3001]
    rep = eng.generate(prompt, 10)
    model = om.Model(_oracle_desc(cfg))
    oc = om.speculative_decode(model, prompt[-1], len(prompt) - 1, [c["k"] for c in rep["cycles"]], 10, prompt=prompt)
    _check_traces(rep, oc)
    want = _control_plane_log(rep, conf, cfg.L, cfg.E)
    for c, w in zip(rep["cycles"], want):
        got = [(KINDS[ev[0]], ev[2], ev[3], ev[4], ev[5], ev[6]) for ev in c["log"]]
        assert got == w
    assert rep["total_new_experts"] > 0
    eng.close()


def test_shared_host_store_attach_path(cuda, tmp_path):
    """The multi-rank store (bench.py under torchrun): rank 0 creates and fills a /dev/shm XC store,
    another engine attaches to it (role 1, no fill) and decodes the same tokens with the same
    bytes on the link -- the attach path reads the blob sizes from the shared file."""
    import os
    import paper_2511_14102_b200 as m
    cfg = m.ModelConfig.named("tiny")
    path = "/dev/shm/mspq_test_store_%d" % os.getpid()
    conf = {"policy": "speculative", "cache_capacity": 3, "k": 3}
    try:
        owner = m.Engine(cfg, kmax=8, trace_level=1, host_store_path=path, host_store_role=0)
        guest = m.Engine(cfg, kmax=8, trace_level=1, host_store_path=path, host_store_role=1)
        reps = []
        for eng in (owner, guest):
            eng.configure(conf)
            reps.append(eng.generate([3, 9, 27], 20))
        assert reps[0]["tokens"] == reps[1]["tokens"]
        assert reps[0]["h2d_bytes"] == reps[1]["h2d_bytes"] > 0
        assert owner.info()["expert_wire_bytes_mean"] == guest.info()["expert_wire_bytes_mean"]
        guest.close()
        owner.close()
    finally:
        for p in (path, path + ".ready"):
            if os.path.exists(p):
                os.unlink(p)


@pytest.mark.parametrize("codec", ["none", "xc"])
def test_prefetch_issue_order_changes_nothing_but_timing(cuda, codec):
    """"prefetch_defer" (default on) issues each layer's plan prefetches behind the previous
    layer's demand copies instead of in plan order at draft time: tokens, routing, the hit/miss
    log and the bytes moved are unchanged."""
    import paper_2511_14102_b200 as m
    cfg = m.ModelConfig.named("tiny")
    reps = []
    for defer in (False, True):
        eng = m.Engine(cfg, kmax=8, trace_level=2, expert_codec=codec)
        eng.configure({"policy": "speculative", "cache_capacity": 3, "k": 4, "prefetch_defer": defer})
        reps.append(eng.generate([5, 17, 101, 9], 32))
        eng.close()
    a, b = reps
    assert a["tokens"] == b["tokens"]
    assert a["h2d_bytes"] == b["h2d_bytes"] > 0
    for ca, cb in zip(a["cycles"], b["cycles"]):
        for key in ["draft_tokens", "target_argmax", "target", "log", "new_experts"]:
            assert ca[key] == cb[key], key


def test_verify_overlap_changes_nothing_but_timing(cuda):
    """verify_overlap runs a layer's GEMM in two parts (resident experts first, in-flight ones
    after their copies land): tokens, routing and the hit/miss log are unchanged."""
    import paper_2511_14102_b200 as m
    cfg = m.ModelConfig.named("tiny")
    reps = []
    for ov in (False, True):
        eng = m.Engine(cfg, kmax=8, trace_level=2)
        eng.configure({"policy": "speculative", "cache_capacity": 3, "k": 3, "verify_overlap": ov})
        reps.append(eng.generate([5, 17, 101], 24))
        eng.close()
    a, b = reps
    assert a["tokens"] == b["tokens"]
    for ca, cb in zip(a["cycles"], b["cycles"]):
        for key in ["draft_tokens", "target_argmax", "target", "log", "new_experts"]:
            assert ca[key] == cb[key], key


def test_cycle_record_layer_times_are_ordered(cuda):
    """The per-layer event times (tools/cycle_timeline.py reads them) follow the verify chain:
    K1 done <= controller done <= GEMM start < GEMM end <= next layer's K1 done, all inside the
    cycle's span."""
    eng, cfg = _engine()
    eng.configure({"policy": "speculative", "cache_capacity": 3, "k": 3})
    rep = eng.generate([5, 6, 7], 12)
    for c in rep["cycles"]:
        lt = c["layer_times"]
        assert len(lt) == cfg.L and all(len(v) == 4 for v in lt)
        t0, t1 = c["start_s"], c["start_s"] + c["span_s"]
        prev_end = t0
        for w0, k0, ge, rt in lt:
            assert prev_end <= rt <= w0 <= k0 < ge <= t1 + 1e-6
            prev_end = ge
    eng.close()


@pytest.mark.parametrize("estimator", ["linear", "elb"])
@pytest.mark.parametrize("cap", [3, 6])
def test_live_governor_k_sequence_matches_reference_governor(cuda, ref, estimator, cap):
    """The live governor's k per cycle equals the reference select_k (perfmodel.cpp:166-183, run
    from oracle/_ref) fed the run's own re-fitted profile, the EMA acceptance of the outcomes so
    far and the |E_new(k)| estimate: the reference's linear g*k (sim.cpp:75-78, 404) or the elb
    estimator restated in oracle/control_plane.elb_estimate over the oracle's own cache replay."""
    eng, cfg = _engine()
    conf = {"policy": "speculative", "cache_capacity": cap, "k": "governor",
            "governor": {"k_min": 1, "k_max": 8, "k_slo": 8}, "estimator": estimator}
    eng.configure(conf)
    rep = eng.generate([42, 7, 300], 72)
    want = cp.live_governor_ks(rep, conf, cfg.L, cfg.E, cfg.K, estimator, kmax=8)
    assert [c["k"] for c in rep["cycles"]] == [w["k"] for w in want]
    assert [c["est_new_experts"] for c in rep["cycles"]] == [w["est"] for w in want]
    for w in want:
        req = {"profile": rep["profile"], "p": w["p"], "alpha": 0.1, "k_min": 1, "k_max": 8, "k_slo": 8}
        if estimator == "elb":
            req["est"] = w["table"]
        else:
            req["g"] = w["g"]
        assert ref.governor(req)["select_k"] == w["select_k"]
    eng.close()


def test_live_collect_plans_and_sync_fetch(cuda):
    """collect_plans in live mode (sim.cpp:377-392): each cycle record carries the device
    planner's prefetch items (= the causal planner restatement's) and the verify schedule K3 ran
    (= reorder_verification of the window, scheduler.cpp:339-357); sync_fetch_s is the measured
    time of the verify-time copies (demand misses and staged refills), > 0 whenever a demand miss
    was fetched."""
    eng, cfg = _engine()
    conf = {"policy": "speculative", "cache_capacity": 3, "k": 4, "collect_plans": True}
    eng.configure(conf)
    rep = eng.generate([9, 8, 7], 30)
    c = cp.sim_config(conf)
    cache = cp.Cache(c["capacity_mode"], c["cache_capacity"])
    head = 2
    for cyc in rep["cycles"]:
        out = cp.live_cycle(cache, cp.ELB.build(cyc["elb"], cyc["elb_gates"]), cyc["target"], c)
        got = [(p["issue_after_token"], (p["layer"], p["expert"]), p["phase"]) for p in cyc["prefetch_plan"]]
        assert got == [(r, tuple(k), ph) for (r, k, ph) in out["plan_items"]]
        T = cyc["k"] + 1
        window = list(range(head, head + T))
        routing = [[cyc["target"][s][l] for s in range(T)] for l in range(cfg.L)]
        want = cp.reorder_verification(window, routing)
        assert [lay["groups"] for lay in cyc["execution_plan"]] == want
        assert cyc["sync_fetch_s"] > 0 or cyc["sync_count"] == 0
        head += cyc["accepted"] + 1
    eng.close()


def test_live_fidelity_and_entropy_equal_reference_on_exported_trace(cuda, ref):
    """The live report's draft->target routing fidelity (both granularities) and per-layer
    routing entropy equal the reference's classify_fidelity / layer_entropy (trace.cpp:401-462,
    run from oracle/_ref) on the reference trace the same run exports (to_reference_trace)."""
    import paper_2511_14102_b200 as m
    eng, cfg = _engine()
    eng.configure({"policy": "speculative", "cache_capacity": 3, "k": 4})
    rep = eng.generate([3, 1, 4, 1, 5], 48)
    eng.close()
    want = ref.trace_analysis(m.to_reference_trace(rep, cfg))
    assert rep["fidelity"] == want["fidelity"]
    assert rep["layer_entropy"] == want["layer_entropy"]
    assert 0.0 < rep["fidelity"]["token_layer"]["hard_rate"] <= 1.0


def test_device_compare_policies_and_sweep_k_equal_reference(cuda, ref):
    """compare_policies / sweep_k (sim.cpp:539-574) over the device control plane equal the
    reference's rows on the same trace."""
    import paper_2511_14102_b200 as m
    tr = ref.generate_trace(4, 12, 2, 120, seed=3)
    base = {"policy": "speculative", "cache_capacity": 4, "k": 4}
    pols, caps = ["lru", "lookahead", "speculative"], [3, 6]
    assert m.compare_policies(tr, base, pols, caps) == ref.compare_policies(tr, base, pols, caps)
    assert m.sweep_k(tr, base, [1, 2, 5, 8]) == ref.sweep_k(tr, base, [1, 2, 5, 8])


def test_hardware_profile_refit_is_measured(cuda):
    """The B200 re-fit of HardwareProfile (perfmodel.hpp:15-30): PCIe bandwidth, init latency and
    per-copy overhead from timed copies, draft time from the captured draft graph, and verify
    samples from timed target passes at windows 1/5/9 with the expected expert union resident."""
    eng, cfg = _engine()
    eng.configure({"policy": "speculative", "cache_capacity": 3, "k": "governor",
                   "governor": {"k_min": 1, "k_max": 8, "k_slo": 8}})
    info = eng.info()
    prof = info["profile"]
    vs = info["verify_samples_measured"]
    assert [w for w, _ in vs] == [1.0, 5.0, 9.0]  # kmax 8: windows up to 9
    assert all(t > 0 for _, t in vs) and vs[-1][1] >= vs[0][1]
    assert prof["verify_samples"] == vs
    assert prof["pcie_init_latency_s"] == info["pcie_init_latency_measured"] > 0
    assert prof["pcie_overhead_s"] == info["pcie_overhead_measured"] >= 0
    assert prof["draft_per_token_s"] == info["draft_step_s"] > 0
    eng.close()


@pytest.mark.parametrize("codec", ["xc", "none"])
@pytest.mark.parametrize("policy", ["lru", "speculative"])
def test_refetch_from_hbm_moves_bytes_not_decisions(cuda, codec, policy):
    """An expert evicted and requested again inside one verify layer is copied HBM -> HBM from its
    first-request buffer (parked until the layer's GEMM) instead of crossing the link again: the
    tokens, routing and hit/miss log are the run without it, the link carries fewer bytes."""
    import paper_2511_14102_b200 as m
    cfg = m.ModelConfig.named("tiny")
    conf = {"policy": policy, "cache_capacity": 2, "k": 8, "prefetch_budget": 1}
    reps = {}
    for on in (False, True):
        eng = m.Engine(cfg, kmax=8, trace_level=2, expert_codec=codec)
        eng.configure(dict(conf, refetch_from_hbm=on))
        reps[on] = eng.generate([3, 1, 4, 1, 5], 40)
        eng.close()
    a, b = reps[False], reps[True]
    assert a["tokens"] == b["tokens"] and a["total_new_experts"] == b["total_new_experts"]
    for ca, cb in zip(a["cycles"], b["cycles"]):
        for key in ["k", "draft_tokens", "target_argmax", "target", "log", "new_experts"]:
            assert ca[key] == cb[key], key
    assert a["refetch_hbm"] == 0 and b["refetch_hbm"] > 0
    assert b["h2d_bytes"] < a["h2d_bytes"]
    if codec == "none":
        S = cfg.expert_bytes_bf16()
        assert a["h2d_bytes"] - b["h2d_bytes"] == b["refetch_hbm"] * S
