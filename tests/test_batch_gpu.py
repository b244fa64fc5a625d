"""Batched multi-stream decode (mspq_generate_batch, include/mspq_capi.h).

Several request streams share one layer-major verify pass per cycle: their windows are
concatenated into one batch (attention with per-token stream/position metadata, one controller
step over every slot, one grouped GEMM per layer).  Batching changes the schedule, never the
text: every stream's tokens must equal its own greedy decode (the CPU oracle's and the solo
engine's), and the batch's cache hit/miss sequence must equal oracle/control_plane.live_cycle
under lru replayed over the concatenated window targets."""
import pytest

from oracle import control_plane as cp
from oracle import model as om
from helpers import _events, device_events, oracle_model

pytestmark = pytest.mark.gpu
PROMPTS = [[7, 100, 3, 250, 11], [42], [1, 2, 3], [9, 9, 9, 9, 9, 9, 9, 9]]
CONF = {"policy": "lru", "cache_capacity": 3, "k": 4}


def _engine(streams, name="tiny", codec="xc"):
    import paper_2511_14102_b200 as m
    cfg = m.ModelConfig.named(name)
    return m.Engine(cfg, kmax=8, trace_level=2, max_streams=streams, expert_codec=codec), cfg


@pytest.mark.parametrize("codec", ["xc", "none"])
def test_batch_streams_equal_solo_greedy_and_oracle(cuda, codec):
    eng, cfg = _engine(4, codec=codec)
    eng.configure(CONF)
    n_new = 24
    rep = eng.generate_batch(PROMPTS, n_new)
    assert rep["streams"] == len(PROMPTS)
    model = oracle_model(cfg)
    solo, _ = _engine(1, codec=codec)
    solo.configure(CONF)
    for i, p in enumerate(PROMPTS):
        got = rep["tokens"][i]
        assert len(got) == n_new
        oc = om.speculative_decode(model, p[-1], len(p) - 1, [1] * n_new, n_new, prompt=p)
        want = [t for o in oc for t in o["committed"]][:n_new]
        assert got == want, ("stream", i)
        assert solo.generate(p, n_new)["tokens"] == want
    # every cycle batches the active streams' windows back to back
    for cyc in rep["cycles"]:
        assert len(cyc["target"]) == len(cyc["streams"]) * (cyc["k"] + 1)
        assert len(cyc["tokens"]) == len(cyc["streams"])
    eng.close()
    solo.close()


def test_batch_hit_miss_sequence_equals_lru_oracle(cuda):
    eng, cfg = _engine(3)
    eng.configure(CONF)
    rep = eng.generate_batch(PROMPTS[:3], 20)
    c = cp.sim_config(CONF)
    cache = cp.Cache(c["capacity_mode"], c["cache_capacity"])
    fetched = refetch = 0
    for cyc in rep["cycles"]:
        log = []
        out = cp.live_cycle(cache, cp.ELB.build([]), cyc["target"], c, log)
        assert device_events(cyc["log"]) == _events(log), ("hit/miss log", cyc["cycle"])
        assert cyc["new_experts"] == out["fetched"]
        fetched += out["fetched"]
        refetch += out["refetch"]
    assert rep["total_new_experts"] == fetched > 0
    assert rep["refetch_hbm"] == refetch > 0  # windows of 3 streams re-request evicted experts
    assert rep["h2d_bytes"] > 0
    eng.close()


def test_batch_rejects_bad_requests(cuda):
    import paper_2511_14102_b200 as m
    eng, _ = _engine(2)
    eng.configure(CONF)
    with pytest.raises(m.MspqError):
        eng.generate_batch(PROMPTS[:3], 8)  # more streams than max_streams
    eng.configure({"policy": "speculative", "cache_capacity": 3, "k": 4})
    with pytest.raises(m.MspqError):
        eng.generate_batch(PROMPTS[:2], 8)  # the batch path runs the lru controller only
    eng.close()
