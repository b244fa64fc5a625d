"""NVLink peer-expert tier with home partitioning (include/mspq_capi.h (3)).

The tier changes WHERE a fetched expert's bytes come from (a peer's HBM home region instead of
the pinned host store over PCIe), never WHAT is fetched: tokens, routing, the hit/miss event
log and the fetch counts must equal the plain engine's, while the PCIe bytes go to zero once
every home is attached.  The box has one GPU, so the peers are engines on the same device: in
this process (mspq_engine_peer_attach) and in two processes exchanging CUDA IPC handles over a
gloo group (mspq_engine_peer_attach_ipc) -- the same code path a multi-GPU box takes over
NVLink / NVSwitch."""
import os

import pytest

pytestmark = pytest.mark.gpu
CONF = {"policy": "speculative", "cache_capacity": 3, "k": 4}
PROMPT = [5, 17, 101, 9]


def _engine(codec="xc"):
    import paper_2511_14102_b200 as m
    cfg = m.ModelConfig.named("tiny")
    eng = m.Engine(cfg, kmax=8, trace_level=2, expert_codec=codec)
    eng.configure(CONF)
    return eng


def _same_decisions(a, b):
    assert a["tokens"] == b["tokens"]
    assert a["total_new_experts"] == b["total_new_experts"] > 0
    for ca, cb in zip(a["cycles"], b["cycles"]):
        for key in ["k", "draft_tokens", "target_argmax", "target", "elb", "log", "new_experts"]:
            assert ca[key] == cb[key], key


@pytest.mark.parametrize("codec", ["xc", "none"])
def test_peer_tier_in_process_moves_bytes_not_decisions(cuda, codec):
    base = _engine(codec)
    want = base.generate(PROMPT, 32)
    base.close()
    e0, e1 = _engine(codec), _engine(codec)
    e0.home_create(2, 0)
    e1.home_create(2, 1)
    e0.peer_attach(1, e1)
    e1.peer_attach(0, e0)
    got = e0.generate(PROMPT, 32)
    _same_decisions(got, want)
    pt = got["peer_tier"]
    assert got["h2d_bytes"] == 0 and pt["pcie_fetches"] == 0
    assert pt["peer_fetches"] > 0 and pt["home_local_fetches"] > 0
    assert pt["peer_fetches"] + pt["home_local_fetches"] + got["refetch_hbm"] == got["total_new_experts"]
    S = e0.model.expert_bytes_bf16()
    assert pt["peer_bytes"] == pt["peer_fetches"] * S and pt["home_local_bytes"] == pt["home_local_fetches"] * S
    e0.close()
    e1.close()


def test_peer_tier_unattached_peer_falls_back_to_pcie(cuda):
    base = _engine()
    want = base.generate(PROMPT, 24)
    base.close()
    e0 = _engine()
    e0.home_create(2, 0)  # rank 1's experts have no attached home: they still cross PCIe
    got = e0.generate(PROMPT, 24)
    _same_decisions(got, want)
    pt = got["peer_tier"]
    assert pt["peer_fetches"] == 0 and pt["pcie_fetches"] > 0 and pt["home_local_fetches"] > 0
    assert got["h2d_bytes"] > 0
    e0.close()


def _rank_main(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eng = _engine()
        h = eng.home_create(world, rank)
        hs = [None] * world
        dist.all_gather_object(hs, h)
        for r in range(world):
            if r != rank:
                eng.peer_attach_ipc(r, hs[r])
        dist.barrier()
        rep = eng.generate(PROMPT, 32)
        dist.barrier()  # keep every home mapped until all ranks are done reading
        q.put((rank, {k: rep[k] for k in ("tokens", "total_new_experts", "cycles", "h2d_bytes", "peer_tier")}))
        eng.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_peer_tier_two_processes_over_cuda_ipc(cuda):
    import socket

    import torch.multiprocessing as mp
    base = _engine()
    want = base.generate(PROMPT, 32)
    base.close()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    for r in range(2):
        assert isinstance(out[r], dict), out[r]
        _same_decisions(out[r], want)
        pt = out[r]["peer_tier"]
        assert out[r]["h2d_bytes"] == 0 and pt["peer_fetches"] > 0 and pt["home_local_fetches"] > 0


def _store_rank_main(rank, world, port, path, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2511_14102_b200 as m
        cfg = m.ModelConfig.named("tiny")
        eng = m.Engine(cfg, kmax=8, trace_level=2, host_store_path=path, host_store_role=0 if rank == 0 else 1)
        eng.configure(CONF)
        rep = eng.generate(PROMPT, 32)
        dist.barrier()  # the owner keeps the store mapped until every rank is done
        q.put((rank, {k: rep[k] for k in ("tokens", "total_new_experts", "cycles", "h2d_bytes")}))
        eng.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_shared_host_store_two_processes(cuda):
    """bench.py's multi-rank layout on one box: rank 0 creates and fills the /dev/shm pinned store,
    rank 1 attaches to it from another process (record + size check), and both decode the same
    tokens with the same cache decisions and the same bytes on the link."""
    import socket

    import torch.multiprocessing as mp
    base = _engine()
    want = base.generate(PROMPT, 32)
    base.close()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    path = "/dev/shm/mspq_test_store2_%d" % os.getpid()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_store_rank_main, args=(r, 2, port, path, q)) for r in range(2)]
    try:
        for p in ps:
            p.start()
        out = dict(q.get(timeout=600) for _ in ps)
        for p in ps:
            p.join(timeout=120)
    finally:
        for f in (path, path + ".ready"):
            if os.path.exists(f):
                os.unlink(f)
    for r in range(2):
        assert isinstance(out[r], dict), out[r]
        _same_decisions(out[r], want)
        assert out[r]["h2d_bytes"] == want["h2d_bytes"] > 0
