"""Multi-GPU path = independent replicas.  CPU (gloo, world_size 2): the bench's
aggregation is max-over-ranks time / sum-over-ranks tokens.  GPU: two engines share one
/dev/shm pinned expert store (rank 0 creates + fills, rank 1 attaches) and decode identically."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    dev_t, wall, tok = [(1.5, 2.0, 40), (2.5, 2.25, 24)][rank]
    r = bench.aggregate(dev_t, wall, tok, world)
    out[rank] = torch.tensor(r, dtype=torch.float64)
    dist.barrier()
    dist.destroy_process_group()


def test_replica_aggregation_gloo_world2():
    out = torch.zeros(2, 3, dtype=torch.float64).share_memory_()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        assert out[r].tolist() == [2.5, 2.25, 64.0]


@pytest.mark.gpu
def test_shared_pinned_store_two_engines(cuda, tmp_path):
    import paper_2511_14102_b200 as m
    path = f"/dev/shm/mspq_test_store_{os.getpid()}"
    cfg = m.ModelConfig.named("tiny")
    try:
        a = m.Engine(cfg, kmax=8, host_store_path=path, host_store_role=0, trace_level=0)
        b = m.Engine(cfg, kmax=8, host_store_path=path, host_store_role=1, trace_level=0)
        conf = {"policy": "speculative", "cache_capacity": 3, "k": 3}
        a.configure(conf)
        b.configure(conf)
        ra, rb = a.generate([9, 8, 7], 20), b.generate([9, 8, 7], 20)
        assert ra["tokens"] == rb["tokens"]
        assert ra["total_new_experts"] == rb["total_new_experts"]
        assert a.read("expert:1:3", 1024) == b.read("expert:1:3", 1024)
        a.close()
        b.close()
    finally:
        for p in (path, path + ".ready"):
            if os.path.exists(p):
                os.unlink(p)
