"""bench.py — decode tokens/s of the B200 MoE-SpeQ hot path (BASELINE.json metric).

Workload (N=1): BASELINE config 3 — Phi-3.5-MoE-shaped (L=32, E=16, top-2, d=4096, ffn=6400,
vocab 32064) random-init model, INT4 draft of itself, governor-tuned speculation length
(k in [1,16]), expert cache capped at 25% of each layer's experts (4 of 16), all 512 bf16
experts (80.5 GB) in pinned host DRAM, fed over PCIe by copy engines.

A "step" = one Engine.generate() call decoding --tokens (default 256) new tokens
for a fresh synthetic 128-token prompt (prompts differ per step; the expert cache and the
governor's learned state stay warm across steps, as in serving).

  value      committed tokens / sum of device-timed decode spans (CUDA events on the engine's
             compute stream, cycle start -> accept), max over ranks
  e2e        same metric through the public API (Engine.generate -> C-ABI mspq_generate) by
             wall clock, including prompt H2D and result D2H each step
  roofline   dominant kernel = K3 (bf16 grouped verify FFN): algorithmic weight bytes per launch
             / mean launch duration (CUDA events around each launch), vs measured HBM GB/s
  path_roofline  the path bound: PCIe bytes the policy moved / measured H2D GB/s
  cpu_baseline   the CPU oracle decode (oracle/model.py + the OpenMP oracle/csrc/decode_ref.c:
             the same model, weights and greedy speculative decode, fp32/f64) on all host cores,
             time-boxed on the bench model ("kind": "port"); cpu_reference_sim = the reference's
             own CPU path (run_simulation from oracle/_ref) on the same shape / cache budget
  --impl reference   the reference's run_simulation on a routing trace this engine produced for
             the bench config (tests/golden/live_trace_phi_cap4.jsonl, exported with
             to_reference_trace) under the B200-fitted profile, all host threads

Multi-GPU (torchrun): independent request streams, one engine per GPU (replicas) over ONE
shared pinned host store in /dev/shm; no data-path collective ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s, Phi-MoE shape, capped expert cache; exposed H2D ms/token"
CONFIG_NO = {"tiny": 1, "mixtral": 2, "phi": 3, "qwen3": 4}  # BASELINE.json configs[] (1-based)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="phi")
    ap.add_argument("--tokens", type=int, default=256, help="new tokens per step (PAPER.md:184)")
    ap.add_argument("--cap", type=int, default=0, help="per-layer cache capacity (0 = 25%% of E)")
    ap.add_argument("--policy", default="speculative")
    ap.add_argument("--k", default="governor")
    ap.add_argument("--unique", type=int, default=0, help="distinct expert payloads (0 = all)")
    ap.add_argument("--codec", default="xc", choices=["xc", "none"],
                    help="host-store format of the bf16 experts: xc = lossless exponent-coded (default)")
    ap.add_argument("--verify-overlap", action="store_true",
                    help="run the verify GEMM of resident experts while a layer's copies are in flight")
    ap.add_argument("--estimator", default="linear", choices=["linear", "elb"],
                    help="governor |E_new(k)| estimator: the reference's linear g*k or the ELB-based one")
    ap.add_argument("--peer-tier", action="store_true",
                    help="NVLink peer-expert tier: every rank keeps the experts e %% N == rank in an HBM home "
                         "region and serves misses from the owner's home (N=1: the GPU's own home)")
    ap.add_argument("--streams", type=int, default=0,
                    help="independent request streams over all ranks (BASELINE config 5: 8); stream s is served "
                         "by rank s %% N, a rank's streams one after another on its engine; 0 = one per rank")
    ap.add_argument("--batch", action="store_true",
                    help="decode a rank's streams together (Engine.generate_batch: one verify pass per cycle over "
                         "every stream's window, shared expert reads and fetches); needs --policy lru")
    ap.add_argument("--same-device", action="store_true",
                    help="test mode: every rank uses cuda:0 (exercises the multi-rank path on a one-GPU box)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="time box of the CPU oracle decode")
    ap.add_argument("--out", default="")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.samples, self.stop, self.index = [], threading.Event(), index
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self.stop.is_set():
            try:
                r = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                v = [x.strip() for x in r.stdout.strip().split(",")]
                if len(v) == 6:
                    self.samples.append(v)
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def aggregate(dev_t, wall, tok, world):
    """Replica aggregation: times are the MAX over ranks, tokens the SUM (whole-job throughput
    = all ranks' tokens / slowest rank).  Timing only -- no data-path collective."""
    import torch
    if world <= 1:
        return dev_t, wall, float(tok)
    import torch.distributed as dist
    t = torch.tensor([dev_t, wall], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n = torch.tensor([float(tok)], dtype=torch.float64)
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    return t[0].item(), t[1].item(), n[0].item()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return j.get("hbm_gbs", 6650.0), j.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


def ncu_traffic():
    """dram read+write bytes per launch of k_umma_grouped from the committed ncu --set full
    capture (profiles/), with that launch's algorithmic bytes for comparison."""
    p = os.path.join(ROOT, "profiles", "r01", "ncu_raw_k_umma_grouped.txt")
    if not os.path.exists(p):
        return None
    v = {}
    for ln in open(p):
        k, _, val = ln.partition(" = ")
        v[k.strip()] = val.strip()
    try:
        rd = float(v["dram__bytes_read.sum"]) * 1e6  # MB in the capture
        wr = float(v["dram__bytes_write.sum"]) * 1e6
    except (KeyError, ValueError):
        return None
    return {"bytes_per_launch": rd + wr, "algorithmic_bytes_per_launch": 7 * 12800 * 4096 * 2,
            "source": "profiles/r01/ncu_raw_k_umma_grouped.txt (W13 GEMM of one verify layer, 7 experts)"}


def prompts(n, V, seed):
    import random
    rng = random.Random(seed)
    return [[rng.randrange(V) for _ in range(128)] for _ in range(n)]


def reference_cpu(shape, cap, tokens, policy, kspec, threads, seconds=10.0, seed=0):
    """The reference's own CPU path (run_simulation from oracle/_ref) on this workload shape:
    Phi-shaped synthetic routing trace, same cache budget/policy/governor.  Returns
    (tokens/s over all threads, sample description)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import ref
    L, E, K, S = shape
    cfg = {"policy": policy, "cache_capacity": cap}
    if kspec == "governor":
        cfg.update(k="governor", governor={"k_min": 1, "k_max": 16, "k_slo": 16})
    else:
        cfg["k"] = int(kspec)
    traces = [ref.generate_trace(L, E, K, tokens, seed=seed + i, expert_bytes=S) for i in range(threads)]
    done = [0] * threads

    def worker(i):
        t_end = time.perf_counter() + seconds
        n = 0
        while time.perf_counter() < t_end:
            r = ref.run_simulation(traces[i], cfg)
            n += r["total_tokens"]
        done[i] = n

    t0 = time.perf_counter()
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(worker, range(threads)))
    dt = time.perf_counter() - t0
    return sum(done) / dt, f"run_simulation on {threads} x {tokens}-token synthetic traces (L={L},N={E},top_k={K}), {seconds:.0f}s"


LIVE_TRACE = os.path.join(ROOT, "tests", "golden", "live_trace_phi_cap4.jsonl")


def cpu_oracle_decode(model_name, seconds, kw=None):
    """The CPU oracle's greedy speculative decode (oracle/model.py; expert FFN and LM head in the
    OpenMP oracle/csrc/decode_ref.c) of the bench model with the same random-init weights, k=1
    cycles, time-boxed: committed tokens / elapsed.  Returns (tokens/s, threads, sample)."""
    from oracle import model as om
    import paper_2511_14102_b200 as m
    cfg = m.ModelConfig.named(model_name, **(kw or {}))
    desc = om.ModelDesc(**cfg.oracle_kwargs())
    model = om.Model(desc, fast=True)
    model.lm()  # weight generation of the LM head is setup, not decode
    prompt = [11, 200, 3001, 17]
    model.kv = [dict() for _ in range(desc.L)]
    if desc.H > 0:
        om.prefill(model, prompt)  # excluded, like the GPU arm's prefill
    t0 = time.perf_counter()
    out = om.speculative_decode(model, prompt[-1], len(prompt) - 1, [1], 10**6, prompt=prompt,
                                deadline=t0 + seconds, prefilled=True)
    n = sum(len(o["committed"]) for o in out)
    cyc = len(out)
    dt = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    return n / dt, threads, (f"oracle greedy speculative decode of the {model_name} model (L={cfg.L}, E={cfg.E}, "
                             f"top-{cfg.K}, d={cfg.d}, ffn={cfg.f}), k=1, {cyc} cycles / {n} tokens in {dt:.1f}s, "
                             f"OpenMP over {threads} threads")


def run_reference_arm(a):
    """The reference's own CPU implementation of the path -- run_simulation (sim.cpp:458-466, built
    unmodified from /root/reference into oracle/_ref) -- on the bench config: the routing trace this
    engine produced for BASELINE config 3 (Phi shape, cap 4/16, speculative, governor), with the
    B200-fitted HardwareProfile that run measured, on all host threads.  value = simulated
    committed tokens per second of CPU time."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor
    from oracle import ref
    threads = os.cpu_count() or 1
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmoespeq_ref.so not built"}))
        return
    if not os.path.exists(LIVE_TRACE):
        print(json.dumps({"impl": "reference", "unavailable": "live routing trace fixture missing (tools/export_live_trace.py)"}))
        return
    lines = open(LIVE_TRACE).read().splitlines()
    head = json.loads(lines[0])
    trace = "\n".join(lines) + "\n"
    meta = head.get("meta", {})
    cfg = {"policy": meta.get("policy", "speculative"), "cache_capacity": int(meta.get("cache_capacity", 4)),
           "k": "governor", "governor": {"k_min": 1, "k_max": 16, "k_slo": 16},
           "profile": json.loads(meta["profile"])}
    rep0 = ref.run_simulation(trace, cfg)
    vals = []

    def worker(_):
        n, t_end = 0, time.perf_counter() + 3.0
        while time.perf_counter() < t_end:
            n += ref.run_simulation(trace, cfg)["total_tokens"]
        return n

    for i in range(a.warmup + a.steps):
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            n = sum(ex.map(worker, range(threads)))
        if i >= a.warmup:
            vals.append(n / (time.perf_counter() - t0))
    value = statistics.mean(vals)
    sample = (f"run_simulation replaying {len(lines) - 1} positions of the live Phi cap-4/16 routing trace "
              f"({os.path.basename(LIVE_TRACE)}), 3 s per step on each of {threads} threads")
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 3000.0, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (routing trace of this engine's bench config)",
            "config": {"workload": f"phi-shaped speculative decode (BASELINE config 3), per-layer cap "
                                   f"{cfg['cache_capacity']}/16, policy {cfg['policy']}, k=governor",
                       "cache_capacity_per_layer": cfg["cache_capacity"]},
            "same_config": True,
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_modeled_b200_tokens_per_s": rep0["total_tokens"] / rep0["total_time_s"],
            "reference_modeled_exposed_h2d_frac": rep0["stall_time_s"] / rep0["total_time_s"],
            "note": "the reference is a trace-driven simulator: its CPU path replays routing decisions and models "
                    "time; it computes no model math. reference_modeled_b200_tokens_per_s is its own prediction "
                    "of this decode under the profile this engine measured on the B200."}
    print(json.dumps(line))


def numa_node_of(local):
    """NUMA node and CPU list of GPU `local` (sysfs via its PCI bus id); (-1, None) if unknown."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(local)
        bus = "%04x:%02x:%02x.0" % (getattr(pr, "pci_domain_id", 0), pr.pci_bus_id, pr.pci_device_id)
        base = "/sys/bus/pci/devices/" + bus
        node = int(open(base + "/numa_node").read().strip())
        cpus = open(base + "/local_cpulist").read().strip()
        return node, cpus
    except Exception:  # noqa: BLE001
        return -1, None


def parse_cpulist(text):
    out = set()
    for part in text.split(","):
        if "-" in part:
            lo, hi = part.split("-")
            out.update(range(int(lo), int(hi) + 1))
        elif part:
            out.add(int(part))
    return out


def xc_ratio_gaussian(d, f, seed=7):
    """Lossless XC codec ratio of one expert with N(0, sigma^2) weights (SURVEY.md §8(d)'s
    distribution; the bench model itself is uniform-init): bf16 tile images of a d x f expert
    (W13 [2f][d] + W2 [d][f], sigma = 1/sqrt(d)) encoded with mspq_xc_encode."""
    import ctypes
    import torch
    from paper_2511_14102_b200._lib import check, lib
    g = torch.Generator(device="cuda").manual_seed(seed)
    w13 = (torch.randn(2 * f, d, device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(d, f, device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    n = 3 * d * f
    img = torch.empty(n, dtype=torch.int16, device="cuda")
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    check(lib().mspq_tile_bf16(P(w13), 2 * f, d, P(img), None))
    check(lib().mspq_tile_bf16(P(w2), d, f, ctypes.c_void_p(img.data_ptr() + 2 * f * d * 2), None))
    n_tiles = n * 2 // 16384
    scratch = torch.empty(lib().mspq_xc_scratch_bytes(n_tiles), dtype=torch.uint8, device="cuda")
    cap = lib().mspq_xc_max_blob_bytes(n_tiles)
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb = ctypes.c_longlong(0)
    check(lib().mspq_xc_encode(P(img), n_tiles, P(scratch), P(out), cap, ctypes.byref(nb), None))
    torch.cuda.synchronize()
    return nb.value / (n * 2)


def spawn_ranks(a):
    """--gpus N without torchrun: relaunch this script under torch.distributed.run, one rank per
    GPU on this node (127.0.0.1 rendezvous), and return its exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    a = parse()
    if a.batch and a.policy != "lru":  # generate_batch runs the lru controller (no draft-driven planner)
        a.policy = "lru"
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a))
    if a.impl == "reference":
        return run_reference_arm(a)
    rank, world, local = dist_env()
    if a.same_device:
        local = 0
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    import paper_2511_14102_b200 as m
    cfgm = m.ModelConfig.named(a.model, unique_experts=a.unique)
    E, K, L = cfgm.E, cfgm.K, cfgm.L
    cap = a.cap or max(K, E // 4)
    # NUMA placement: run this rank on its GPU's node and give every node one copy of the pinned
    # store (a PCIe read then stays on the GPU's own socket); this box has one node
    node, cpus = numa_node_of(local)
    if cpus:
        try:
            os.sched_setaffinity(0, parse_cpulist(cpus))
        except OSError:
            pass
    store = ""
    if world > 1:
        # one shared pinned store per NUMA node and run: rank 0 picks a fresh name (no stale file can be
        # attached), the lowest rank of each node creates its node's copy, the others attach once its
        # ready record is published (live.cpp alloc_host_store)
        name = ["/dev/shm/mspq_store_%s_%d_%d" % (a.model, os.getpid(), time.time_ns() % 10**9)]
        torch.distributed.broadcast_object_list(name, src=0)
        nodes = [None] * world
        torch.distributed.all_gather_object(nodes, node)
        store = "%s_n%d" % (name[0], max(node, 0))
        store_owner = min(r for r in range(world) if nodes[r] == node)
    t_create = time.perf_counter()
    n_streams = a.streams or world
    mine = [st for st in range(n_streams) if st % world == rank]
    eng = m.Engine(cfgm, kmax=16, device=local, host_store_path=store or None,
                   host_store_role=0 if (not store or rank == store_owner) else 1, trace_level=0,
                   expert_codec=a.codec, max_streams=len(mine) if a.batch else 1)
    t_create = time.perf_counter() - t_create
    t_home = 0.0
    if a.peer_tier:
        t_home = time.perf_counter()
        h = eng.home_create(world, rank)
        if world > 1:
            hs = [None] * world
            torch.distributed.all_gather_object(hs, h)
            for r in range(world):
                if r != rank:
                    eng.peer_attach_ipc(r, hs[r])
        t_home = time.perf_counter() - t_home
    conf = {"policy": a.policy, "cache_capacity": cap}
    if a.verify_overlap:
        conf["verify_overlap"] = True
    if a.k == "governor":
        conf.update(k="governor", governor={"k_min": 1, "k_max": 16, "k_slo": 16})
        if a.estimator != "linear":
            conf["estimator"] = a.estimator
    else:
        conf["k"] = int(a.k)
    eng.configure(conf)
    ps = {st: prompts(a.warmup + a.steps, cfgm.V, seed=1000 + st) for st in mine}

    def step(i):  # one step = every stream of this rank decodes --tokens new tokens
        if a.batch:
            return [eng.generate_batch([ps[st][i] for st in mine], a.tokens)]
        return [eng.generate(ps[st][i], a.tokens) for st in mine]

    for i in range(a.warmup):
        step(i)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    reps = []
    with ClockSampler(local) as clk:
        w0 = time.perf_counter()
        for i in range(a.steps):
            reps.extend(step(a.warmup + i))
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    if world > 1:
        torch.distributed.barrier()
    info = eng.info()
    pts = [r["peer_tier"] for r in reps if "peer_tier" in r]
    tok = sum(r["total_tokens"] for r in reps)
    dev_t = sum(r["total_time_s"] for r in reps)
    stall = sum(r["stall_time_s"] for r in reps)
    h2d = sum(r["h2d_bytes"] for r in reps)
    h2d16 = sum(r["h2d_bytes_bf16"] for r in reps)
    fetched = sum(r["total_new_experts"] for r in reps)
    k3_t = sum(r["kernels"]["k3_time_s"] for r in reps)
    k3_b = sum(r["kernels"]["k3_weight_bytes"] for r in reps)
    k3_n = sum(r["kernels"]["k3_launches"] for r in reps)
    dr_t = sum(r["kernels"]["draft_time_s"] for r in reps)
    dr_n = sum(r["kernels"]["draft_steps"] for r in reps)
    launches = sum(r["kernels"]["kernel_launches"] for r in reps)
    ks = [c for r in reps for c in r.get("cycles", [])]
    mean_k = statistics.mean([c["k"] for c in ks]) if ks else None
    if a.batch:  # a batch cycle drafts k tokens for each of its streams
        acc = sum(sum(c["accepted"]) for c in ks) / max(1, sum(c["k"] * len(c["streams"]) for c in ks))
    else:
        acc = sum(c["accepted"] for c in ks) / max(1, sum(c["k"] for c in ks))
    dev_max, wall_max, tok_all = aggregate(dev_t, wall, tok, world)
    if rank != 0:
        eng.close()
        if store and rank == store_owner:  # this rank created its node's store copy
            for p in (store, store + ".ready"):
                try:
                    os.unlink(p)
                except OSError:
                    pass
        return
    hbm, tf, pk_kind = peaks()
    pcie_bw = info["pcie_bw_measured"]
    S16 = info["expert_bytes_bf16"]
    # per committed token roofline: PCIe leg (policy's bytes), HBM leg (draft + verify streaming)
    t_pcie = h2d / pcie_bw
    pb = sum(p["peer_bytes"] for p in pts)
    lb = sum(p["home_local_bytes"] for p in pts)
    # HBM leg: draft + verify weight streaming, plus the peer tier's copies (a local home copy
    # reads and writes this HBM, a peer copy writes it)
    hbm_bytes = dr_n * (reps[0]["kernels"]["draft_step_bytes"]) + k3_b + 2 * lb + pb
    t_hbm = hbm_bytes / (hbm * 1e9)
    t_roof = max(t_pcie, t_hbm)
    k3_ach = (k3_b / k3_n) / (k3_t / k3_n) / 1e9 if k3_t > 0 else 0.0
    line = {
        "metric": METRIC, "value": tok_all / dev_max, "unit": "tokens/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": dev_max / a.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if a.streams else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights from a counter hash, random prompts)",
        "config": {"workload": f"{a.model}-shaped speculative decode (BASELINE config {5 if a.streams else CONFIG_NO.get(a.model, '?')}), "
                               f"{a.tokens} tokens/step/stream, {n_streams} stream(s), "
                               f"per-layer expert cache {cap}/{E}, policy {a.policy}, k={a.k}, INT4 draft, bf16 verify",
                   "shape": {"name": a.model, "L": L, "E": E, "top_k": K, "d": cfgm.d, "ffn": cfgm.f, "vocab": cfgm.V},
                   "cache_capacity_per_layer": cap, "host_store_GB": info["host_store_bytes"] / 1e9,
                   "streams": n_streams, "streams_per_gpu": len(mine),
                   "stream_batching": "one verify pass per cycle over the rank's streams" if a.batch
                   else "a rank's streams one after another",
                   "expert_codec": a.codec,
                   "l2": "inputs larger than L2: each verify layer streams >= 157 MB of experts; no flush needed"},
        "exposed_h2d_ms_per_token": stall / max(tok, 1) * 1e3,
        "exposed_h2d_frac": stall / dev_t if dev_t else None,
        "mean_k": mean_k, "accept_rate": acc,
        "experts_fetched_per_token": fetched / max(tok, 1),
        "estimator": a.estimator,
        "e2e": {"value": tok_all / wall_max, "unit": "tokens/s", "h2d_bytes_per_step": 128 * 4 * len(mine),
                "d2h_bytes_per_step": a.tokens * 4 * len(mine),
                "note": "wall clock of Engine.generate() (host prompt in, host tokens out) including each "
                        "request's prefill of its 128-token prompt; decode_only excludes the prefill",
                "decode_only": tok / max(1e-9, sum(r.get("decode_wall_s", r["wall_s"]) for r in reps)),
                "prefill_s_per_step": sum(p.get("time_s", 0.0) for r in reps
                                          for p in (r.get("prefill") if isinstance(r.get("prefill"), list)
                                                    else [r.get("prefill", {})])) / a.steps,
                "expert_h2d_bytes_per_step": h2d / a.steps},
        "roofline": {"bound": "hbm",
                     "kernel": "K3 bf16 grouped verify FFN on tcgen05 (gather + k_umma_grouped W13 + SiLU + W2), per layer",
                     "achieved": k3_ach, "peak": hbm, "unit": "GB/s", "frac": k3_ach / hbm if hbm else None,
                     "traffic": ncu_traffic(), "peak_kind": pk_kind,
                     "bytes_per_launch": k3_b / max(k3_n, 1), "launch_ms": k3_t / max(k3_n, 1) * 1e3},
        "path_roofline": {"bound": "pcie" if t_pcie >= t_hbm else "hbm", "t_roof_s": t_roof,
                          "t_measured_s": dev_t, "frac": t_roof / dev_t if dev_t else None,
                          "pcie_GBps_achieved": h2d / dev_t / 1e9 if dev_t else None,
                          "pcie_GBps_peak_measured": pcie_bw / 1e9, "t_pcie_s": t_pcie, "t_hbm_s": t_hbm,
                          "wire_bytes_over_bf16": h2d / h2d16 if h2d16 else None,
                          "bf16_equiv_GBps": h2d16 / dev_t / 1e9 if dev_t else None,
                          "note": "PCIe leg = bytes actually moved (XC-coded experts) / measured pinned-H2D GB/s"},
        "draft_step_ms": dr_t / max(dr_n, 1) * 1e3,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "engine_create_s": t_create,
        "numa_node": node,
    }
    try:
        line["xc_ratio"] = {"bench_model_uniform_init": info["expert_wire_bytes_mean"] / info["expert_bytes_bf16"],
                            "gaussian_weights": xc_ratio_gaussian(cfgm.d, cfgm.f)}
    except Exception as e:  # noqa: BLE001
        line["xc_ratio"] = {"error": str(e)}
    if pts:
        line["peer_tier"] = {
            "group": world, "home_bytes_per_gpu": info["home_bytes"], "home_fill_s": t_home,
            "peer_fetches": sum(p["peer_fetches"] for p in pts), "home_local_fetches": sum(p["home_local_fetches"] for p in pts),
            "pcie_fetches": sum(p["pcie_fetches"] for p in pts), "peer_GBps": pb / dev_t / 1e9 if dev_t else None,
            "home_local_GBps": lb / dev_t / 1e9 if dev_t else None,
            "note": "misses served HBM->HBM from the owner's home region (expert id mod N); at N=1 every home is "
                    "this GPU's own, so the copies are local device-to-device, not NVLink"}
        line["config"]["workload"] += ", peer-expert tier (home partitioning)"
    if not a.no_cpu_baseline and world == 1:
        try:
            v, thr, sample = cpu_oracle_decode(a.model, a.cpu_seconds)
            line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "cores": thr, "kind": "port", "sample": sample}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "port",
                                    "sample": f"unavailable: {e}"}
        try:
            v, sample = reference_cpu((L, E, K, S16), cap, 2000, a.policy, a.k, 1, seconds=5.0)
            line["cpu_reference_sim"] = {"value": v, "unit": "tokens/s", "cores": 1, "kind": "reference",
                                         "sample": sample}
        except Exception as e:  # noqa: BLE001
            line["cpu_reference_sim"] = {"value": None, "sample": f"unavailable: {e}"}
    eng.close()
    if store and rank == store_owner:
        for p in (store, store + ".ready"):
            try:
                os.unlink(p)
            except OSError:
                pass
    out = json.dumps(line)
    print(out)
    if a.out:
        with open(a.out, "w") as f:
            f.write(out + "\n")


if __name__ == "__main__":
    main()
