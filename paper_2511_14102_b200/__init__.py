"""B200-native MoE-SpeQ decode hot path (arXiv 2511.14102).

Python mirror of the reference's public API for this path (proj/python/moespeq re-exports
proj/bindings/module.cpp): `run_simulation(trace, config)` keeps its name and meaning but runs
every cache decision on the GPU (device controller, K4); `Engine.generate(...)` is the live
speculative decode (INT4 draft -> ELB -> 3-phase prefetch over copy engines -> bf16 grouped
verify -> accept -> governor).  Configs use the reference run-config JSON schema
(run_config.hpp:30-50).  All compute goes through libmspq.so (include/mspq_capi.h); there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass

from . import _lib
from ._lib import MspqError, check, lib, take_string

__version__ = "0.1.0"

POLICIES = ["lru", "lookahead", "sp-sooner", "sp-later", "speculative"]

# BASELINE.json shapes (tiny ffn chosen = 512; Qwen3-30B-A3B moe_intermediate = 768) with the
# named models' attention heads (H query, Hkv KV, head dim Dh; tiny chosen 4/2/64)
MODEL_SHAPES = {
    "tiny": dict(L=4, E=8, K=2, d=256, f=512, V=512, H=4, Hkv=2, Dh=64),
    "mixtral": dict(L=32, E=8, K=2, d=4096, f=14336, V=32000, H=32, Hkv=8, Dh=128),
    "phi": dict(L=32, E=16, K=2, d=4096, f=6400, V=32064, H=32, Hkv=8, Dh=128),
    "qwen3": dict(L=48, E=128, K=8, d=2048, f=768, V=151936, H=32, Hkv=4, Dh=128),
}


@dataclass
class ModelConfig:
    """Model / draft config: ModelShape (trace.hpp:29-37) + the dims a real model needs."""
    L: int
    E: int
    K: int
    d: int
    f: int
    V: int
    P: int = 4096
    seed: int = 1234
    embed_scale: float = 1.0
    pos_scale: float = 0.5
    router_scale: float = 3.0
    moe_scale: float = 0.06
    lm_scale: float = 1.0
    eps: float = 1e-6
    unique_experts: int = 0
    H: int = 0      # attention query heads (0 = attention-free layers)
    Hkv: int = 0    # KV heads
    Dh: int = 0     # head dim

    @classmethod
    def named(cls, name, **kw):
        d = dict(MODEL_SHAPES[name])
        d.update(kw)
        return cls(**d)

    def _f32(self, x):
        return ctypes.c_float(x).value

    def desc(self) -> _lib.ModelDesc:
        f32 = self._f32
        return _lib.ModelDesc(self.L, self.E, self.K, self.d, self.f, self.V, self.P, self.seed,
                              self.embed_scale, self.pos_scale,
                              f32(self.router_scale * math.sqrt(3.0 / self.d)),
                              f32(math.sqrt(3.0 / self.d)),
                              f32(self.moe_scale * math.sqrt(3.0 / self.f)),
                              f32(self.lm_scale * math.sqrt(3.0 / self.d)), self.eps,
                              self.unique_experts, self.H, self.Hkv, self.Dh,
                              f32(math.sqrt(3.0 / self.d)),
                              f32(self.moe_scale * math.sqrt(3.0 / max(1, self.H * self.Dh))))

    def oracle_kwargs(self) -> dict:
        """The fields oracle/model.py ModelDesc takes (tests build the CPU oracle from these)."""
        return dict(L=self.L, E=self.E, K=self.K, d=self.d, f=self.f, V=self.V, P=self.P, seed=self.seed,
                    embed_scale=self.embed_scale, pos_scale=self.pos_scale, router_scale=self.router_scale,
                    moe_scale=self.moe_scale, lm_scale=self.lm_scale, eps=self.eps, H=self.H, Hkv=self.Hkv,
                    Dh=self.Dh)

    def expert_bytes_bf16(self):
        return lib().mspq_bf16_blob_bytes(self.d, self.f)

    def expert_bytes_int4(self):
        return lib().mspq_int4_blob_bytes(self.d, self.f)


def _cfg_json(config) -> bytes:
    if isinstance(config, (bytes, str)):
        return config.encode() if isinstance(config, str) else config
    return json.dumps(config).encode()


def run_simulation(trace_jsonl: str, config: dict, device: int = 0) -> dict:
    """run_simulation (sim.hpp:86) with the expert-cache control plane on the GPU.
    trace: reference JSONL text; config: reference run-config dict.  Returns the SimReport
    JSON dict (sim.cpp:468-510)."""
    out = ctypes.c_void_p()
    check(lib().mspq_replay(device, trace_jsonl.encode(), _cfg_json(config), ctypes.byref(out)))
    return json.loads(take_string(out))


replay = run_simulation


def compare_policies(trace_jsonl: str, config: dict, policies, capacities, device: int = 0) -> list:
    """compare_policies (sim.cpp:539-552) on the device control plane: one run_simulation per
    (policy, capacity); rows {"policy", "capacity", "coverage", "tpot"} (PolicyRow, sim.hpp:88-93)."""
    out = ctypes.c_void_p()
    check(lib().mspq_compare_policies(device, trace_jsonl.encode(), _cfg_json(config), json.dumps(list(policies)).encode(),
                                      json.dumps([int(c) for c in capacities]).encode(), ctypes.byref(out)))
    return json.loads(take_string(out))


def sweep_k(trace_jsonl: str, config: dict, ks, device: int = 0) -> list:
    """sweep_k (sim.cpp:563-574): fixed-k runs; rows {"k", "tpot", "mean_accepted", "coverage",
    "ttft"} (SweepRow, sim.hpp:101-107)."""
    out = ctypes.c_void_p()
    check(lib().mspq_sweep_k(device, trace_jsonl.encode(), _cfg_json(config), json.dumps([int(k) for k in ks]).encode(),
                             ctypes.byref(out)))
    return json.loads(take_string(out))


def governor(request: dict) -> dict:
    """Amortization-Roofline governor evaluation (perfmodel.cpp:85-217) in the product."""
    out = ctypes.c_void_p()
    check(lib().mspq_governor(json.dumps(request).encode(), ctypes.byref(out)))
    return json.loads(take_string(out))


class Engine:
    """Live engine: owns the device model (bf16 non-expert + INT4 draft experts resident),
    the pinned host expert store, the capped HBM slot pool and the device cache controller."""

    def __init__(self, model: ModelConfig, kmax: int = 16, device: int = 0,
                 host_store_path: str | None = None, host_store_role: int = 0,
                 slot_extra: int = 0, trace_level: int = 1, log_cap: int = 0,
                 expert_codec: str = "xc", max_streams: int = 1):
        self.model = model
        self._desc = model.desc()
        self._path = (host_store_path or "").encode()
        if expert_codec not in ("none", "xc"):
            raise ValueError("expert_codec must be 'none' or 'xc'")
        self._opts = _lib.EngineOpts(device, kmax, self._path, host_store_role, slot_extra,
                                     log_cap, trace_level, 1 if expert_codec == "xc" else 0, max_streams)
        self._h = ctypes.c_void_p()
        check(lib().mspq_engine_create(ctypes.byref(self._desc), ctypes.byref(self._opts),
                                       ctypes.byref(self._h)))

    def configure(self, config: dict):
        """Expert-cache budget / policy / governor (reference run-config schema)."""
        check(lib().mspq_engine_configure(self._h, _cfg_json(config)))

    def generate(self, prompt, max_new_tokens: int) -> dict:
        arr = (ctypes.c_int32 * len(prompt))(*prompt)
        out = ctypes.c_void_p()
        check(lib().mspq_generate(self._h, arr, len(prompt), max_new_tokens, ctypes.byref(out)))
        return json.loads(take_string(out))

    def generate_batch(self, prompts, max_new_tokens: int) -> dict:
        """Several independent request streams decoded together (mspq_generate_batch): one
        layer-major verify pass per cycle over every stream's window, sharing the expert weight
        reads; each stream's tokens equal its own greedy decode."""
        flat = [t for p in prompts for t in p]
        arr = (ctypes.c_int32 * len(flat))(*flat)
        lens = (ctypes.c_int32 * len(prompts))(*[len(p) for p in prompts])
        out = ctypes.c_void_p()
        check(lib().mspq_generate_batch(self._h, arr, lens, len(prompts), max_new_tokens, ctypes.byref(out)))
        return json.loads(take_string(out))

    def info(self) -> dict:
        out = ctypes.c_void_p()
        check(lib().mspq_engine_info(self._h, ctypes.byref(out)))
        return json.loads(take_string(out))

    def read(self, name: str, nbytes: int):
        buf = (ctypes.c_uint8 * nbytes)()
        check(lib().mspq_engine_read(self._h, name.encode(), buf, nbytes))
        return bytes(buf)

    # ---- peer-expert tier (include/mspq_capi.h (3)): home partitioning by expert id mod G
    def home_create(self, group: int, rank: int) -> bytes:
        """Allocate and fill this engine's HBM home region (experts e with e % group == rank);
        returns the 64-byte CUDA IPC handle other ranks attach with."""
        h = (ctypes.c_uint8 * 64)()
        check(lib().mspq_engine_home_create(self._h, group, rank, h))
        return bytes(h)

    def peer_attach_ipc(self, peer_rank: int, handle: bytes):
        """Map another process's home region (its home_create handle)."""
        buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
        check(lib().mspq_engine_peer_attach_ipc(self._h, peer_rank, buf))

    def peer_attach(self, peer_rank: int, peer: "Engine"):
        """Attach a peer engine of this process (same or another GPU)."""
        check(lib().mspq_engine_peer_attach(self._h, peer_rank, peer._h))

    def close(self):
        if self._h:
            lib().mspq_engine_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def to_reference_trace(report: dict, model: ModelConfig, meta: dict | None = None) -> str:
    """Per-committed-position reference trace (trace.hpp:43-49, JSONL trace.cpp:286-311) from a
    live generate() report recorded with trace_level >= 1.

    Position p's target_sets = the target model's routing when the verify processed token p
    (window slot s of the cycle that committed it, or slot 0 = head of the next cycle for a
    bonus token); draft_sets/gates = the draft's routing of the same token (ELB row s) when the
    draft processed it; acc = the draft's token at p was accepted (bonus tokens: false).
    An accepted token in the unpredicted last window slot was never routed by the draft; its
    draft_sets are taken from its target routing and its position listed in
    meta["draft_from_target"].  The last committed token (never verified) ends the trace.
    Feeding the result to
    run_simulation / classify_fidelity / layer_entropy analyses a live run with the
    reference's own tools."""
    L, K = model.L, model.K
    recs = []  # (target_sets, draft_sets, gates, acc)
    synth = []
    cyc = report["cycles"]
    for ci, c in enumerate(cyc):
        if "target" not in c:
            raise ValueError("report needs trace_level >= 1")
        k = c["k"]
        # slot 0 = head: the previous cycle's bonus token (or the last prompt token)
        if ci > 0:
            recs.append((c["target"][0], c["elb"][0], c["elb_gates"][0], False))
        for s in range(1, c["accepted"] + 1):
            if s >= k:  # accepted token in the unpredicted last slot: no draft routing
                synth.append(len(recs))
                recs.append((c["target"][s], c["target"][s], None, True))
            else:
                recs.append((c["target"][s], c["elb"][s], c["elb_gates"][s], True))
    meta = dict(meta or {})
    meta["draft_from_target"] = ",".join(map(str, synth))
    return _emit_trace(recs, model, meta)


def _emit_trace(recs, model, meta):
    head = {"shape": {"L": model.L, "N": model.E, "top_k": model.K, "shared": 0,
                      "expert_bytes": model.expert_bytes_bf16()},
            "meta": dict({"source": "mspq-live"}, **(meta or {}))}
    out = [json.dumps(head, separators=(",", ":"))]
    # gates must be on every record or none (trace.cpp parse): fall back to 1.0 for synthesized
    for p, (tg, dr, gt, acc) in enumerate(recs):
        gates = gt if gt is not None else [[1.0] * model.K for _ in range(model.L)]
        out.append(json.dumps({"pos": p, "target": [[l, tg[l]] for l in range(model.L)],
                               "draft": [[l, dr[l]] for l in range(model.L)],
                               "gates": [[l, gates[l]] for l in range(model.L)], "acc": acc},
                              separators=(",", ":")))
    return "\n".join(out) + "\n"
