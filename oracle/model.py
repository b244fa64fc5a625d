"""TEST INFRASTRUCTURE ONLY — numpy restatement of the MoE-SpeQ decode math.

"Parity unpinned by the reference": /root/reference has no model, weights, gating, GEMMs or
logits.  This file *defines* the numerics the device must reproduce, from the
paper: bf16 router / norms / non-expert params, INT4 symmetric group-128
draft experts (round-to-nearest on GPTQ's symmetric grid, scale = 2*amax/15,
zero = 8 -- not Hessian-based GPTQ; pinned in tests/test_pin_thirdparty_cpu.py), greedy
verification = accepted prefix + one target token, reordered grouped verify
(PAPER.md:495-496).  Order-sensitive fp32 pieces (fixed-order dots, RMSNorm sums, the exp used
by softmax/SiLU) are in csrc/model_ref.c so they are bit-identical to the kernels; expert FFN
dot products are computed here in float64 (the device result must lie within tolerance).

Weights come from a counter-based hash, so any single tensor can be regenerated on the CPU
without materialising the model.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "libmspq_oracle.so")
_SRCS = [os.path.join(_HERE, "csrc", "model_ref.c"), os.path.join(_HERE, "csrc", "decode_ref.c")]
_lib = None


def build():
    os.makedirs(os.path.join(_HERE, "_build"), exist_ok=True)
    if (not os.path.exists(_SO)) or any(os.path.getmtime(_SO) < os.path.getmtime(s) for s in _SRCS):
        import subprocess
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-o", _SO]
                              + _SRCS + ["-lm"])


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        L.orc_warp_dot.restype = ctypes.c_float
        L.orc_warp_dot.argtypes = [P, P, ctypes.c_int]
        L.orc_sumsq_cta.restype = ctypes.c_float
        L.orc_sumsq_cta.argtypes = [P, ctypes.c_int]
        L.orc_rmsnorm.argtypes = [P, P, ctypes.c_int, ctypes.c_float, P]
        L.orc_det_exp.restype = ctypes.c_float
        L.orc_det_exp.argtypes = [ctypes.c_float]
        L.orc_router_topk.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P]
        L.orc_lm_head.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P]
        L.orc_act.argtypes = [P, P, ctypes.c_int, P]
        L.orc_gen_bf16.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_float, P]
        L.orc_expert_ffn.restype = ctypes.c_int
        L.orc_expert_ffn.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_float, ctypes.c_float, ctypes.c_int, ctypes.c_int, P, P, P]
        L.orc_weight_row.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_float,
                                     ctypes.c_int, P]
        L.orc_lm_head_mt.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P]
        L.orc_gen_rows_mt.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                      ctypes.c_float, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------------- bf16 helpers
def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


# ----------------------------------------------------------------------------- counter RNG
M64 = (1 << 64) - 1
GOLD = 0x9E3779B97F4A7C15
STEP = 0xD1B54A32D192ED03


def _mix_py(z: int) -> int:
    z = (z + GOLD) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _mix_np(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(GOLD)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def tensor_key(seed: int, tensor: int) -> int:
    return _mix_py((seed ^ _mix_py(tensor)) & M64)


def uniform(seed: int, tensor: int, n: int, start: int = 0) -> np.ndarray:
    """val(idx) in (-1, 1), exact in fp32: ((u>>40) - 2^23 + 0.5) * 2^-23."""
    key = np.uint64(tensor_key(seed, tensor))
    idx = np.arange(start, start + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _mix_np(key + idx * np.uint64(STEP))
    hi = (z >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return ((hi.astype(np.float32) + np.float32(0.5)) * np.float32(1.0 / 8388608.0)).astype(np.float32)


# tensor ids
T_EMBED, T_POS, T_LM, T_FINAL_GAMMA = 1, 2, 3, 4


def t_gamma(l):
    return 0x100 + l * 16


def t_router(l):
    return 0x100 + l * 16 + 1


def t_expert(l, e, m):
    return 0x1000000 + ((l * 1024 + e) * 4 + m)


def gen_np(seed, tensor, rows, cols, scale) -> np.ndarray:
    v = uniform(seed, tensor, rows * cols)
    return f32_to_bf16(v * np.float32(scale)).reshape(rows, cols)


def gen(seed, tensor, rows, cols, scale) -> np.ndarray:
    """bf16 [rows, cols] = gen_np (the pinned numpy definition) via its C restatement."""
    out = np.empty(rows * cols, dtype=np.uint16)
    lib().orc_gen_bf16(tensor_key(seed, tensor), 0, rows * cols, ctypes.c_float(np.float32(scale)), _p(out))
    return out.reshape(rows, cols)


def gen_gamma(seed, tensor, d) -> np.ndarray:
    v = uniform(seed, tensor, d)
    return f32_to_bf16(np.float32(1.0) + v * np.float32(0.125))


# ----------------------------------------------------------------------------- INT4 (GPTQ sym)
def quantize(w_bf16: np.ndarray, group: int = 128):
    """Per row, per 128-column group: scale = bf16(amax / 7.5), q = clamp(rint(w/scale)+8, 0, 15)."""
    w = bf16_to_f32(w_bf16).reshape(w_bf16.shape[0], -1, group)
    amax = np.abs(w).max(axis=2)
    s32 = (amax / np.float32(7.5)).astype(np.float32)
    sb = f32_to_bf16(s32)
    sf = bf16_to_f32(sb)
    sf_safe = np.where(sf == 0, np.float32(1.0), sf).astype(np.float32)
    q = np.rint((w / sf_safe[:, :, None]).astype(np.float32)) + np.float32(8)
    q = np.clip(q, 0, 15).astype(np.uint8).reshape(w_bf16.shape)
    sb = np.where(sf == 0, f32_to_bf16(np.ones_like(sf)), sb)
    return q, sb


def dequantize(q: np.ndarray, sb: np.ndarray, group: int = 128) -> np.ndarray:
    rows, cols = q.shape
    s = bf16_to_f32(sb)
    return ((q.astype(np.float32) - np.float32(8)).reshape(rows, -1, group) * s[:, :, None]).reshape(rows, cols)


def pack_int4(q: np.ndarray) -> np.ndarray:
    """[rows, cols] nibbles -> [rows, cols/8] uint32, nibble n of word w = column 8w+n."""
    rows, cols = q.shape
    q = q.astype(np.uint32).reshape(rows, cols // 8, 8)
    out = np.zeros((rows, cols // 8), dtype=np.uint32)
    for n in range(8):
        out |= q[:, :, n] << np.uint32(4 * n)
    return out


# ----------------------------------------------------------------------------- model
@dataclass
class ModelDesc:
    L: int
    E: int
    K: int
    d: int
    f: int
    V: int
    P: int = 4096          # positional table rows
    seed: int = 1234
    embed_scale: float = 1.0
    pos_scale: float = 0.5
    router_scale: float = 3.0
    moe_scale: float = 0.06
    lm_scale: float = 1.0
    eps: float = 1e-6
    H: int = 0             # attention query heads (0 = attention-free layers)
    Hkv: int = 0           # KV heads (grouped-query attention)
    Dh: int = 0            # head dim

    # scales passed to the device as fp32 (computed once, identically on both sides)
    def a_qkv(self):
        return float(np.float32(math.sqrt(3.0 / self.d)))

    def a_o(self):
        return float(np.float32(self.moe_scale * math.sqrt(3.0 / max(1, self.H * self.Dh))))

    def a_router(self):
        return float(np.float32(self.router_scale * math.sqrt(3.0 / self.d)))

    def a_up(self):
        return float(np.float32(math.sqrt(3.0 / self.d)))

    def a_down(self):
        return float(np.float32(self.moe_scale * math.sqrt(3.0 / self.f)))

    def a_lm(self):
        return float(np.float32(self.lm_scale * math.sqrt(3.0 / self.d)))

    def expert_bytes_bf16(self):
        return 3 * self.d * self.f * 2

    def expert_bytes_int4(self):
        return 3 * self.d * self.f // 2 + 3 * self.d * self.f // 128 * 2


CONFIGS = {
    # BASELINE.json configs (ffn for tiny chosen: 512; Qwen3 moe_intermediate 768); attention heads
    # of the named models (Phi-3.5-MoE / Mixtral-8x7B: 32 q, 8 kv, dim 128; Qwen3-30B-A3B: 32 q,
    # 4 kv, dim 128; tiny chosen: 4 q, 2 kv, dim 64)
    "tiny": dict(L=4, E=8, K=2, d=256, f=512, V=512, H=4, Hkv=2, Dh=64),
    "mixtral": dict(L=32, E=8, K=2, d=4096, f=14336, V=32000, H=32, Hkv=8, Dh=128),
    "phi": dict(L=32, E=16, K=2, d=4096, f=6400, V=32064, H=32, Hkv=8, Dh=128),
    "qwen3": dict(L=48, E=128, K=8, d=2048, f=768, V=151936, H=32, Hkv=4, Dh=128),
}


def t_attn(l, m):
    """attention tensors of layer l: 0 = Wqkv [(H+2Hkv)Dh][d], 1 = Wo [d][H Dh], 2 = RMSNorm gamma"""
    return 0x800000 + l * 16 + m


class Model:
    """CPU model: weights regenerated lazily from the counter hash.  With `fast` (default for
    full-width experts) the expert FFN and LM head run in csrc/decode_ref.c over all host cores,
    generating each expert's rows on the fly instead of caching fp32 matrices."""

    def __init__(self, desc: ModelDesc, fast: bool | None = None):
        self.m = desc
        self._cache = {}
        self.fast = (desc.d * desc.f >= 1 << 22) if fast is None else fast
        # the shared KV cache (draft and target write the same rows; rollback = later windows
        # overwrite): kv[l][pos] = (k [Hkv, Dh], v [Hkv, Dh]) fp32 holding bf16 values
        self.kv = [dict() for _ in range(desc.L)]

    def _get(self, key, fn):
        if key not in self._cache:
            self._cache[key] = fn()
        return self._cache[key]

    def embed_row(self, tok):
        m = self.m
        return self._get(("emb", tok), lambda: f32_to_bf16(
            uniform(m.seed, T_EMBED, m.d, start=tok * m.d) * np.float32(m.embed_scale)))

    def pos_row(self, p):
        m = self.m
        return self._get(("pos", p), lambda: f32_to_bf16(
            uniform(m.seed, T_POS, m.d, start=p * m.d) * np.float32(m.pos_scale)))

    def gamma(self, l):
        m = self.m
        t = T_FINAL_GAMMA if l < 0 else t_gamma(l)
        return self._get(("gamma", l), lambda: gen_gamma(m.seed, t, m.d))

    def router(self, l):
        m = self.m
        return self._get(("router", l), lambda: gen(m.seed, t_router(l), m.E, m.d, m.a_router()))

    def lm(self):
        m = self.m
        if self.fast:
            def mk():
                out = np.empty((m.V, m.d), dtype=np.uint16)
                lib().orc_gen_rows_mt(tensor_key(m.seed, T_LM), 0, m.V, m.d, ctypes.c_float(np.float32(m.a_lm())),
                                      _p(out))
                return out
            return self._get("lm", mk)
        return self._get("lm", lambda: gen(m.seed, T_LM, m.V, m.d, m.a_lm()))

    def _gen_mt(self, tensor, rows, cols, scale):
        out = np.empty((rows, cols), dtype=np.uint16)
        lib().orc_gen_rows_mt(tensor_key(self.m.seed, tensor), 0, rows, cols, ctypes.c_float(np.float32(scale)),
                              _p(out))
        return out

    def attn_weights(self, l):
        """(Wqkv fp64 [(H+2Hkv)Dh, d], Wo fp64 [d, H Dh], gamma bf16); cached unless fast."""
        m = self.m
        nq, nkv = m.H * m.Dh, m.Hkv * m.Dh

        def mk():
            wqkv = self._gen_mt(t_attn(l, 0), nq + 2 * nkv, m.d, m.a_qkv())
            wo = self._gen_mt(t_attn(l, 1), m.d, nq, m.a_o())
            return (bf16_to_f32(wqkv).astype(np.float64), bf16_to_f32(wo).astype(np.float64),
                    gen_gamma(m.seed, t_attn(l, 2), m.d))
        if self.fast:
            return mk()
        return self._get(("attn", l), mk)

    def attention(self, h, l, positions, draft_cache=True, ctx=None):
        """Attention block of layer l for the window rows h [M, d] at consecutive positions:
        RMSNorm -> QKV (double) -> the window's K/V rounded to bf16 and written to the shared cache
        -> causal attention over the cache rows before the window (ctx(j) or self.kv) and the
        window's own rows -> O projection.  Returns the [M, d] fp32 residual update."""
        m = self.m
        M = h.shape[0]
        nq, nkv, G = m.H * m.Dh, m.Hkv * m.Dh, m.H // m.Hkv
        wqkv, wo, ga = self.attn_weights(l)
        xa = np.stack([bf16_to_f32(self.rmsnorm(np.ascontiguousarray(h[i]), ga)) for i in range(M)]).astype(np.float64)
        qkv = (xa @ wqkv.T).astype(np.float32)
        q = qkv[:, :nq].reshape(M, m.H, m.Dh).astype(np.float64)
        k_new = bf16_to_f32(f32_to_bf16(qkv[:, nq:nq + nkv])).reshape(M, m.Hkv, m.Dh)
        v_new = bf16_to_f32(f32_to_bf16(qkv[:, nq + nkv:])).reshape(M, m.Hkv, m.Dh)
        p0 = positions[0]
        for i in range(M):
            self.kv[l][p0 + i] = (k_new[i], v_new[i])
        if p0 > 0:
            rows = [ctx(j) if ctx is not None else self.kv[l][j] for j in range(p0)]
            kc = np.stack([r[0] for r in rows]).astype(np.float64)
            vc = np.stack([r[1] for r in rows]).astype(np.float64)
        else:
            kc = np.zeros((0, m.Hkv, m.Dh))
            vc = np.zeros((0, m.Hkv, m.Dh))
        out = np.empty((M, nq), dtype=np.float64)
        scale = 1.0 / math.sqrt(m.Dh)
        for i in range(M):
            keys = np.concatenate([kc, k_new[:i + 1].astype(np.float64)])      # [n, Hkv, Dh]
            vals = np.concatenate([vc, v_new[:i + 1].astype(np.float64)])
            for hh in range(m.H):
                g = hh // G
                sc = keys[:, g, :] @ q[i, hh] * scale
                pr = np.exp(sc - sc.max())
                out[i, hh * m.Dh:(hh + 1) * m.Dh] = (pr @ vals[:, g, :]) / pr.sum()
        o = bf16_to_f32(f32_to_bf16(out.astype(np.float32))).astype(np.float64)
        return (o @ wo.T).astype(np.float32)

    def expert(self, l, e):
        """bf16 (gate [f,d], up [f,d], down [d,f])."""
        m = self.m
        return self._get(("x", l, e), lambda: (
            gen(m.seed, t_expert(l, e, 0), m.f, m.d, m.a_up()),
            gen(m.seed, t_expert(l, e, 1), m.f, m.d, m.a_up()),
            gen(m.seed, t_expert(l, e, 2), m.d, m.f, m.a_down())))

    def expert_q(self, l, e):
        """INT4 (q, scales) for gate, up, down."""
        def mk():
            g, u, dn = self.expert(l, e)
            return quantize(g), quantize(u), quantize(dn)
        return self._get(("q", l, e), mk)

    # -- pieces -----------------------------------------------------------------------------
    def rmsnorm(self, h, gamma):
        out = np.empty(self.m.d, dtype=np.uint16)
        lib().orc_rmsnorm(_p(h), _p(gamma), self.m.d, ctypes.c_float(self.m.eps), _p(out))
        return out

    def route(self, xn, l):
        m = self.m
        logits = np.empty(m.E, dtype=np.float32)
        ids = np.empty(m.K, dtype=np.int32)
        wts = np.empty(m.K, dtype=np.float32)
        wr = np.ascontiguousarray(self.router(l))
        lib().orc_router_topk(_p(xn), _p(wr), m.E, m.d, m.K, _p(logits), _p(ids), _p(wts))
        return ids, wts, logits

    def ffn_batch(self, xn_rows, l, e, draft: bool, with_act=False):
        """Expert (l, e) on M normed rows [M, d] bf16 -> y [M, d] fp32 (decode_ref.c) (+ the bf16
        SiLU(gate) * up rows [M, f] with `with_act`)."""
        m = self.m
        xn_rows = np.ascontiguousarray(xn_rows, dtype=np.uint16)
        M = xn_rows.shape[0]
        y = np.empty((M, m.d), dtype=np.float32)
        act = np.empty((M, m.f), dtype=np.uint16) if with_act else None
        rc = lib().orc_expert_ffn(m.seed, l, e, m.d, m.f, ctypes.c_float(m.a_up()), ctypes.c_float(m.a_down()),
                                  1 if draft else 0, M, _p(xn_rows), _p(y), _p(act) if with_act else None)
        if rc:
            raise MemoryError("orc_expert_ffn")
        return (y, act) if with_act else y

    def ffn(self, xn, l, e, draft: bool):
        m = self.m
        if self.fast:
            y, a = self.ffn_batch(xn[None, :], l, e, draft, with_act=True)
            return y[0], a[0]
        x = bf16_to_f32(xn)
        G, U, D = self.expert_f32(l, e, draft)
        gv = np.ascontiguousarray(G @ x, dtype=np.float32)
        uv = np.ascontiguousarray(U @ x, dtype=np.float32)
        a = np.empty(m.f, dtype=np.uint16)
        lib().orc_act(_p(gv), _p(uv), m.f, _p(a))
        y = (D @ bf16_to_f32(a)).astype(np.float32)
        return y, a

    def expert_f32(self, l, e, draft):
        """Dequantised (draft) or widened (target) fp32 matrices, cached."""
        def mk():
            if draft:
                (gq, gs), (uq, us), (dq, ds) = self.expert_q(l, e)
                return dequantize(gq, gs), dequantize(uq, us), dequantize(dq, ds)
            g, u, dn = self.expert(l, e)
            return bf16_to_f32(g), bf16_to_f32(u), bf16_to_f32(dn)
        return self._get(("f32", l, e, draft), mk)

    def lm_head(self, xn_rows):
        m = self.m
        T = xn_rows.shape[0]
        logits = np.empty((T, m.V), dtype=np.float32)
        am = np.empty(T, dtype=np.int32)
        lm = np.ascontiguousarray(self.lm())
        fn = lib().orc_lm_head_mt if self.fast else lib().orc_lm_head
        fn(_p(np.ascontiguousarray(xn_rows)), _p(lm), T, m.V, m.d, _p(logits), _p(am))
        return logits, am

    # -- one token ---------------------------------------------------------------------------
    def forward(self, tok, pos, draft: bool):
        """Returns (argmax token, per-layer (ids, wts), final logits)."""
        am, routing, logits = forward_batch(self, [tok], [pos], draft, with_logits=True)[0]
        return am, routing, logits


def forward_batch(model: Model, toks, poss, draft: bool, h_in=None, h_trace=None, with_logits=False,
                  hmid_trace=None):
    """Forward pass of a window of M tokens at consecutive positions poss (layer-major, tokens
    grouped by expert: one weight generation per (layer, expert) in fast mode).  With attention
    (model.m.H > 0) each layer first runs the shared-KV attention block (Model.attention: the
    window's K/V rows are written into the model's cache, draft or target alike).
    Returns [(argmax, routing)] per token (+ logits with `with_logits`).  With `h_in` = {layer:
    [M, d] fp32}, the residual entering that layer is replaced (teacher forcing from the device).
    `h_trace` (a list) receives the [M, d] residual entering each layer and, last, the final
    one; `hmid_trace` the residual after each layer's attention block (what the router sees)."""
    m = model.m
    M = len(toks)
    h = np.stack([(bf16_to_f32(model.embed_row(t)) + bf16_to_f32(model.pos_row(p))).astype(np.float32)
                  for t, p in zip(toks, poss)])
    routing = [[] for _ in range(M)]
    for l in range(m.L):
        if h_in is not None and l in h_in:
            h = np.asarray(h_in[l], dtype=np.float32).copy()
        if h_trace is not None:
            h_trace.append(h.copy())
        if m.H > 0:
            h = (h + model.attention(h, l, poss)).astype(np.float32)
        if hmid_trace is not None:
            hmid_trace.append(h.copy())
        xn = np.stack([model.rmsnorm(np.ascontiguousarray(h[i]), model.gamma(l)) for i in range(M)])
        rt = [model.route(xn[i], l) for i in range(M)]
        for i in range(M):
            routing[i].append((rt[i][0].copy(), rt[i][1].copy()))
        ys = {}
        for e in sorted({int(x) for i in range(M) for x in rt[i][0]}):
            rows = [i for i in range(M) if e in rt[i][0].tolist()]
            if model.fast:
                yb = model.ffn_batch(xn[rows], l, e, draft)
            else:
                yb = np.stack([model.ffn(xn[i], l, e, draft)[0] for i in rows])
            for j, i in enumerate(rows):
                ys[(i, e)] = yb[j]
        for i in range(M):
            acc = np.zeros(m.d, dtype=np.float32)
            for j in range(m.K):
                e = int(rt[i][0][j])
                acc = (acc + (np.float32(rt[i][1][j]) * ys[(i, e)]).astype(np.float32)).astype(np.float32)
            h[i] = (h[i] + acc).astype(np.float32)
    if h_trace is not None:
        h_trace.append(h.copy())
    xf = np.stack([model.rmsnorm(np.ascontiguousarray(h[i]), model.gamma(-1)) for i in range(M)])
    lg, am = model.lm_head(xf)
    if with_logits:
        return [(int(am[i]), routing[i], lg[i]) for i in range(M)]
    return [(int(am[i]), routing[i]) for i in range(M)]


def prefill(model: Model, prompt, chunk=32):
    """The engine's prefill (live.cpp): the target runs the prompt's tokens 0..n-2 (their KV rows)
    in windows of up to `chunk` tokens (32, the engine's prefill window).  Returns the windows' target routing
    [[slot][layer] (ids, wts)] per window (for the control-plane replay)."""
    out = []
    n = len(prompt) - 1
    for s0 in range(0, n, chunk):
        toks = prompt[s0:min(n, s0 + chunk)]
        res = forward_batch(model, toks, list(range(s0, s0 + len(toks))), draft=False)
        out.append([r[1] for r in res])
    return out


def check_layers(model: Model, h_caps, ids, draft: bool, tol=2e-3, h_mids=None, positions=None, ctx=None):
    """Teacher-forced per-layer check of a device pass over M tokens.  h_caps [L+1][M][d] = the
    device residual entering each layer (index L = the final residual); ids [L][M][K] = the
    device's routing.  For every layer: routing from the device's own h must be bit-exact, and
    h + sum_j w_j FFN_j(xn) must equal the device's next residual within
    tol * max|h| (accumulation order only).  Returns (worst relative error, margins[L][M] = the
    router's logit gap at the top-K boundary relative to the largest |logit|) for near-tie reporting; raises AssertionError on a
    mismatch.  With attention, h_mids [L][M][d] = the device residual after each layer's attention
    block, positions = the window's positions and ctx(l, j) -> (k, v) the device KV rows before
    the window: the attention block is checked first (h_caps[l] + attn == h_mids[l] within tol),
    then routing and the MoE from h_mids[l]."""
    m = model.m
    M = h_caps.shape[1]
    worst = 0.0
    margins = [[float("inf")] * M for _ in range(m.L)]
    for l in range(m.L):
        h = np.ascontiguousarray(h_caps[l], dtype=np.float32)
        if m.H > 0:
            att = h + model.attention(h, l, positions, ctx=(lambda j, l=l: ctx(l, j)))
            dev_mid = np.asarray(h_mids[l], dtype=np.float32)
            err = float(np.abs(att - dev_mid).max()) / (float(np.abs(dev_mid).max()) + 1e-6)
            worst = max(worst, err)
            assert err <= tol, ("attention output", l, err)
            h = np.ascontiguousarray(dev_mid)
        xn = np.stack([model.rmsnorm(np.ascontiguousarray(h[i]), model.gamma(l)) for i in range(M)])
        rt = [model.route(xn[i], l) for i in range(M)]
        for i in range(M):
            assert rt[i][0].tolist() == list(ids[l][i]), ("routing", l, i, rt[i][0].tolist(), list(ids[l][i]))
            lg = np.sort(rt[i][2])[::-1]
            gaps = [lg[j] - lg[j + 1] for j in range(min(m.K, m.E - 1))]  # order inside the top-K counts too
            if gaps:
                margins[l][i] = float(min(gaps)) / (float(np.abs(lg).max()) + 1e-30)
        nxt = h.copy()
        for e in sorted({int(x) for i in range(M) for x in rt[i][0]}):
            rows = [i for i in range(M) if e in rt[i][0].tolist()]
            yb = model.ffn_batch(xn[rows], l, e, draft) if model.fast else \
                np.stack([model.ffn(xn[i], l, e, draft)[0] for i in rows])
            for j, i in enumerate(rows):
                w = float(rt[i][1][list(rt[i][0]).index(e)])
                nxt[i] += np.float32(w) * yb[j]
        dev = np.asarray(h_caps[l + 1], dtype=np.float32)
        scale = float(np.abs(dev).max()) + 1e-6
        err = float(np.abs(nxt - dev).max()) / scale
        worst = max(worst, err)
        assert err <= tol, ("layer output", l, err)
    return worst, margins


def speculative_decode(model: Model, last_token: int, start_pos: int, ks, max_new: int, prompt=None, chunk=32,
                       deadline=None, prefilled=False):
    """Greedy speculative decoding with the INT4 draft: each cycle drafts k
    tokens from the head (previous bonus), verifies the k+1-slot window with the bf16 target
    (slot i target argmax predicts slot i+1), accepts the longest matching prefix plus the
    target's token at the first mismatch.  Yields per-cycle records; `ks` supplies k per cycle
    (the governor's choice is a host-timing decision, so the oracle consumes it).  With attention
    the prompt is prefilled first (`prompt`, windows of `chunk` tokens).  `deadline`
    (time.perf_counter() value, bench CPU baseline) stops after the cycle that passes it;
    `prefilled`: the model's KV cache already holds the prompt (prefill not repeated)."""
    out, tok, pos, committed = [], last_token, start_pos, 0
    ci = 0
    if model.m.H > 0 and not prefilled:  # attention: fresh shared KV cache, then the prompt's prefill
        assert prompt is not None and prompt[-1] == last_token and len(prompt) - 1 == start_pos
        model.kv = [dict() for _ in range(model.m.L)]
        model.prefill_routing = prefill(model, prompt, chunk)
    while committed < max_new:
        k = min(ks[ci] if ci < len(ks) else ks[-1], max_new - committed)
        k = max(k, 1)
        draft_toks, elb_rows = [], []
        t, p = tok, pos
        for i in range(k):
            nt, routing, _ = model.forward(t, p, draft=True)
            elb_rows.append(routing)
            draft_toks.append(nt)
            t, p = nt, p + 1
        window = [tok] + draft_toks
        res = forward_batch(model, window, [pos + s for s in range(len(window))], draft=False)
        tgt_argmax = [r[0] for r in res]
        tgt_routing = [r[1] for r in res]
        acc = 0
        while acc < k and draft_toks[acc] == tgt_argmax[acc]:
            acc += 1
        bonus = tgt_argmax[acc]
        new = draft_toks[:acc] + [bonus]
        new = new[:max_new - committed]
        out.append(dict(k=k, draft=draft_toks, elb=elb_rows, target=tgt_routing,
                        target_argmax=tgt_argmax, accepted=acc, committed=new))
        committed += len(new)
        pos += acc + 1
        tok = bonus
        ci += 1
        if deadline is not None:
            import time
            if time.perf_counter() >= deadline:
                break
    return out
