"""Thin torch-tensor wrappers over the kernel entry points of the C-ABI (for tests and
benchmarks).  torch is only used for device memory and streams."""
from __future__ import annotations

import torch

from ._lib import check, lib


def _p(t):
    return None if t is None else t.data_ptr()


def _s(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def int4_blob_bytes(d, f):
    return lib().mspq_int4_blob_bytes(d, f)


def bf16_blob_bytes(d, f):
    return lib().mspq_bf16_blob_bytes(d, f)


def fill_bf16(seed, tensor, scale, n, kind=0, start=0, device="cuda"):
    out = torch.empty(n, dtype=torch.int16, device=device)
    check(lib().mspq_fill_bf16(seed, tensor, scale, kind, _p(out), n, start, _s()))
    return out


def fill_expert(seed, layer, expert, d, f, a_up, a_down, device="cuda"):
    out = torch.empty(bf16_blob_bytes(d, f) // 2, dtype=torch.int16, device=device)
    check(lib().mspq_fill_expert(seed, layer, expert, d, f, a_up, a_down, _p(out), _s()))
    return out


def quantize_int4(w_i16, rows, cols):
    q = torch.empty(rows * cols // 8, dtype=torch.int32, device=w_i16.device)
    s = torch.empty(rows * cols // 128, dtype=torch.int16, device=w_i16.device)
    check(lib().mspq_quantize_int4(_p(w_i16), rows, cols, _p(q), _p(s), _s()))
    return q, s


def embed(embed_w, pos_w, tokens, positions, d):
    T = tokens.numel()
    h = torch.empty(T, d, dtype=torch.float32, device=tokens.device)
    check(lib().mspq_embed(_p(embed_w), _p(pos_w), _p(tokens), _p(positions), T, d, _p(h), _s()))
    return h


def gate_topk(h, gamma, router, E, K, eps=1e-6, y=None, entry_of=None, prev_wts=None,
              elb_ids=None, elb_gates=None, elb_row=None, layer=0, L=1, want_logits=True,
              y_splits=1, y_split_stride=0):
    T, d = h.shape
    dev = h.device
    xn = torch.empty(T, d, dtype=torch.int16, device=dev)
    ids = torch.empty(T, K, dtype=torch.int32, device=dev)
    wts = torch.empty(T, K, dtype=torch.float32, device=dev)
    logits = torch.empty(T, E, dtype=torch.float32, device=dev) if want_logits and router is not None else None
    check(lib().mspq_gate_topk(_p(h), _p(y), _p(entry_of), _p(prev_wts), y_splits, y_split_stride,
                               _p(gamma), _p(router),
                               _p(xn), _p(ids), _p(wts), _p(logits), _p(elb_ids), _p(elb_gates),
                               _p(elb_row), None, layer, L, T, d, E, K, eps, _s()))
    return xn, ids, wts, logits


class Schedule:
    def __init__(self, T, K, E, device="cuda"):
        G = min(E, T * K)
        self.T, self.K, self.E, self.G = T, K, E, G
        z = lambda n: torch.zeros(n, dtype=torch.int32, device=device)
        self.n_groups, self.group_expert, self.group_buf = z(1), z(G), z(G)
        self.group_off, self.entry_tok, self.entry_of = z(G + 1), z(T * K), z(T * K)
        self.entry_group = z(T * K)

    def ptrs(self):
        return [_p(self.n_groups), _p(self.group_expert), _p(self.group_buf), _p(self.group_off),
                _p(self.entry_tok), _p(self.entry_of), _p(self.entry_group)]


def build_schedule(ids, E):
    T, K = ids.shape
    s = Schedule(T, K, E, ids.device)
    check(lib().mspq_build_schedule(_p(ids), T, K, E, None, *s.ptrs(), _s()))
    return s


def tile_bf16(src_i16, rows, cols):
    dst = torch.empty(rows * cols, dtype=torch.int16, device=src_i16.device)
    check(lib().mspq_tile_bf16(_p(src_i16), rows, cols, _p(dst), _s()))
    return dst


def moe_bf16_tc(s: Schedule, xn, pool_tiled, blob_bytes, d, f, split1=1, split2=1):
    """K3 on tcgen05; returns y summed over the split planes [T*K][d]."""
    T, K, G = s.T, s.K, s.G
    N = T * K
    ws = torch.empty(lib().mspq_moe_bf16_tc_ws_bytes(d, f, T, K, G, split1), dtype=torch.uint8,
                     device=xn.device)
    y = torch.empty(split2, N, d, dtype=torch.float32, device=xn.device)
    check(lib().mspq_moe_bf16_tc(_p(s.n_groups), _p(s.group_expert), _p(s.group_buf), _p(s.group_off),
                                 _p(s.entry_tok), _p(s.entry_group), _p(xn), _p(pool_tiled), blob_bytes,
                                 d, f, T, K, G, split1, split2, _p(ws), _p(y), _s()))
    return y.sum(0) if split2 > 1 else y[0], y


def tile_int4(q_i32, s_i16, rows, cols):
    tq = torch.empty_like(q_i32)
    ts = torch.empty_like(s_i16)
    check(lib().mspq_tile_int4(_p(q_i32), _p(s_i16), rows, cols, _p(tq), _p(ts), _s()))
    return tq, ts


def moe_int4_tc(s: Schedule, xn, blobs_tiled, blob_bytes, layer, E, d, f, split1=1, split2=1):
    """K2 on tcgen05 over tile-major INT4 blobs; returns y summed over split planes."""
    T, K, G = s.T, s.K, s.G
    N = T * K
    ws = torch.empty(lib().mspq_moe_bf16_tc_ws_bytes(d, f, T, K, G, split1), dtype=torch.uint8,
                     device=xn.device)
    y = torch.empty(split2, N, d, dtype=torch.float32, device=xn.device)
    check(lib().mspq_moe_int4_tc(_p(s.n_groups), _p(s.group_expert), _p(s.group_buf), _p(s.group_off),
                                 _p(s.entry_tok), _p(s.entry_group), _p(xn), _p(blobs_tiled), blob_bytes,
                                 layer, E, d, f, T, K, G, split1, split2, _p(ws), _p(y), _s()))
    return y.sum(0) if split2 > 1 else y[0], y


def lm_head(xn, lm, V):
    T, d = xn.shape
    logits = torch.empty(T, V, dtype=torch.float32, device=xn.device)
    check(lib().mspq_lm_head(_p(xn), _p(lm), T, V, d, _p(logits), _s()))
    return logits


def argmax(logits):
    T, V = logits.shape
    out = torch.empty(T, dtype=torch.int32, device=logits.device)
    check(lib().mspq_argmax(_p(logits), T, V, _p(out), _s()))
    return out


def accept_scan(draft, target_argmax):
    k = draft.numel()
    res = torch.empty(2, dtype=torch.int32, device=draft.device)
    check(lib().mspq_accept_scan(_p(draft), _p(target_argmax), k, _p(res), _s()))
    return res


# ---------------------------------------------------------------- lossless expert codec
def xc_encode(tiles_i16):
    """bf16 tile images (int16 view, n_tiles * 8192 values, device) -> uint8 blob (device)."""
    import ctypes
    n = tiles_i16.numel() // 8192
    scratch = torch.empty(lib().mspq_xc_scratch_bytes(n), dtype=torch.uint8, device=tiles_i16.device)
    out = torch.empty(lib().mspq_xc_max_blob_bytes(n), dtype=torch.uint8, device=tiles_i16.device)
    nb = ctypes.c_longlong(0)
    check(lib().mspq_xc_encode(_p(tiles_i16), n, _p(scratch), _p(out), out.numel(), ctypes.byref(nb), _s()))
    return out[: nb.value].clone()


def xc_decode(blob_u8, n_tiles, tile0=0, tile1=None, dst=None, n_ctas=0):
    tile1 = n_tiles if tile1 is None else tile1
    if dst is None:
        dst = torch.zeros(n_tiles * 8192, dtype=torch.int16, device=blob_u8.device)
    check(lib().mspq_xc_decode(_p(blob_u8), tile0, tile1, _p(dst), n_ctas, _s()))
    return dst
