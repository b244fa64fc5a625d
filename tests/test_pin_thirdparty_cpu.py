"""Pin the model-math oracle to independent implementations already in the image (CPU).

The reference has no model, so oracle/model.py + oracle/csrc/*.c define the decode
math.  Here that definition is checked against third-party code that was written without it:

  * transformers 5.5 MixtralSparseMoeBlock (MixtralTopKRouter: softmax -> top-k -> renormalise;
    MixtralExperts: SiLU(gate) * up -> down) and Qwen3MoeSparseMoeBlock (norm_topk_prob), run in
    fp32 on the oracle's own bf16 weights and normalised inputs: expert ids equal wherever the
    router's top-K boundary margin exceeds 1e-5, routing weights to 1e-6, the MoE output within
    5e-3 of its scale (the oracle rounds the SiLU*up activation to bf16, as the device does: up to
    2^-9 relative per element, which transformers' fp32 path does not);
  * transformers MixtralRMSNorm against the oracle's fixed-order RMSNorm (bf16 output);
  * GPTQ's symmetric quantizer as published (Frantar et al. 2022, the reference code's
    Quantizer.find_params/quantize with sym=True, bits=4: xmax = max(|xmin|, xmax), scale =
    2 xmax / 15, zero = 8, q = clamp(round(w / scale) + zero, 0, 15)), restated in torch: the
    oracle's INT4 draft is round-to-nearest on exactly that grid per 128-column group, with the
    scale rounded to bf16 (the device stores bf16 scales);
  * vLLM 0.22's GPTQ packing (pack_quantized_values_into_int32 along the input dimension) equals
    the oracle's nibble order (model.py pack_int4), so a GPTQ checkpoint's qweight maps onto it.
"""
import numpy as np
import pytest
import torch

from oracle import model as om


def _moe_inputs(desc, M=24, seed=5):
    rng = np.random.default_rng(seed)
    model = om.Model(desc, fast=False)
    h = (rng.standard_normal((M, desc.d)) * 0.7).astype(np.float32)
    xn = np.stack([model.rmsnorm(np.ascontiguousarray(h[i]), model.gamma(0)) for i in range(M)])
    return model, h, xn


def _fill_experts(experts, model, desc, layer):
    with torch.no_grad():
        for e in range(desc.E):
            g, u, dn = model.expert(layer, e)
            gu = np.concatenate([om.bf16_to_f32(g), om.bf16_to_f32(u)], axis=0)
            experts.gate_up_proj[e].copy_(torch.from_numpy(gu))
            experts.down_proj[e].copy_(torch.from_numpy(om.bf16_to_f32(dn)))


def _oracle_moe(model, xn, layer):
    desc = model.m
    ids, wts, ys, margins = [], [], [], []
    for i in range(xn.shape[0]):
        r_ids, r_w, logits = model.route(xn[i], layer)
        srt = np.sort(logits)[::-1]
        margins.append(min(srt[j] - srt[j + 1] for j in range(desc.K)))
        acc = np.zeros(desc.d, dtype=np.float32)
        for j in range(desc.K):
            y, _ = model.ffn(xn[i], layer, int(r_ids[j]), draft=False)
            acc = (acc + np.float32(r_w[j]) * y).astype(np.float32)
        ids.append(r_ids.tolist())
        wts.append(r_w)
        ys.append(acc)
    return ids, np.array(wts), np.stack(ys), np.array(margins)


def _compare(block, model, xn, layer):
    desc = model.m
    ids, wts, ys, margins = _oracle_moe(model, xn, layer)
    x = torch.from_numpy(om.bf16_to_f32(xn))
    with torch.no_grad():
        _, hf_w, hf_ids = block.gate(x)
        hf_y = block(x[None]).reshape(xn.shape[0], desc.d).numpy()
    checked = 0
    for i in range(xn.shape[0]):
        if margins[i] <= 1e-5:
            continue
        checked += 1
        assert hf_ids[i].tolist() == ids[i], (i, hf_ids[i].tolist(), ids[i])
        assert np.allclose(hf_w[i].numpy(), wts[i], atol=1e-6)
        err = np.abs(hf_y[i] - ys[i]).max() / (np.abs(hf_y[i]).max() + 1e-30)
        assert err <= 5e-3, (i, err)
    assert checked >= xn.shape[0] - 2


def test_routing_and_experts_match_transformers_mixtral_block():
    from transformers import MixtralConfig
    from transformers.models.mixtral.modeling_mixtral import MixtralSparseMoeBlock
    desc = om.ModelDesc(L=2, E=8, K=2, d=256, f=512, V=64, moe_scale=1.0)
    model, _, xn = _moe_inputs(desc)
    cfg = MixtralConfig(hidden_size=desc.d, intermediate_size=desc.f, num_local_experts=desc.E,
                        num_experts_per_tok=desc.K, hidden_act="silu")
    block = MixtralSparseMoeBlock(cfg).float().eval()
    with torch.no_grad():
        block.gate.weight.copy_(torch.from_numpy(om.bf16_to_f32(model.router(1))))
    _fill_experts(block.experts, model, desc, 1)
    _compare(block, model, xn, 1)


def test_routing_and_experts_match_transformers_qwen3_moe_block():
    from transformers import Qwen3MoeConfig
    from transformers.models.qwen3_moe.modeling_qwen3_moe import Qwen3MoeSparseMoeBlock
    desc = om.ModelDesc(L=1, E=32, K=8, d=128, f=128, V=64, moe_scale=1.0)
    model, _, xn = _moe_inputs(desc, M=16)
    cfg = Qwen3MoeConfig(hidden_size=desc.d, moe_intermediate_size=desc.f, num_experts=desc.E,
                         num_experts_per_tok=desc.K, norm_topk_prob=True, hidden_act="silu")
    block = Qwen3MoeSparseMoeBlock(cfg).float().eval()
    with torch.no_grad():
        block.gate.weight.copy_(torch.from_numpy(om.bf16_to_f32(model.router(0))))
    _fill_experts(block.experts, model, desc, 0)
    _compare(block, model, xn, 0)


def test_rmsnorm_matches_transformers():
    from transformers.models.mixtral.modeling_mixtral import MixtralRMSNorm
    desc = om.ModelDesc(L=1, E=4, K=2, d=512, f=128, V=64)
    model = om.Model(desc, fast=False)
    norm = MixtralRMSNorm(desc.d, eps=desc.eps).float()
    with torch.no_grad():
        norm.weight.copy_(torch.from_numpy(om.bf16_to_f32(model.gamma(0))))
    h = (np.random.default_rng(1).standard_normal((8, desc.d)) * 3).astype(np.float32)
    want = norm(torch.from_numpy(h)).detach().numpy()
    for i in range(8):
        got = om.bf16_to_f32(model.rmsnorm(h[i], model.gamma(0)))
        assert np.abs(got - want[i]).max() <= 2 ** -8 * np.abs(want[i]).max()


def _gptq_sym_quantize(w, group=128, bits=4):
    """GPTQ's Quantizer (find_params + quantize, sym=True) per group of 128 input columns, with
    the bf16 scale storage of this engine."""
    maxq = 2 ** bits - 1
    rows, cols = w.shape
    x = w.reshape(rows, cols // group, group)
    xmin = torch.minimum(x.min(dim=2).values, torch.zeros(1))
    xmax = torch.maximum(x.max(dim=2).values, torch.zeros(1))
    xmax = torch.maximum(xmin.abs(), xmax)
    tmp = xmin < 0
    xmin = torch.where(tmp, -xmax, xmin)
    zero_range = (xmin == 0) & (xmax == 0)
    xmin = torch.where(zero_range, torch.full_like(xmin, -1.0), xmin)
    xmax = torch.where(zero_range, torch.full_like(xmax, 1.0), xmax)
    scale = ((xmax - xmin) / maxq).to(torch.bfloat16).float()
    zero = torch.full_like(scale, (maxq + 1) / 2)
    q = torch.clamp(torch.round(x / scale[:, :, None]) + zero[:, :, None], 0, maxq)
    return q.reshape(rows, cols).to(torch.uint8), scale


def test_int4_draft_is_gptq_symmetric_rtn():
    desc = om.ModelDesc(L=1, E=2, K=1, d=512, f=256, V=64)
    w = om.gen(desc.seed, om.t_expert(0, 1, 0), desc.f, desc.d, desc.a_up())
    q, s = om.quantize(w)
    wq = torch.from_numpy(om.bf16_to_f32(w).copy())
    gq, gs = _gptq_sym_quantize(wq)
    # the scale: bf16(2 amax / 15) (model.py writes amax / 7.5, the same number)
    assert np.array_equal(om.bf16_to_f32(s), gs.numpy())
    assert np.array_equal(q, gq.numpy())
    # an all-zero group: GPTQ widens the range to [-1, 1]; the engine keeps scale 1 and q = 8
    z = np.zeros((2, 128), dtype=np.uint16)
    qz, _ = om.quantize(z)
    gz, _ = _gptq_sym_quantize(torch.zeros(2, 128))
    assert np.array_equal(qz, gz.numpy())


def test_int4_packing_matches_vllm_gptq_packing():
    qu = pytest.importorskip("vllm.model_executor.layers.quantization.utils.quant_utils")
    from vllm.scalar_type import scalar_types
    rng = np.random.default_rng(2)
    q = rng.integers(0, 16, size=(64, 256), dtype=np.uint8)  # [rows = out, cols = in]
    ours = om.pack_int4(q)  # [out, in/8], nibble n of word w = input column 8w+n
    # vLLM/GPTQ qweight is [in/8, out] packed along the input dimension (packed_dim 0)
    theirs = qu.pack_quantized_values_into_int32(torch.from_numpy(q.T.astype(np.int32)), scalar_types.uint4b8,
                                                 packed_dim=0)
    assert np.array_equal(ours.T.view(np.int32), theirs.numpy())
