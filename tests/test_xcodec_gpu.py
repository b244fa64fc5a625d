"""Lossless expert codec (csrc/xcodec.cu): GPU encode -> GPU decode reproduces the bf16 tile
images bit for bit, the blob follows the documented format (an independent CPU decoder,
tests/xcodec_ref.py, reads the same bytes), chunked decodes compose, and adversarial tiles
(zeros, denormals, inf/NaN, incompressible bits) survive via escapes / raw tiles."""
import numpy as np
import pytest
import torch

import xcodec_ref as xr

pytestmark = pytest.mark.gpu


def _tiles_of_expert(d, f, seed=5, layer=1, expert=3):
    from paper_2511_14102_b200 import ops
    blob = ops.fill_expert(seed, layer, expert, d, f, 1.0, 1.0)
    w13 = ops.tile_bf16(blob[: 2 * f * d], 2 * f, d)
    w2 = ops.tile_bf16(blob[2 * f * d:], d, f)
    return torch.cat([w13.view(-1), w2.view(-1)])


def _roundtrip(tiles):
    from paper_2511_14102_b200 import ops
    n = tiles.numel() // 8192
    blob = ops.xc_encode(tiles)
    out = ops.xc_decode(blob, n)
    torch.cuda.synchronize()
    assert torch.equal(out, tiles)
    return blob


@pytest.mark.parametrize("d,f", [(256, 512), (2048, 768), (4096, 6400)])
def test_expert_roundtrip_bit_exact_and_smaller(cuda, d, f):
    tiles = _tiles_of_expert(d, f)
    blob = _roundtrip(tiles)
    ratio = blob.numel() / (tiles.numel() * 2)
    # sign+mantissa byte + ~2 bits of exponent code per value (uniform-init weights)
    assert ratio < 0.70, ratio


def test_gaussian_weights_compress_like_trained_weights(cuda):
    """Exponent entropy of N(0, s^2) bf16 weights is ~2.5 bits: ratio ~0.66-0.68."""
    g = torch.Generator(device="cuda").manual_seed(1)
    w = (torch.randn(64 * 8192, generator=g, device="cuda") * 0.02).to(torch.bfloat16).view(torch.int16)
    blob = _roundtrip(w)
    ratio = blob.numel() / (w.numel() * 2)
    assert 0.6 < ratio < 0.70, ratio


def test_cpu_reference_decoder_reads_gpu_blob(cuda):
    tiles = _tiles_of_expert(256, 512)
    from paper_2511_14102_b200 import ops
    blob = ops.xc_encode(tiles).cpu().numpy()
    n, lens, toff = xr.blob_header(blob)
    assert n == tiles.numel() // 8192 and toff[-1] == blob.size
    want = tiles.cpu().numpy().view(np.uint16).reshape(n, 8192)
    for t in [0, 17, n - 1]:
        assert np.array_equal(xr.decode_tile(blob, t), want[t])


def test_chunked_decode_composes(cuda):
    from paper_2511_14102_b200 import ops
    tiles = _tiles_of_expert(2048, 768)
    n = tiles.numel() // 8192
    blob = ops.xc_encode(tiles)
    dst = torch.zeros_like(tiles)
    for a, b in [(0, 7), (7, 300), (300, n)]:
        ops.xc_decode(blob, n, a, b, dst=dst, n_ctas=3)
    torch.cuda.synchronize()
    assert torch.equal(dst, tiles)


def test_adversarial_tiles(cuda):
    n = 6
    v = torch.zeros(n, 8192, dtype=torch.int32)
    v[1] = torch.randint(0, 65536, (8192,), generator=torch.Generator().manual_seed(2))  # incompressible
    v[2, ::2] = 0x7F80  # +inf
    v[2, 1::2] = 0x0001  # smallest denormal
    v[3] = 0x7FC1  # NaN payload
    v[3, :100] = 0x8000  # -0
    v[4] = torch.randint(0, 65536, (8192,), generator=torch.Generator().manual_seed(3)) & 0x807F  # exp 0
    v[5, :4096] = 0x3F80  # 1.0 next to tiny values: exponent gaps > 15 -> escapes
    v[5, 4096:] = 0x0C00
    tiles = v.numpy().astype(np.uint16).view(np.int16)
    t = torch.from_numpy(tiles.reshape(-1).copy()).cuda()
    blob = _roundtrip(t)
    b = blob.cpu().numpy()
    for i in range(n):
        assert np.array_equal(xr.decode_tile(b, i), tiles[i].view(np.uint16))
