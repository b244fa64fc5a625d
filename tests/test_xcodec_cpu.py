"""The XC blob format on the CPU (no GPU): the CPU restatement of the encoder round-trips through
the independent CPU decoder on Gaussian-like, escape-heavy and incompressible tiles, and the
code lengths are a complete prefix code within the 12-bit table."""
import numpy as np

import xcodec_ref as xr


def _tiles(seed):
    rng = np.random.default_rng(seed)
    g = (rng.standard_normal(8192) * 0.02).astype(np.float32)
    gauss = (g.view(np.uint32) >> 16).astype(np.uint16)                     # bf16 truncation
    esc = np.where(np.arange(8192) % 2 == 0, 0x3F80, 0x0C00).astype(np.uint16)  # exponent gaps > 15
    noise = rng.integers(0, 65536, 8192, dtype=np.uint32).astype(np.uint16)   # incompressible
    zeros = np.zeros(8192, dtype=np.uint16)
    return np.stack([gauss, esc, noise, zeros])


def test_cpu_encoder_roundtrips_through_cpu_decoder():
    tiles = _tiles(4)
    blob = xr.encode_tiles(tiles)
    n, lens, toff = xr.blob_header(blob)
    assert n == len(tiles) and toff[-1] == len(blob)
    for t in range(n):
        assert np.array_equal(xr.decode_tile(blob, t), tiles[t]), t
    assert toff[3] - toff[2] == 80 + 16384  # the noise tile is stored raw
    # a blob of Gaussian tiles (one code per blob, built from its own histogram): sign|mantissa
    # byte + ~2.5 bits of exponent code
    g = xr.encode_tiles(np.stack([_tiles(s)[0] for s in range(3)]))
    assert len(g) < 0.72 * 3 * 16384


def test_code_lengths_are_a_complete_prefix_code():
    for counts in ([1] * 17, [10 ** 6 // (2 ** i) + 1 for i in range(17)], [5, 0, 0, 1] + [0] * 13):
        lens = xr.huffman_lengths(counts)
        assert max(lens) <= xr.LUT_BITS
        assert abs(sum(2.0 ** -l for l in lens) - 1.0) < 1e-12  # Kraft equality: the table is full
