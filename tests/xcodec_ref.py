"""CPU restatement of the expert-codec blob format (paper_2511_14102_b200/csrc/xcodec.cu header
comment) -- test infrastructure only: an independent decoder that the GPU-encoded blobs must
round-trip through, so the format is pinned by two implementations, not one."""
import numpy as np

MAGIC, SYMS, ESC, LUT_BITS, THDR, VALS = 0x31424358, 17, 16, 12, 80, 8192


def canonical_codes(lens):
    codes, code = {}, 0
    for l in range(1, LUT_BITS + 1):
        for s in range(SYMS):
            if lens[s] == l:
                codes[s] = (code, l)
                code += 1
        code <<= 1
    return codes


def blob_header(blob):
    b = np.asarray(blob, dtype=np.uint8)
    magic, n_tiles, hdr_bytes, _ = b[:16].view(np.uint32)
    assert magic == MAGIC, hex(int(magic))
    lens = [int(x) for x in b[16:16 + SYMS]]
    toff = b[64:64 + 4 * (int(n_tiles) + 1)].view(np.uint32).astype(np.int64)
    return int(n_tiles), lens, toff


def decode_tile(blob, t):
    b = np.asarray(blob, dtype=np.uint8)
    n_tiles, lens, toff = blob_header(b)
    tile = b[toff[t]:toff[t + 1]]
    h0 = int(tile[:4].view(np.uint32)[0])
    em, mode = h0 & 0xFF, h0 >> 8
    if mode:
        return tile[THDR:THDR + 2 * VALS].view(np.uint16).copy()
    seg = tile[16:80].view(np.uint16)
    sm = tile[THDR:THDR + VALS]
    words = tile[THDR + VALS:].view(np.uint32) if (len(tile) - THDR - VALS) % 4 == 0 else \
        tile[THDR + VALS:len(tile) - (len(tile) - THDR - VALS) % 4].view(np.uint32)
    dec = {(c, l): s for s, (c, l) in canonical_codes(lens).items()}
    out = np.zeros(VALS, dtype=np.uint16)
    for lane in range(32):
        bits = "".join(format(int(w), "032b") for w in words[int(seg[lane]):int(seg[lane]) + 64 * 4 * 20 // 32 + 2])
        p = 0
        for j in range(64):
            for q in range(4):
                v = 128 * j + 4 * lane + q
                code, l = 0, 0
                while (code, l) not in dec:
                    code = (code << 1) | (bits[p] == "1")
                    l += 1
                    p += 1
                    assert l <= LUT_BITS
                s = dec[(code, l)]
                if s == ESC:
                    e = int(bits[p:p + 8], 2)
                    p += 8
                else:
                    e = em - s
                smb = int(sm[v])
                out[v] = ((smb & 0x80) << 8) | (e << 7) | (smb & 0x7F)
    return out
