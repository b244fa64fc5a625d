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


def huffman_lengths(counts, max_len=LUT_BITS):
    """Length-limited Huffman code lengths as the encoder builds them (xcodec.cu huff_lengths)."""
    import heapq
    cnt = [max(int(c), 1) for c in counts]
    while True:
        heap = [(c, i) for i, c in enumerate(cnt)]
        heapq.heapify(heap)
        parent = {}
        nxt = SYMS
        while len(heap) > 1:
            a, b = heapq.heappop(heap), heapq.heappop(heap)
            parent[a[1]] = parent[b[1]] = nxt
            heapq.heappush(heap, (a[0] + b[0], nxt))
            nxt += 1
        lens = []
        for i in range(SYMS):
            l, p = 0, i
            while p in parent:
                p = parent[p]
                l += 1
            lens.append(l)
        if max(lens) <= max_len:
            return lens
        cnt = [(c >> 1) | 1 for c in cnt]


def encode_tiles(tiles_u16):
    """CPU restatement of the encoder (tests only): [n, 8192] uint16 tile images -> blob bytes."""
    tiles = np.asarray(tiles_u16, dtype=np.uint16).reshape(-1, VALS)
    n = tiles.shape[0]
    exps = (tiles >> 7) & 0xFF
    emax = exps.max(axis=1)
    syms = np.minimum(emax[:, None] - exps, ESC)
    lens = huffman_lengths(np.bincount(syms.ravel(), minlength=SYMS))
    codes = canonical_codes(lens)
    out = []
    for t in range(n):
        sm = (((tiles[t] >> 8) & 0x80) | (tiles[t] & 0x7F)).astype(np.uint8)
        streams = []
        for lane in range(32):
            bits = []
            for j in range(64):
                for q in range(4):
                    v = 128 * j + 4 * lane + q
                    s = int(syms[t, v])
                    c, l = codes[s]
                    bits.append(format(c, "0%db" % l))
                    if s == ESC:
                        bits.append(format(int(exps[t, v]), "08b"))
            b = "".join(bits)
            b += "0" * (-len(b) % 32)
            streams.append([int(b[i:i + 32], 2) for i in range(0, len(b), 32)])
        seg, words = [], []
        for st in streams:
            seg.append(len(words))
            words.extend(st)
        size = (THDR + VALS + 4 * len(words) + 15) & ~15
        if size >= THDR + 2 * VALS:  # raw tile
            tile = np.zeros(THDR + 2 * VALS, dtype=np.uint8)
            tile[:4] = np.array([int(emax[t]) | (1 << 8)], dtype=np.uint32).view(np.uint8)
            tile[THDR:] = tiles[t].view(np.uint8)
        else:
            tile = np.zeros(size, dtype=np.uint8)
            tile[:8] = np.array([int(emax[t]), len(words)], dtype=np.uint32).view(np.uint8)
            tile[16:80] = np.array(seg, dtype=np.uint16).view(np.uint8)
            tile[THDR:THDR + VALS] = sm
            tile[THDR + VALS:THDR + VALS + 4 * len(words)] = np.array(words, dtype=np.uint32).view(np.uint8)
        out.append(tile)
    hdr = 64 + ((4 * (n + 1) + 15) & ~15)
    off = [hdr]
    for tile in out:
        off.append(off[-1] + len(tile))
    head = np.zeros(hdr, dtype=np.uint8)
    head[:16] = np.array([MAGIC, n, hdr, 0], dtype=np.uint32).view(np.uint8)
    head[16:16 + SYMS] = np.array(lens, dtype=np.uint8)
    head[64:64 + 4 * (n + 1)] = np.array(off, dtype=np.uint32).view(np.uint8)
    return np.concatenate([head] + out)
