"""Pinned H2D rate of one ~100 MB expert blob copied whole, in N chunks on one stream, and in N
chunks alternating over two streams (the per-copy gap between back-to-back chunks on one stream is
what the chunked codec pipeline pays)."""
import torch

nbytes = 102 << 20
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(chunks, streams, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for s in streams:
        s.wait_stream(cur)
    for _ in range(reps):
        for c in range(chunks):
            a, b = nbytes * c // chunks, nbytes * (c + 1) // chunks
            s = streams[c % len(streams)]
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
    for s in streams:
        cur.wait_stream(s)
    e1.record(cur)
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


run(1, [s1])
for n in (1, 2, 4, 8, 16, 32):
    print(f"{n:3d} chunks: 1 stream {run(n, [s1]):6.2f} GB/s   2 streams {run(n, [s1, s2]):6.2f} GB/s")
