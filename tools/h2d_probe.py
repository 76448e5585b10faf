"""Pinned host -> device copy bandwidth of the bench's e2e id volume (25.2 GB),
one stream vs chunks over several streams: the e2e leg's link bound.

    python tools/h2d_probe.py
"""
import torch, time, json
n = 25232932864 // 2
h = torch.empty(n, dtype=torch.int16, pin_memory=True)
d = torch.empty(n, dtype=torch.int16, device='cuda')
torch.cuda.synchronize()
def run(nstreams, nchunks):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    ch = n // nchunks
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(nchunks):
        s = ss[i % nstreams]
        with torch.cuda.stream(s):
            d[i*ch:(i+1)*ch].copy_(h[i*ch:(i+1)*ch], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0
for cfg in [(1,1),(1,8),(2,8),(4,16),(1,1),(2,2)]:
    t = min(run(*cfg) for _ in range(2))
    print(json.dumps({"streams": cfg[0], "chunks": cfg[1], "s": t, "GBps": n*2/t/1e9}))
