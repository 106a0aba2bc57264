"""Host->device bandwidth from pinned memory on this box (the ceiling of bench.py's e2e):
one 614 MB copy (a C2 step's X, Y), the same bytes in 37 MB chunks (a wave's rows) on one
stream and alternating over two streams.  CUDA events; best of 5."""
import json

import torch

nbytes = 614_400_000
chunk = 36_864_000
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def one():
    d.copy_(h, non_blocking=True)


def chunks(streams):
    for i, o in enumerate(range(0, nbytes, chunk)):
        s = streams[i % len(streams)]
        with torch.cuda.stream(s):
            n = min(chunk, nbytes - o)
            d[o:o + n].copy_(h[o:o + n], non_blocking=True)


res = {}
for name, fn in [("single", one), ("chunks_1stream", lambda: chunks([s1])), ("chunks_2streams", lambda: chunks([s1, s2]))]:
    ms = timed(fn)
    res[name] = {"ms": ms, "GB/s": nbytes / ms / 1e6}
print(json.dumps(res))
