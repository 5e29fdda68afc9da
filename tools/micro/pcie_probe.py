"""H2D / D2H bandwidth from pinned host memory, 1 vs 2 concurrent streams
(the e2e transfers; measurement only)."""
import time

import torch


def run(nbytes=8 << 30, chunks=64, streams=1, d2h=False):
    h = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    d = torch.empty_like(h, device="cuda")
    ss = [torch.cuda.Stream() for _ in range(streams)]
    step = h.numel() // chunks
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for c in range(chunks):
        with torch.cuda.stream(ss[c % streams]):
            sl = slice(c * step, (c + 1) * step)
            if d2h:
                h[sl].copy_(d[sl], non_blocking=True)
            else:
                d[sl].copy_(h[sl], non_blocking=True)
    torch.cuda.synchronize()
    return nbytes / (time.perf_counter() - t0) / 1e9


if __name__ == "__main__":
    for d2h in (False, True):
        for streams in (1, 2, 4):
            run(1 << 30, 8, streams, d2h)
            print(("D2H" if d2h else "H2D"), streams, "streams", round(run(streams=streams, d2h=d2h), 1), "GB/s")
