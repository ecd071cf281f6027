"""Pinned H2D of a 15.3 GB stack: one copy vs two halves on two streams vs many chunks
alternating over 2 or 4 streams (how bwm_monitor_host should issue the contiguous copy)."""
import time

import torch

nbytes = 228 * 4096 * 4096 * 4
host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
host.fill_(1)
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(nstreams, chunk):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    off, i = 0, 0
    while off < nbytes:
        n = min(chunk, nbytes - off)
        with torch.cuda.stream(streams[i % nstreams]):
            dev[off:off + n].copy_(host[off:off + n], non_blocking=True)
        off += n
        i += 1
    torch.cuda.synchronize()
    return nbytes / (time.perf_counter() - t0) / 1e9


for ns, ch in [(1, nbytes), (2, nbytes // 2 + 1), (2, 256 << 20), (2, 64 << 20), (2, 32 << 20), (4, 64 << 20),
               (3, 64 << 20)]:
    run(ns, ch)
    print(f"{ns} streams, chunk {ch / 2**20:9.0f} MiB: " + " ".join(f"{run(ns, ch):.1f}" for _ in range(3)) + " GB/s",
          flush=True)
