"""Host->device bandwidth for the e2e path's copy shapes (pinned host memory).

1-D contiguous copies vs the strided 2-D column-chunk copies bwm_monitor_host issues
(time-major stack: a pixel chunk is N rows of `width` bytes at pitch P*4)."""
import time

import torch

N, P = 228, 4096 * 4096
host = torch.empty((N, P), dtype=torch.float32, pin_memory=True)
host.fill_(1.0)
dev = torch.empty((N, P), dtype=torch.float32, device="cuda")
torch.cuda.synchronize()


def bw(fn, nbytes, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t0) / 1e9


flat_h = host.view(-1)
flat_d = dev.view(-1)
n1 = 1 << 30
print("1D 4 GB contiguous          %.1f GB/s" % bw(lambda: flat_d[: n1].copy_(flat_h[: n1], non_blocking=True), 4 * n1))
print("full stack contiguous       %.1f GB/s" % bw(lambda: dev.copy_(host, non_blocking=True), host.nbytes, 2))
for chunk in (1 << 18, 1 << 20, 1 << 22):
    def chunked():
        for p0 in range(0, P, chunk):
            dev[:, p0:p0 + chunk].copy_(host[:, p0:p0 + chunk], non_blocking=True)
    print(f"2D column chunks {chunk:>8d} px  %.1f GB/s" % bw(chunked, host.nbytes, 2))
streams = [torch.cuda.Stream() for _ in range(4)]
def rows_4streams():
    rows = N // 4
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            dev[i * rows:(i + 1) * rows].copy_(host[i * rows:(i + 1) * rows], non_blocking=True)
print("row blocks on 4 streams     %.1f GB/s" % bw(rows_4streams, host.nbytes, 2))
