"""bench.py — bfastmonitor throughput on B200 (BASELINE.json metric: Mpixels/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C2]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

A step = one fused bfastmonitor pass (libbwm kernel launch) over one synthetic NDVI-like
stack resident in HBM.  N=1 runs BASELINE config 2 (4096x4096 px, N=228 dates, n=114,
k=3, h=28, 20% NaN).  For N>1 every rank runs its own config-2 stack (pixel tiles are
independent: no data-path collective; weak scaling); the step time is the max over ranks.

Rank 0 prints ONE JSON line: value (device-resident input), e2e (numpy stack in pinned
host memory -> monitor_batch -> numpy BreakMap, H2D/D2H inside the timed region),
roofline of the kernel against the measured HBM copy bandwidth, the CPU baseline (the
float64 oracle port of the reference fused backend on a bounded sample, host cores), clocks
sampled during the timed region, and the number of libbwm kernel launches.

--impl reference times the reference algorithm's CPU implementation (the oracle port, all
host threads) on bounded samples of the same workload; see DESIGN.md.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "Mpixels/s for bfastmonitor at 1/2/4/8 B200; HBM GB/s vs peak; CPU speedup"
UNIT = "Mpixels/s"


def default_workload(gpus: int) -> str:
    """BASELINE.json: config 2 (C2) is the 1-GPU configuration, config 3 (C3, the 16384^2
    scene) the 2/4/8-GPU one — the north-star gate."""
    return "C2" if gpus == 1 else "C3"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=["C1", "C2", "C3", "C4", "C5"],
                    help="default: C2 for --gpus 1, C3 (the 16384^2 scene, one pixel band per rank, strong "
                         "scaling) for --gpus >= 2; C1/C2/C4/C5 with N > 1: every rank runs the whole config "
                         "(weak scaling)")
    ap.add_argument("--pixels", type=int, default=None,
                    help="override the workload's pixel count (e.g. a C3-shaped scene small enough for "
                         "two ranks sharing one GPU)")
    ap.add_argument("--nan-mode", default="fill", choices=["fill", "mask"],
                    help="fill: the reference's gap fill (headline); mask: per-pixel masked fits (extension)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-file", action="store_true",
                    help="also time monitor_file on a BTS1 copy of the stack (page cache: /dev/shm or /tmp)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without a GPU: every rank resolves its pixel band, rank 0 gathers them "
                         "over gloo and prints them (tests/test_bench_host.py)")
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="pixels in the CPU baseline sample (default: the SURVEY §8(d) tile, 1024^2 for "
                         "C1-C3 geometry, 512^2 for C4/C5)")
    args = ap.parse_args(argv)
    if args.steps < 1 or args.warmup < 0 or args.e2e_steps < 1:
        ap.error("--steps and --e2e-steps must be >= 1, --warmup >= 0")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.pixels is not None and args.pixels < 1:
        ap.error("--pixels must be >= 1")
    if args.workload is None:
        args.workload = default_workload(args.gpus)
    return args


def free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launcher_command(argv, gpus: int, port: int) -> list:
    """`python bench.py --gpus N ...` without a torchrun environment re-executes itself under
    torch.distributed.run, one rank per GPU (the driver's own launch line)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *argv]


def check_world(gpus: int, env=None) -> int:
    """World size from the launcher environment; it must equal --gpus."""
    env = os.environ if env is None else env
    world = int(env.get("WORLD_SIZE", "1"))
    if world != gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {gpus}: launch one rank per GPU "
                         f"(torchrun --nproc-per-node {gpus}) or run `python bench.py --gpus {gpus}` to spawn them")
    return world


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def bytes_per_pixel(w, beta=False, mean=False):
    """Algorithmic bytes per pixel: y read once + first_idx + max_abs + valid."""
    b = 4 * w.n_obs + 4 + 4 + 1
    if beta:
        b += 4 * (2 + 2 * w.harmonics)
    if mean:
        b += 4
    return b


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms while running."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.reader = None
        self.error = "nvidia-smi unavailable"

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return self
        import threading

        self.reader = threading.Thread(target=self._read, daemon=True)
        self.reader.start()
        t0 = time.monotonic()                  # nvidia-smi takes a few 100 ms to start: wait for
        while not self.lines and self.proc.poll() is None and time.monotonic() - t0 < 5.0:
            time.sleep(0.01)                   # its first sample so short timed regions are covered
        if not self.lines:
            self.error = "nvidia-smi produced no samples"
        return self

    def __exit__(self, *exc):
        if self.proc is None:
            return
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            self.proc.wait()
        self.reader.join(timeout=5)

    def summary(self):
        if not self.lines:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.error], "samples": 0}
        rows = [[c.strip() for c in line.split(",")] for line in self.lines if line.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i] == "Active"})
        loaded = [s for s in sm if smax and s >= 0.3 * max(smax)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons, "samples": len(rows)}


def dist_setup(n_gpus):
    """One rank per GPU: NCCL over NVLink when every rank has its own device; gloo when ranks
    share one (a 1-GPU check of the multi-rank path)."""
    import torch

    world = check_world(n_gpus)
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        ndev = torch.cuda.device_count()
        dev = local % ndev
        torch.cuda.set_device(dev)
        if ndev >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
        return world, rank, dev
    if torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    v = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return float(v.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


REF_DIR = REPO / "baseline" / "_ref"


def reference_module():
    """The UNMODIFIED reference package `breakwatch` (pip-installed into baseline/_ref, which
    travels to the GPU box; /root/reference/pkg/src where it exists), or None."""
    for d in (REF_DIR, Path("/root/reference/pkg/src")):
        if (d / "breakwatch" / "__init__.py").exists():
            if str(d) not in sys.path:
                sys.path.insert(0, str(d))
            import breakwatch

            return breakwatch
    return None


def default_cpu_sample(w) -> int:
    """the reference is timed on a 1024^2 tile (C1-C3 geometry; C1 in full) or a
    512^2 tile (C4/C5) and scaled per pixel."""
    if w.name == "C1":
        return w.n_pixels
    return 1 << 20 if w.n_obs <= 228 else 1 << 18


class CpuArm:
    """One bounded sample of the workload on the host cores, timed through the reference's own
    public API: breakwatch.profile_run(stack, MonitorConfig(..., crit_value=lambda),
    threads=os.cpu_count()) — fused backend, numba kernels, BLAS pinned to one thread by the
    reference itself (engine.py:288-293).  Without the reference package it falls back to the
    oracle port under the same BLAS pin (kind "port")."""

    def __init__(self, w, t, sample_px: int, threads: int, nan_mode: str = "fill"):
        from paper_1807_01751_b200.synth import host_stack

        self.w, self.t, self.threads, self.nan_mode = w, t, threads, nan_mode
        self.sample = int(sample_px)
        self.y = host_stack(self.sample, t, w.freq, w.n_hist, w.nan_frac, seed=99, clustered=w.clustered,
                            cols=int(np.sqrt(self.sample)))
        self.ref = reference_module() if nan_mode == "fill" else None
        if self.ref is not None:
            self.kind = "reference"
            self.stack = self.ref.SeriesStack(self.y, self.ref.TimeAxis(t))
            self.cfg = self.ref.MonitorConfig(history=w.n_hist, bandwidth=w.bandwidth, harmonics=w.harmonics,
                                              freq=w.freq, crit_value=w.crit)
            self.what = (f"reference breakwatch {getattr(self.ref, '__version__', '')} profile_run "
                         f"(fused backend, {self.ref._kernels.ACTIVE} kernels, BLAS pinned to 1 thread by the "
                         f"reference), imported from {Path(self.ref.__file__).parent.parent}")
        else:
            self.kind = "port"
            self.what = ("oracle port of the reference fused backend (oracle/bfast_oracle.py), BLAS pinned to "
                         "1 thread as engine.py:288-293 does" if nan_mode == "fill" else
                         "masked-mode oracle (oracle/bfast_oracle.py:monitor_masked, per-pixel float64)")

    def once(self) -> float:
        """Seconds for one pass over the sample."""
        t0 = time.perf_counter()
        if self.ref is not None:
            self.ref.profile_run(self.stack, self.cfg, threads=self.threads)
        else:
            from threadpoolctl import threadpool_limits

            from oracle import bfast_oracle as bo

            w = self.w
            with threadpool_limits(limits=1, user_api="blas"):
                if self.nan_mode == "mask":
                    bo.monitor_masked(self.y, self.t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit)
                else:
                    bo.monitor(self.y, self.t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit,
                               threads=self.threads)
        return time.perf_counter() - t0

    def describe(self, value: float, seconds: float) -> dict:
        return {"value": value, "unit": UNIT, "cores": self.threads, "kind": self.kind,
                "sample": f"{self.sample} px of the {self.w.name} geometry (N={self.w.n_obs}, n={self.w.n_hist}, "
                          f"k={self.w.harmonics}, h={self.w.bandwidth}, lambda pinned), {seconds:.1f} s of CPU "
                          f"work; {self.what}; {self.threads} threads ({cpu_model()})"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown CPU"


def cpu_baseline(w, t, sample_px, threads, nan_mode="fill", reps=3):
    """Best of `reps` passes of the CPU arm (after one warm pass: numba compile, page faults)."""
    if nan_mode == "mask":                  # per-pixel float64 Python loop: a small sample, one thread
        sample_px, threads, reps = min(sample_px, 4096), 1, 1
    arm = CpuArm(w, t, sample_px, threads, nan_mode)
    arm.once()
    times = [arm.once() for _ in range(reps)]
    best = min(times)
    return arm.describe(arm.sample / best / 1e6, sum(times))


def run_reference_arm(args):
    """--impl reference: the reference's CPU implementation of the path on the host cores, on
    bounded samples of the same workload; rank 0 alone works under torchrun."""
    from paper_1807_01751_b200.synth import WORKLOADS, time_axis

    check_world(args.gpus) if "WORLD_SIZE" in os.environ else None
    if int(os.environ.get("RANK", "0")) != 0:
        return
    w = WORKLOADS[args.workload]
    t = time_axis(w)
    threads = os.cpu_count() or 1
    sample = args.cpu_sample or default_cpu_sample(w)
    arm = CpuArm(w, t, min(sample, 1 << 16), threads, args.nan_mode)
    probe = arm.once()                           # warm (numba compile) + rate estimate
    rate = arm.sample / max(arm.once(), 1e-6)
    # each step one sample: the SURVEY tile when the whole run fits ~3 minutes, else smaller
    while sample > (1 << 16) and (args.steps + args.warmup) * sample / rate > 180.0:
        sample //= 4
    if sample != arm.sample:
        arm = CpuArm(w, t, sample, threads, args.nan_mode)
    for _ in range(args.warmup):
        arm.once()
    times = [arm.once() for _ in range(args.steps)]
    dt = sum(times)
    value = arm.sample * args.steps / dt / 1e6
    cpu = arm.describe(value, dt)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic NDVI-like stack (numpy, seeded)",
        "config": {"workload": f"{w.name}: {w.rows}x{w.cols} px, N={w.n_obs}, n={w.n_hist}, k={w.harmonics}, "
                               f"h={w.bandwidth}, {int(w.nan_frac * 100)}% NaN; CPU sample {arm.sample} px/step",
                   "lambda": w.crit, "nan_mode": args.nan_mode, "probe_s": probe},
        "cpu_baseline": cpu,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def h2d_link_gbs(host, nbytes: int = 1 << 30) -> float:
    """Measured pinned host -> device copy rate (GB/s): two nbytes halves on two streams."""
    import torch

    flat = host.view(-1).view(torch.uint8)[: 2 * nbytes]
    dev = torch.empty(2 * nbytes, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(2)]

    def once():
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                dev[i * nbytes:(i + 1) * nbytes].copy_(flat[i * nbytes:(i + 1) * nbytes], non_blocking=True)
        torch.cuda.synchronize()

    once()
    t0 = time.perf_counter()
    for _ in range(3):
        once()
    dt = time.perf_counter() - t0
    del dev
    return 3 * 2 * nbytes / dt / 1e9


def e2e_file(ynp, t, cfg, steps, world):
    """monitor_file on a BTS1 file of the same stack (dataio.monitor_file -> bwm_monitor_file):
    file read (page cache) + H2D + kernel + D2H; the file lives in /dev/shm (RAM) when it fits."""
    import shutil
    import tempfile

    from paper_1807_01751_b200 import SeriesStack, TimeAxis, monitor_file, write_stack

    need = ynp.nbytes + (1 << 30)
    for d in ("/dev/shm", tempfile.gettempdir()):
        try:
            if shutil.disk_usage(d).free > need:
                break
        except OSError:
            continue
    else:
        return {"skipped": f"no directory with {need / 1e9:.1f} GB free"}
    path = os.path.join(d, f"bench_{os.getpid()}.bts")
    try:
        t0 = time.perf_counter()
        write_stack(SeriesStack(ynp, TimeAxis(t)), path)
        t_write = time.perf_counter() - t0
        monitor_file(path, cfg)                               # warm: staging slots, plan
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(steps):
            bm = monitor_file(path, cfg)
        dt = max_over_ranks(time.perf_counter() - t0, world)
        assert bm.break_count > 0
        return {"value": world * ynp.shape[1] * steps / dt / 1e6, "unit": UNIT, "ms_per_step": 1e3 * dt / steps,
                "file_gb": ynp.nbytes / 1e9, "dir": d, "write_s": t_write,
                "path": "monitor_file(BTS1 path): pread row blocks into pinned slots (reader threads) "
                        "overlapped with H2D, kernel, finalize, D2H"}
    finally:
        try:
            os.remove(path)
        except OSError:
            pass


def host_budget_pixels(n_obs: int, world: int, want: int) -> int:
    """Pixels of a rank's pinned e2e stack that fit the host: half the available RAM split
    over the ranks (the box's RAM, not HBM, bounds the end-to-end run at C3)."""
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:  # pragma: no cover
        return want
    cap = int(0.5 * avail / max(world, 1) / (4 * n_obs))
    return max(256, min(want, (cap // 256) * 256))


def dry_run(args):
    """The rank/band plan of a real run, without touching a GPU."""
    import torch
    import torch.distributed as dist

    from paper_1807_01751_b200.sharding import shard_bounds
    from paper_1807_01751_b200.synth import WORKLOADS

    world = check_world(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    w = WORKLOADS[args.workload]
    scene_px = args.pixels or w.n_pixels
    band = shard_bounds(scene_px, world, align=256)[rank] if args.workload == "C3" else (0, scene_px)
    bands = [band]
    if world > 1:
        dist.init_process_group("gloo")
        got = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(got, torch.tensor(band, dtype=torch.int64))
        bands = [tuple(int(v) for v in g) for g in got]
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "workload": w.name, "pixels_total": scene_px,
                          "scaling": "strong" if args.workload == "C3" else "weak", "bands": bands}), flush=True)


def run_ours(args):
    import torch

    from paper_1807_01751_b200 import MonitorConfig, SeriesStack, TimeAxis, _lib, monitor_batch
    from paper_1807_01751_b200.device import DevicePlan
    from paper_1807_01751_b200.sharding import shard_bounds
    from paper_1807_01751_b200.synth import WORKLOADS, device_stack, time_axis

    world, rank, local = dist_setup(args.gpus)
    dev = torch.device("cuda", torch.cuda.current_device())
    w = WORKLOADS[args.workload]
    t = time_axis(w)
    scene_px = args.pixels or w.n_pixels
    strong = args.workload == "C3"
    if strong:                                   # one 256-px-aligned pixel band of the scene per rank
        a, b = shard_bounds(scene_px, world, align=256)[rank]
        P, p_first = b - a, a
    else:                                        # every rank runs the whole config (weak scaling)
        P, p_first = scene_px, 0
    need = P * w.n_obs * 4
    if need > 0.9 * torch.cuda.get_device_properties(dev).total_memory:
        raise SystemExit(f"{w.name}: {need / 1e9:.0f} GB per rank does not fit one GPU; use more ranks "
                         f"(--gpus) or --pixels")
    plan = DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, dev, nan_mode=args.nan_mode)
    y = device_stack(P, t, w.freq, w.n_hist, w.nan_frac, seed=20261017 + rank, device=dev, clustered=w.clustered,
                     cols=w.cols, first_pixel=p_first, scene_rows=(scene_px + w.cols - 1) // w.cols)
    torch.cuda.synchronize()
    res = plan.run_device(y)                    # allocates the output maps once
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        plan.run_device(y, out=res, check_zero=False)
    torch.cuda.synchronize()

    # ---- device-resident timed region -------------------------------------------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    with ClockSampler(dev.index if dev.index is not None else local) as clocks:
        barrier(world)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("bench_timed")
        t_begin = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_begin.record(stream)
        for i in range(args.steps):
            starts[i].record(stream)
            plan.run_device(y, out=res, check_zero=False)
            ends[i].record(stream)
        t_end.record(stream)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        barrier(world)
    launches = _lib.launch_count() - launches0
    elapsed_ms = max_over_ranks(t_begin.elapsed_time(t_end), world)
    kernel_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    k_avg = sum(kernel_ms) / len(kernel_ms)
    ms_per_step = elapsed_ms / args.steps
    total_px = scene_px if strong else world * P
    value = total_px / (ms_per_step * 1e-3) / 1e6
    peak, peak_kind = peaks()
    bpp = bytes_per_pixel(w)
    achieved = P * bpp / (k_avg * 1e-3) / 1e9
    z = int(res._zero_tensor.item())
    if z != _lib.INT64_MAX:
        raise RuntimeError(f"synthetic stack produced a zero-sigma pixel {z}")
    n_breaks = int((res.first_idx > 0).sum().item())

    # ---- whole-box result maps (N > 1): one gather of the 9 B/px device maps, timed apart ----
    gather = None
    if world > 1:
        import torch.distributed as dist

        from paper_1807_01751_b200.sharding import gather_device_maps

        on_dev = dist.get_backend() == "nccl"
        mv = [res.valid, res.first_idx, res.max_abs] if on_dev else [res.valid.cpu(), res.first_idx.cpu(),
                                                                     res.max_abs.cpu()]
        barrier(world)
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        maps = gather_device_maps(*mv, rank, world)
        torch.cuda.synchronize()
        g_ms = max_over_ranks((time.perf_counter() - g0) * 1e3, world)
        gather = {"ms": g_ms, "bytes": total_px * 9, "collective": "gather of packed u8/i32/f32 maps to rank 0 "
                  f"({dist.get_backend()})", "note": "whole-box maps on rank 0; not part of the step"}
        if rank == 0:
            assert int(maps[0].numel()) == total_px
            gather["breaks"] = int((maps[1] > 0).sum().item())

    # ---- end to end through the public API: pinned host stack -> BreakMap ------------------
    e2e = None
    if not args.no_e2e:
        Pe = host_budget_pixels(w.n_obs, world, P)
        host = torch.empty((w.n_obs, Pe), dtype=torch.float32, pin_memory=True)
        host.copy_(y[:, :Pe])
        del y, res
        torch.cuda.empty_cache()
        ynp = host.numpy()
        stack = SeriesStack(ynp, TimeAxis(t))
        cfg = MonitorConfig(history=w.n_hist, bandwidth=w.bandwidth, harmonics=w.harmonics, freq=w.freq,
                            crit_value=w.crit, nan_mode=args.nan_mode)
        bm = monitor_batch(stack, cfg)          # warm: pipeline buffers, plan cache, pinned outputs
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            bm = monitor_batch(stack, cfg)
        dt = max_over_ranks(time.perf_counter() - t0, world)
        e2e = {"value": world * Pe * args.e2e_steps / dt / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(ynp.nbytes), "d2h_bytes_per_step": int(Pe * 18 + 16),
               "steps": args.e2e_steps, "ms_per_step": 1e3 * dt / args.e2e_steps, "pixels_per_rank": Pe,
               "path": "monitor_batch(SeriesStack(pinned numpy)) -> bwm_monitor_host: contiguous H2D of the "
                       "stack, one kernel launch, device-side finalize to the reference dtypes, D2H of "
                       "valid/detected/first_break(int64)/max_abs_mo(float64)"}
        if Pe < P:
            e2e["note"] = f"host RAM bounds the pinned stack: {Pe} of the rank's {P} px per step"
        assert bm.break_count > 0
        # the e2e roofline: this box's pinned H2D link rate (two 1 GiB copies on two streams,
        # the way bwm_monitor_host splits the stack) against the stack bytes per step
        link = h2d_link_gbs(host, min(1 << 30, ynp.nbytes // 2))
        e2e["h2d_link_gbs"] = link
        e2e["h2d_link_frac"] = ynp.nbytes / (e2e["ms_per_step"] * 1e-3) / 1e9 / link
        if args.e2e_file:
            e2e["file"] = e2e_file(ynp, t, cfg, args.e2e_steps, world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(w, t, args.cpu_sample or default_cpu_sample(w), os.cpu_count() or 1, args.nan_mode)

    prof = REPO / "profiles" / "traffic.json"
    entry = {}
    if prof.exists():
        entry = json.loads(prof.read_text()).get(w.name + ("-mask" if args.nan_mode == "mask" else "")) or {}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic NDVI-like stack generated in HBM (torch Philox), seed 20261017+rank",
            "config": {"workload": f"{w.name}: {scene_px} px " + (f"split over {world} GPUs" if strong else "per GPU")
                                   + f", N={w.n_obs} dates, n={w.n_hist}, "
                                   f"k={w.harmonics}, h={w.bandwidth}, "
                                   + ("clustered cloud-disc NaNs" if w.clustered else f"{int(w.nan_frac * 100)}% NaN"),
                       "nan_mode": args.nan_mode,
                       "pixels_total": total_px, "pixels_per_rank": P, "lambda": w.crit,
                       "l2": f"input {w.n_obs * P * 4 / 1e9:.1f} GB per GPU >> 126 MB L2 (no flush needed)",
                       "parallelism": f"pixel bands, {world} rank(s), no collective on the data path"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": entry.get("dram_bytes_per_launch"),
                         "traffic_source": entry.get("source"), "peak_kind": peak_kind,
                         "bytes_per_pixel": bpp, "kernel_ms": k_avg, "launch": plan.info(),
                         "tensor_pipe": entry.get("tensor_pipe")},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gather": gather,
            "breaks_rank0": n_breaks,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # plain `python bench.py --gpus N`: spawn the N ranks (one per GPU) and pass rank 0's line through
        raise SystemExit(subprocess.run(launcher_command(argv, args.gpus, free_port())).returncode)
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.dry_run:
        dry_run(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
