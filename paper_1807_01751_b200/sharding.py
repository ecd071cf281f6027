"""Pixel sharding across GPUs (one process per GPU, torch.distributed for the plumbing).

BFAST-monitor pixels are independent (reference engine.py:345-409 computes each column from
its own series plus shared constants), so a stack shards into contiguous pixel ranges with
no collective on the data path.  Ranges are aligned to `align` pixels so every shard keeps
the 16-byte row alignment the TMA kernel wants.  Results are bit-identical for any
sharding (tests/test_gpu_parity.py::test_shard_invariance): a pixel's arithmetic never
depends on where it runs.

The only collective is the optional gather of the (small) result maps to rank 0 for a
whole-box result — NCCL on the GPU box, gloo in the CPU tests.
"""

from __future__ import annotations

from typing import Optional

import numpy as np


def shard_bounds(n_pixels: int, world: int, align: int = 4) -> list[tuple[int, int]]:
    """Contiguous [start, stop) pixel ranges, one per rank, starts aligned to `align`."""
    if world < 1 or n_pixels < 0:
        raise ValueError("world must be >= 1 and n_pixels >= 0")
    units = (n_pixels + align - 1) // align
    bounds = []
    for r in range(world):
        a = min(n_pixels, (units * r // world) * align)
        b = min(n_pixels, (units * (r + 1) // world) * align)
        bounds.append((a, b))
    return bounds


def local_block(data, rank: int, world: int, align: int = 4):
    """This rank's pixel columns of a time-major (N, P) stack (a view, no copy)."""
    a, b = shard_bounds(int(data.shape[1]), world, align)[rank]
    return data[:, a:b], a


MAP_FIELDS = ("valid", "first_break", "max_abs_mo")


def gather_maps(local: dict, rank: int, world: int, group=None) -> Optional[dict]:
    """Gather per-rank result maps (1-D numpy arrays, contiguous shards) to rank 0.

    Uses torch.distributed.all_gather_object-free tensors: every map is gathered with
    all_gather on a padded tensor (shards may differ by `align` pixels), then trimmed.
    Returns the concatenated maps on rank 0, None elsewhere.
    """
    import torch
    import torch.distributed as dist

    if world == 1:
        return {k: np.asarray(v) for k, v in local.items()}
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    n_local = torch.tensor([len(next(iter(local.values())))], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    sizes = [int(s.item()) for s in sizes]
    width = max(sizes)
    out = {}
    for key in sorted(local):
        arr = np.asarray(local[key])
        t = torch.zeros(width, dtype=torch.float64, device=device)
        t[: arr.size] = torch.as_tensor(arr.astype(np.float64), device=device)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        if rank == 0:
            full = np.concatenate([p[:s].cpu().numpy() for p, s in zip(parts, sizes)])
            out[key] = full.astype(arr.dtype)
    return out if rank == 0 else None


def gather_device_maps(valid, first_idx, max_abs, rank: int, world: int, group=None):
    """Whole-box result maps on rank 0 from the per-rank DEVICE maps (the kernel's raw u8 /
    i32 / f32 outputs, 9 B per pixel), packed into one byte tensor per rank and gathered to
    rank 0 with one collective over NVLink (NCCL; gloo with CPU tensors in the tests).  Returns
    (valid, first_idx, max_abs) tensors on rank 0 in global pixel order, None elsewhere."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return valid, first_idx, max_abs
    n = int(valid.numel())
    packed = torch.cat([first_idx.contiguous().view(torch.uint8), max_abs.contiguous().view(torch.uint8),
                        valid.contiguous().view(torch.uint8)])          # 4-byte fields first: aligned views
    sizes = [torch.zeros(1, dtype=torch.int64, device=valid.device) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([n], dtype=torch.int64, device=valid.device), group=group)
    sizes = [int(s.item()) for s in sizes]
    width = 9 * max(sizes)
    buf = torch.zeros(width, dtype=torch.uint8, device=valid.device)
    buf[: packed.numel()] = packed
    # gather (not all_gather): only rank 0 receives, so each rank sends its maps once over
    # NVLink instead of to every peer
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
    dist.gather(buf, gather_list=parts, dst=0, group=group)
    if rank != 0:
        return None
    v, f, m = [], [], []
    for p, s in zip(parts, sizes):
        f.append(p[:4 * s].view(torch.int32))
        m.append(p[4 * s:8 * s].view(torch.float32))
        v.append(p[8 * s:9 * s])
    return torch.cat(v), torch.cat(f), torch.cat(m)
