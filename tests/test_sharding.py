"""Multi-process pixel sharding on CPU (gloo, world_size 2): each rank monitors its shard
(the CPU oracle stands in for the GPU kernel here), the maps are gathered to rank 0 and must
equal the unsharded result bit for bit — the host-side logic of bench.py / sharding.py."""

import os
import socket

import numpy as np
import pytest

from paper_1807_01751_b200.sharding import gather_maps, local_block, shard_bounds


@pytest.mark.parametrize("P,world,align", [(1000, 2, 4), (1001, 3, 4), (7, 4, 4), (4096 * 3 + 5, 8, 256)])
def test_shard_bounds_cover_and_align(P, world, align):
    b = shard_bounds(P, world, align)
    assert len(b) == world
    assert b[0][0] == 0 and b[-1][1] == P
    for (a0, b0), (a1, _) in zip(b[:-1], b[1:]):
        assert b0 == a1
    assert all(a % align == 0 for a, _ in b)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, y, t, q):
    import torch.distributed as dist

    from oracle import bfast_oracle as bo

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        block, start = local_block(y, rank, world, align=4)
        r = bo.monitor(block, t, 100, 50, 3, 23.0, 4.9)
        maps = gather_maps({"valid": r.valid.astype(np.uint8), "first_break": r.first_break,
                            "max_abs_mo": r.max_abs_mo}, rank, world)
        if rank == 0:
            q.put({k: v for k, v in maps.items()})
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_gather_matches_unsharded():
    import torch.multiprocessing as mp

    from oracle import bfast_oracle as bo
    from paper_1807_01751_b200.synth import host_stack

    t = np.arange(1.0, 201.0)
    y = host_stack(1003, t, 23.0, 100, 0.1, seed=4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, y, t, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = bo.monitor(y, t, 100, 50, 3, 23.0, 4.9)
    assert np.array_equal(got["valid"].astype(bool), ref.valid)
    assert np.array_equal(got["first_break"], ref.first_break)
    # the float64 oracle's BLAS rounding depends on block width; the GPU kernel itself is
    # bit-identical under any sharding (test_gpu_parity.py::test_shard_invariance)
    np.testing.assert_allclose(got["max_abs_mo"], ref.max_abs_mo, rtol=1e-12, atol=0)


def _worker_dev(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1807_01751_b200.sharding import gather_device_maps

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 5 + 3 * rank                      # ragged shards
        base = 100 * rank
        valid = torch.tensor([(base + i) % 2 for i in range(n)], dtype=torch.uint8)
        first = torch.arange(base, base + n, dtype=torch.int32)
        mx = torch.arange(base, base + n, dtype=torch.float32) * 0.5
        out = gather_device_maps(valid, first, mx, rank, world)
        if rank == 0:
            q.put([t.numpy().copy() for t in out])
    finally:
        dist.destroy_process_group()


def test_gloo_device_map_gather():
    """The packed-byte gather bench.py uses for whole-box maps (NCCL on the GPU box)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_dev, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    v, f, m = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_f = np.concatenate([np.arange(0, 5), np.arange(100, 108)]).astype(np.int32)
    assert np.array_equal(f, want_f)
    assert np.array_equal(m, want_f.astype(np.float32) * 0.5)
    assert np.array_equal(v, (want_f % 2).astype(np.uint8))
