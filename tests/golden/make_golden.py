"""Generate golden fixtures by running the REFERENCE (breakwatch, read-only at
/root/reference/pkg/src) on seeded inputs.  Run in the build container:

    python tests/golden/make_golden.py

Inputs come from paper_1807_01751_b200.synth.host_stack (numpy PCG64, seeded) or the
reference's own generator; small inputs are stored verbatim, large ones by SHA-256 so the
test can regenerate and verify them.  Outputs are the reference's monitor_batch results
(fused backend, numba kernels, lambda pinned).  The MOSUM matrix itself is stored only as
the sparse set of (j, pixel) windows within rtol 1e-4 of the boundary — what the parity
test needs to classify borderline pixels.

/root/reference is not needed (and does not exist) on the GPU box: the tests read only
the committed .npz files.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import breakwatch as bw  # noqa: E402  (the reference)

from oracle.bfast_oracle import near_pairs  # noqa: E402
from paper_1807_01751_b200.synth import WORKLOADS, host_stack, time_axis  # noqa: E402
from tests.golden_cases import edge_stack  # noqa: E402

STORE_INPUT_MAX = 1 << 20   # bytes


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_reference(y, t, n, h, k, f, crit):
    stack = bw.SeriesStack(y, bw.TimeAxis(t))
    cfg = bw.MonitorConfig(history=n, bandwidth=h, harmonics=k, freq=f, crit_value=crit)
    bm = bw.monitor_batch(stack, cfg, keep_mosum=True)
    design = bw.build_design_matrix(bw.TimeAxis(t), f, k)
    mapping = bw.fit_mapping(design, n).matrix
    filled = np.zeros((y.shape[0], y.shape[1]))
    for px in range(y.shape[1]):
        try:
            filled[:, px] = bw.fill_gaps(y[:, px])
        except bw.AllNanSeriesError:
            pass
    beta = mapping @ filled[:n]
    bound = bw.boundary_values(n, y.shape[0], crit)
    return bm, beta, bound


def save(name, y, t, n, h, k, f, crit, meta=None, store_input=None):
    bm, beta, bound = run_reference(y, t, n, h, k, f, crit)
    store = store_input if store_input is not None else y.nbytes <= STORE_INPUT_MAX
    arrays = dict(
        t=t, first_break=bm.first_break.astype(np.int32), max_abs_mo=bm.max_abs_mo,
        valid=bm.valid, near=near_pairs(bm.mosum, bound), bound=bound,
        mosum_mean=bm.mosum.mean(axis=0),
    )
    if beta.nbytes <= 4 * STORE_INPUT_MAX:
        arrays["beta"] = beta
    if store:
        arrays["y"] = y
        if bm.mosum.nbytes <= STORE_INPUT_MAX:
            arrays["mosum"] = bm.mosum
    info = dict(n=n, h=h, k=k, freq=f, crit=crit, shape=list(y.shape), y_sha256=sha(y),
                breaks=int(bm.break_count), **(meta or {}))
    np.savez_compressed(HERE / f"{name}.npz", info=json.dumps(info), **arrays)
    print(f"{name}: shape={y.shape} breaks={bm.break_count} near={len(arrays['near'])} stored_input={store}")


def main():
    # 1. the reference's own engine test scenario (test_engine.py:150-158)
    spec = bw.SynthSpec(n_pixels=300, n_obs=200, freq=23.0, noise_std=0.02, break_mag=0.4, seed=11)
    stack = bw.generate(spec)[0]
    data = stack.data.copy()
    rng = np.random.default_rng(11)
    data[rng.random(data.shape) < 0.05] = np.nan
    data[:, 7] = np.nan
    data[:, 42] = np.nan
    save("engine_gaps", data, stack.time_axis.values, 100, 50, 3, 23.0, 4.9, {"source": "reference generate"})

    # 2. configs of BASELINE.json at parity-test size
    w = WORKLOADS["C1"]
    t = time_axis(w)
    y = host_stack(w.n_pixels, t, w.freq, w.n_hist, w.nan_frac, seed=20261018)
    save("c1", y, t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit, {"workload": "C1", "seed": 20261018})

    w = WORKLOADS["C4"]
    t = time_axis(w)
    y = host_stack(64 * 64, t, w.freq, w.n_hist, w.nan_frac, seed=20261021)
    save("c4_tile", y, t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit,
         {"workload": "C4 64x64 tile", "seed": 20261021})

    w = WORKLOADS["C5"]
    t = time_axis(w)
    y = host_stack(96 * 96, t, w.freq, w.n_hist, w.nan_frac, seed=20261022, clustered=True, cols=96)
    save("c5_tile", y, t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit,
         {"workload": "C5 96x96 tile", "seed": 20261022})

    # 3. edge cases (inputs stored verbatim)
    rng = np.random.default_rng(7)
    N, n = 60, 30
    y = edge_stack(rng, N, 300, n)
    t = np.arange(1.0, N + 1)
    save("edges_h10_k2", y, t, n, 10, 2, 12.0, 2.5)
    save("edges_h1_k1", y, t, n, 1, 1, 12.0, 2.5)
    save("edges_hn_k3", y, t, n, n, 3, 12.0, 2.5)
    N, n = 80, 40
    t = np.arange(1.0, N + 1)
    y = host_stack(1001, t, 20.0, n, 0.1, seed=5)        # odd pixel count: tail tile
    save("odd_pixels_k8", y, t, n, 12, 8, 20.0, 3.1)
    y = host_stack(3, t, 20.0, n, 0.0, seed=6, dead_frac=0.0)
    save("three_pixels", y, t, n, 20, 2, 20.0, 3.1)
    t = np.cumsum(np.random.default_rng(9).uniform(0.5, 3.0, N)) + 1.0
    y = host_stack(700, t, 30.0, n, 0.25, seed=9)
    save("irregular_h70", y, t, n, 38, 3, 30.0, 2.9)    # h > 64 would need the lag path: see below
    N, n = 300, 150
    t = np.arange(1.0, N + 1)
    y = host_stack(600, t, 23.0, n, 0.3, seed=10)
    save("lag_h100", y, t, n, 100, 2, 23.0, 3.0)        # h = 100 > 64: lagging-cursor kernel

    # 4. zero-sigma contract: an all-zero pixel fails the batch (test_engine.py:206-215)
    y = host_stack(20, np.arange(1.0, 201.0), 23.0, 100, 0.0, seed=14, dead_frac=0.0)
    y[:, 5] = 0.0
    y[:, 9] = 0.0
    try:
        run_reference(y, np.arange(1.0, 201.0), 100, 50, 3, 23.0, 4.9)
        raise SystemExit("reference did not raise ZeroResidualError")
    except bw.ZeroResidualError as e:
        np.savez_compressed(HERE / "zero_sigma.npz", y=y, info=json.dumps({"message": str(e), "pixel": 5}))
        print("zero_sigma:", e)

    # 5. pinned lambda values of the reference's own tests
    (HERE / "pinned.json").write_text(json.dumps({
        "crit_20k": {"request": dict(alpha=0.05, h_frac=0.5, horizon=2.0, n_sim=100, reps=20000, seed=1),
                     "value": 4.868679234617514, "source": "pkg/tests/test_mosum.py:20"},
        "crit_100k": {"request": dict(alpha=0.05, h_frac=0.5, horizon=2.0, n_sim=100, reps=100000, seed=1),
                      "value": 4.892936439219294, "source": "pkg/tests/test_acceptance.py:39"},
        "crit_c1": {"request": dict(alpha=0.05, h_frac=28 / 114, horizon=2.0, n_sim=114, reps=50000, seed=7),
                    "value": 2.96519227, "source": "SURVEY.md §8(d), resolve_crit_value at C1 geometry"},
    }, indent=1))


def save_masked_common(name, y, t, n, h, k, f, crit, keep):
    """Masked-mode fixture with gaps on the SAME dates in every pixel: the reference, run on
    the compacted series (dates `keep`, history n_v = #kept dates < n, bandwidth
    h_v = floor(h n_v / n)), gives what masked mode must return — the breaks mapped back to
    the original dates and the MOSUM rows to the kept monitoring dates."""
    keep = np.asarray(keep)
    yk, tk = y[keep], t[keep]
    n_v = int(np.sum(keep < n))
    h_v = (h * n_v) // n
    bm, beta, _ = run_reference(yk, tk, n_v, h_v, k, f, crit)
    N = y.shape[0]
    mon = keep[n_v:]                                  # original monitoring dates kept
    first = np.where(bm.first_break > 0, mon[np.maximum(bm.first_break - n_v - 1, 0)] + 1, 0)
    mosum = np.full((N - n, y.shape[1]), np.nan, dtype=np.float32)
    mosum[mon - n] = bm.mosum
    arrays = dict(t=t, y=y, first_break=first.astype(np.int32), max_abs_mo=bm.max_abs_mo, valid=bm.valid,
                  mosum_mean=bm.mosum.mean(axis=0), beta=beta, mosum=mosum, keep=keep,
                  near=near_pairs(bm.mosum, bw.boundary_values(n_v, len(keep), crit)),
                  bound=bw.boundary_values(n, N, crit))
    info = dict(n=n, h=h, k=k, freq=f, crit=crit, shape=list(y.shape), y_sha256=sha(y),
                breaks=int(bm.break_count), nan_mode="mask", n_v=n_v, h_v=h_v,
                source="reference on the compacted series")
    np.savez_compressed(HERE / f"{name}.npz", info=json.dumps(info), **arrays)
    print(f"{name}: shape={y.shape} n_v={n_v} h_v={h_v} breaks={bm.break_count}")


def masked():
    """Fixtures for nan_mode="mask", pinned by the reference itself."""
    # NaN-free input: masked == fill == reference
    t = np.arange(1.0, 229.0)
    y = host_stack(1000, t, 23.0, 114, 0.0, seed=31, dead_frac=0.0)
    save("mask_nanfree", y, t, 114, 28, 3, 23.0, 2.96519227, {"nan_mode": "mask", "seed": 31})
    # gaps on common dates
    rng = np.random.default_rng(32)
    y = host_stack(1000, t, 23.0, 114, 0.0, seed=32, dead_frac=0.0)
    keep = np.sort(rng.choice(228, size=171, replace=False))
    y[np.setdiff1d(np.arange(228), keep)] = np.nan
    save_masked_common("mask_common_c1", y, t, 114, 28, 3, 23.0, 2.96519227, keep)
    tt = np.cumsum(np.random.default_rng(33).uniform(8.0, 24.0, 400)) + 1.0
    y = host_stack(700, tt, 365.25, 200, 0.0, seed=33, dead_frac=0.0)
    keep = np.flatnonzero(np.random.default_rng(34).random(400) > 0.35)
    y[np.setdiff1d(np.arange(400), keep)] = np.nan
    save_masked_common("mask_common_irregular", y, tt, 200, 50, 3, 365.25, 3.0, keep)
    t = np.arange(1.0, 121.0)
    y = host_stack(300, t, 40.0, 60, 0.0, seed=35, dead_frac=0.0)
    keep = np.flatnonzero(np.random.default_rng(36).random(120) > 0.5)
    y[np.setdiff1d(np.arange(120), keep)] = np.nan
    save_masked_common("mask_common_k8_h60", y, t, 60, 60, 8, 40.0, 2.7, keep)


if __name__ == "__main__":
    if sys.argv[1:] == ["masked"]:
        masked()
    else:
        main()
        masked()
