"""Masked mode without the history re-read: how accurate is beta from the kernel's Gram matrix alone?

The masked kernel forms G_v = G_full - Gm from tf32 hi + lo splits of the float32 x_t x_t^T
(Gm accumulated in float32 by the tensor cores) and refines beta with the exact residuals
X_v r of a second history sweep.  Dropping that sweep means refining with e = g - G_v beta
(converges to G_v^-1 g) and the one-pass RSS q - g^T beta.  This script measures the max
relative error of max|MO| of that scheme (float64 everywhere except the kernel's G_v and
float32 design) against the float64 oracle (oracle/bfast_oracle.py:monitor_masked).

    python experiments/emulate_masked_gv.py [C2|C4|C5] [--px 1500]
"""
import argparse
import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import bfast_oracle as bo  # noqa: E402  (checker only)
from paper_1807_01751_b200.model import TimeAxis, kernel_basis  # noqa: E402
from paper_1807_01751_b200.synth import WORKLOADS, host_stack, time_axis  # noqa: E402


def tf32(x):
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0xFFF + ((b >> 13) & 1)) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="C2")
    ap.add_argument("--px", type=int, default=1500)
    ap.add_argument("--split", choices=("hilo", "exact"), default="hilo",
                    help="x x^T terms as tf32 hi + lo (the kernel) or the exact float32 product")
    ap.add_argument("--centre", action="store_true",
                    help="accumulate deviations x x^T - mean_history(x x^T); the mean times the missing count "
                         "is added back in float64")
    ap.add_argument("--acc", choices=("f32", "f64", "mma"), default="mma",
                    help="accumulation of the Gram complement: float32 per date, float64, or as the tensor "
                         "core does it (one float32 rounding of the accumulator per 8-date K-step and split)")
    a = ap.parse_args()
    w = WORKLOADS[a.workload]
    t = time_axis(w)
    N, n, h, k = w.n_obs, w.n_hist, w.bandwidth, w.harmonics
    p = 2 + 2 * k
    y = host_stack(a.px, t, w.freq, n, w.nan_frac, seed=5, clustered=w.clustered, cols=min(a.px, 128))
    ref = bo.monitor_masked(y, t, n, h, k, w.freq, w.crit)
    X = kernel_basis(TimeAxis(t), w.freq, k, n).design          # [p][N] centred trend, float64
    x32 = X.astype(np.float32).astype(np.float64)
    prod64 = X[:, None, :] * X[None, :, :]
    tbar = prod64[:, :, :n].mean(axis=2) if a.centre else np.zeros((X.shape[0], X.shape[0]))
    prod = (prod64 - tbar[:, :, None]).astype(np.float32)       # x_i x_j per date (centred), float32
    hi = tf32(prod)
    lo = tf32(prod - hi)
    terms = hi.astype(np.float64) + lo.astype(np.float64)         # what the MMA multiplies
    if a.split == "exact":
        terms = prod.astype(np.float64)
    gfull = terms[:, :, :n].sum(axis=2) + n * tbar
    errs = {"one_pass": [], "two_pass": []}
    conds = []
    for px in range(a.px):
        if not ref.valid[px]:
            continue
        col = y[:, px].astype(np.float64)
        ok = np.isfinite(col)
        hist = np.flatnonzero(ok[:n])
        mon = np.flatnonzero(ok[n:]) + n
        nv = hist.size
        hv = (h * nv) // n
        miss = np.flatnonzero(~ok[:n])
        if a.acc == "mma":
            gm = np.zeros((p, p), np.float32)
            mask = ~ok[:n]
            for k0 in range(0, n, 8):
                m = mask[k0:k0 + 8]
                for part in ((hi, lo) if a.split == "hilo" else (prod,)):
                    blk = (part[:, :, k0:k0 + m.size].astype(np.float64) * m).sum(axis=2)
                    gm = (gm.astype(np.float64) + blk).astype(np.float32)
        else:
            gm = np.zeros((p, p), np.float32 if a.acc == "f32" else np.float64)
            for s in miss:                                       # float32 accumulation per date
                gm = (gm + terms[:, :, s].astype(gm.dtype)).astype(gm.dtype)
        Gv = gfull - (gm.astype(np.float64) + miss.size * tbar)
        c = col[hist[0]]
        yc = (col - c).astype(np.float32).astype(np.float64)
        Xv = x32[:, hist]
        g = Xv @ yc[hist]
        beta = np.linalg.solve(Gv, g)
        conds.append(np.linalg.cond(Gv))
        idx = np.concatenate([hist, mon])
        r = yc[idx] - x32[:, idx].T @ beta
        for kind in errs:
            rss = (yc[hist] @ yc[hist] - g @ beta) if kind == "one_pass" else r[:nv] @ r[:nv]
            sig = math.sqrt(rss / (nv - p))
            mo = bo.mosum_block(r[:, None], nv, hv, np.array([1.0 / (sig * math.sqrt(nv))]))[:, 0]
            mx = np.abs(mo).max()
            errs[kind].append(abs(mx - ref.max_abs_mo[px]) / ref.max_abs_mo[px])
    for kind, e in errs.items():
        e = np.array(e)
        print(f"{a.workload} split={a.split} acc={a.acc} centre={a.centre} {kind}: px {e.size} max rel err {e.max():.2e} p99.9 {np.quantile(e, 0.999):.2e} "
              f"(cond G_v median {np.median(conds):.1f}, max {np.max(conds):.1f})")


if __name__ == "__main__":
    main()
