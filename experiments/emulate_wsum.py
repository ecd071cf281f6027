"""Float32 emulation of the window-sum MOSUM formulation against the float64 oracle.

The fused kernels compute the MOSUM window sum of residuals as
    sum_window r_s = sum_window (y_s - c) - S_t^T beta_Q,   S_t = sum_window z_s
(linear in y), so the monitoring pass needs no per-date fitted value of the lagged date and
window 0 needs no residual conversion.  The intercept part of S_t^T beta_Q is the constant
h/R00 * beta_Q[0] (z_t[0] = 1/R00 for every t, design row 0 = 1) and goes into the initial
window sum in float64; the per-date dot covers k >= 1.

This script replays the kernel's float32 operation order with numpy float32 (each op
rounded) on synthetic stacks of the BASELINE geometries and reports the max relative error
of max|MO| and break-index mismatches outside the borderline band, next to the same numbers
for the residual-ring formulation the kernels used before.

    python experiments/emulate_wsum.py [C1 C4 C5 ...] [--px 8192]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import bfast_oracle as bo  # noqa: E402  (checker only)
from paper_1807_01751_b200.model import TimeAxis, kernel_basis  # noqa: E402
from paper_1807_01751_b200.mosum import boundary_values  # noqa: E402
from paper_1807_01751_b200.synth import WORKLOADS, host_stack, time_axis  # noqa: E402

f32 = np.float32


def tables(t, w):
    basis = kernel_basis(TimeAxis(t), w.freq, w.harmonics, w.n_hist)
    X = basis.design                       # [p][N] f64
    p, N = X.shape
    n, h = w.n_hist, w.bandwidth
    Q, R = np.linalg.qr(X[:, :n].T)        # n x p, p x p
    sg = np.sign(np.diag(R))
    Q, R = Q * sg, (R.T * sg).T
    Z = np.linalg.solve(R.T, X)            # [p][N], z_t = R^-T x_t
    Z[:, :n] = Q.T
    S = np.zeros((N - n, p))
    for j in range(N - n):
        tt = n + j
        S[j] = Z[:, tt - h + 1: tt + 1].sum(axis=1)
    return Q, R, Z, S


def emulate(y, t, w, Q, R, Z, S, formulation):
    N, P = y.shape
    n, h = w.n_hist, w.bandwidth
    p = Q.shape[1]
    fin = np.isfinite(y)
    first = np.argmax(fin, axis=0)
    valid = fin.any(axis=0)
    c = np.where(valid, y[first, np.arange(P)], 0).astype(f32)
    last = np.zeros(P, f32)
    yt = np.empty((N, P), f32)
    for s in range(N):
        v = (y[s] + (-c)).astype(f32)
        last = np.where(fin[s], v, last).astype(f32)
        yt[s] = last
    Qf, Zf, Sf = Q.astype(f32), Z.astype(f32), S.astype(f32)
    hi = np.zeros((p, P), f32)
    lo = np.zeros((p, P), f32)
    part = np.zeros((p, P), f32)
    qpart = np.zeros(P, f32)
    wpart = np.zeros(P, f32)
    qd = np.zeros(P)
    wd = np.zeros(P)
    wstart = n - h + 1
    for s in range(n):
        part = (part + yt[s] * Qf[s][:, None]).astype(f32)
        qpart = (qpart + yt[s] * yt[s]).astype(f32)
        if s >= wstart:
            wpart = (wpart + yt[s]).astype(f32)
        if (s + 1) % 32 == 0 or s + 1 == n:
            sm = (hi + part).astype(f32)
            bb = (sm - hi).astype(f32)
            e = ((hi - (sm - bb)) + (part - bb)).astype(f32)
            hi, lo = sm, (lo + e).astype(f32)
            part[:] = 0
            qd += qpart
            wd += wpart
            qpart[:] = 0
            wpart[:] = 0
    bq = (hi + lo).astype(f32)
    rss = np.maximum(qd - (bq.astype(np.float64) ** 2).sum(0), 0).astype(f32)
    sc = (np.sqrt(rss * f32(1.0 / (n - p))) * f32(np.sqrt(n))).astype(f32)
    bsc = (sc * f32(w.crit)).astype(f32)

    def fitted(s):
        r = np.zeros(P, f32)
        for k in range(p):
            r = (r + (-bq[k]) * Zf[s, k]).astype(f32) if False else (r + (-bq[k]) * Zf[k, s]).astype(f32)
        return r

    mx = np.zeros(P, f32)
    firstb = np.zeros(P, np.int64)
    if formulation == "ring":
        res = np.empty((N, P), f32)
        for s in range(wstart, N):
            res[s] = (yt[s] + fitted(s)).astype(f32)
        acc = np.zeros(P, f32)
        for s in range(wstart, n):
            acc = (acc + res[s]).astype(f32)
        for s in range(n, N):
            old = res[s - h] if s > n else np.zeros(P, f32)
            acc = (acc + (res[s] - old)).astype(f32)
            a = np.abs(acc)
            mx = np.maximum(mx, a)
            firstb = np.where((firstb == 0) & (a > bsc), s - n + 1, firstb)
    else:
        s0 = h / R[0, 0]
        acc = (wd - s0 * (hi[0].astype(np.float64) + lo[0].astype(np.float64))).astype(f32)
        for s in range(n, N):
            old = yt[s - h] if s > n else np.zeros(P, f32)
            acc = (acc + (yt[s] - old)).astype(f32)
            num = acc
            for k in range(1, p):
                num = (num + (-bq[k]) * Sf[s - n, k]).astype(f32)
            a = np.abs(num)
            mx = np.maximum(mx, a)
            firstb = np.where((firstb == 0) & (a > bsc), s - n + 1, firstb)
    inv = np.where(sc > 0, f32(1) / sc, f32(2.0 ** 100)).astype(f32)
    return valid, firstb, (mx * inv).astype(f32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="*", default=["C1", "C4", "C5"])
    ap.add_argument("--px", type=int, default=8192)
    args = ap.parse_args()
    for name in args.workloads:
        w = WORKLOADS[name]
        t = time_axis(w)
        P = min(args.px, w.n_pixels)
        y = host_stack(P, t, w.freq, w.n_hist, w.nan_frac, seed=7, clustered=w.clustered, cols=min(P, 128))
        Q, R, Z, S = tables(t, w)
        ref = bo.monitor(y, t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit, keep_mosum=True)
        bound = boundary_values(w.n_hist, w.n_obs, w.crit)
        for form in ("ring", "wsum"):
            v, fb, mx = emulate(y, t, w, Q, R, Z, S, form)
            ok = ref.valid & v
            rel = np.abs(mx[ok] - ref.max_abs_mo[ok]) / np.maximum(np.abs(ref.max_abs_mo[ok]), 1e-30)
            mis = np.nonzero(fb != ref.first_idx)[0]
            # borderline: some |MO_j| within 1e-4 b_j of the boundary up to the later index
            border = 0
            for i in mis:
                jmax = max(fb[i], ref.first_idx[i]) or (w.n_obs - w.n_hist)
                mo = np.abs(ref.mosum[:jmax, i])
                if np.any(np.abs(mo - bound[:jmax]) <= 1e-4 * bound[:jmax]):
                    border += 1
            print(f"{name} {form:5s} px={P} max rel err {rel.max():.2e} (p99.9 {np.quantile(rel, 0.999):.2e}); "
                  f"index mismatches {len(mis)} ({border} borderline)")


if __name__ == "__main__":
    main()
