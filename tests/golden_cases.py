"""Loader of the committed golden fixtures (tests/golden/*.npz, made by make_golden.py
from the reference's own outputs)."""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = ["engine_gaps", "c1", "c4_tile", "c5_tile", "edges_h10_k2", "edges_h1_k1", "edges_hn_k3",
         "odd_pixels_k8", "three_pixels", "irregular_h70", "lag_h100"]


@dataclass
class Case:
    name: str
    y: np.ndarray
    t: np.ndarray
    n: int
    h: int
    k: int
    freq: float
    crit: float
    first_break: np.ndarray
    max_abs_mo: np.ndarray
    valid: np.ndarray
    near: np.ndarray
    bound: np.ndarray
    mosum_mean: np.ndarray
    beta: np.ndarray | None
    mosum: np.ndarray | None
    info: dict

    @property
    def first_idx(self) -> np.ndarray:
        return np.where(self.first_break > 0, self.first_break - self.n, 0)


def _regenerate(info: dict, t: np.ndarray) -> np.ndarray:
    from paper_1807_01751_b200.synth import WORKLOADS, host_stack

    name = info["workload"].split()[0]
    w = WORKLOADS[name]
    P = info["shape"][1]
    clustered = w.clustered
    cols = int(round(P ** 0.5)) if clustered else None
    return host_stack(P, t, w.freq, w.n_hist, w.nan_frac, seed=info["seed"], clustered=clustered, cols=cols)


def load(name: str) -> Case:
    z = np.load(GOLDEN / f"{name}.npz")
    info = json.loads(str(z["info"]))
    t = z["t"]
    if "y" in z:
        y = z["y"]
    else:
        y = _regenerate(info, t)
    digest = hashlib.sha256(np.ascontiguousarray(y).tobytes()).hexdigest()
    if digest != info["y_sha256"]:
        raise AssertionError(f"{name}: regenerated input does not match the golden input hash")
    return Case(name, y, t, info["n"], info["h"], info["k"], info["freq"], info["crit"],
                z["first_break"].astype(np.int64), z["max_abs_mo"], z["valid"], z["near"], z["bound"],
                z["mosum_mean"], z["beta"] if "beta" in z else None, z["mosum"] if "mosum" in z else None, info)


def edge_stack(rng, N, P, n):
    y = (0.5 + 0.1 * rng.standard_normal((N, P))).astype(np.float32)
    y[:, 0] = np.nan                                  # dead pixel
    y[:3, 1] = np.nan                                 # short leading gap
    y[:17, 2] = np.nan                                # leading gap longer than a stage
    y[:40, 3] = np.nan                                # leading gap inside the history
    y[:n + 5, 4] = np.nan                             # first finite value in the monitor period
    y[-7:, 5] = np.nan                                # trailing gap
    y[10, 6], y[11, 6], y[12, 6] = np.inf, -np.inf, np.nan   # infinities count as gaps
    y[n - 3:n + 3, 7] = np.nan                        # gap across the history boundary
    y[::2, 8] = np.nan                                # every other date missing
    y[:-1, 9] = np.nan                                # only the last date finite
    y[1:, 10] = np.nan                                # only the first date finite
    mask = rng.random((N, P)) < 0.3
    mask[:, :12] = False
    y[mask] = np.nan
    return y
