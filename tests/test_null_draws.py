"""The null-hypothesis draws of critical_value (reference mosum.py:195-198) without a GPU: the
restatement of numpy's Philox4x64-10 + ziggurat that csrc/bwm_null.cu implements reproduces
numpy bit for bit, and the committed ziggurat tables are numpy's (tools/gen_ziggurat_tables.py).
The device side is checked against numpy in tests/test_gpu_parity.py::test_null_draws_match_numpy."""
import re
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))

import gen_ziggurat_tables as gz  # noqa: E402

HEADER = ROOT / "paper_1807_01751_b200" / "csrc" / "bwm_ziggurat_tables.h"


def _header_tables():
    text = HEADER.read_text()

    def arr(name):
        body = re.search(name + r"\[256\] = \{(.*?)\};", text, re.S).group(1)
        return [v.strip() for v in body.split(",")]

    ki = [int(v.rstrip("ull"), 16) for v in arr("kZigKi")]
    wi = [float.fromhex(v) for v in arr("kZigWi")]
    fi = [float.fromhex(v) for v in arr("kZigFi")]
    return ki, wi, fi


def test_header_tables_are_numpys():
    try:
        ki, wi, fi = gz.extract_tables()
    except Exception as e:                      # no ar/objcopy or no static library: nothing to compare
        pytest.skip(f"cannot read numpy's libnpyrandom.a: {e}")
    hki, hwi, hfi = _header_tables()
    assert hki == ki and hwi == wi and hfi == fi


@pytest.mark.parametrize("seed,rep,n", [(7, 0, 228), (7, 49999, 228), (1, 12345, 1000)])
def test_restated_stream_matches_numpy(seed, rep, n):
    ki, wi, fi = _header_tables()
    ref = np.random.Generator(np.random.Philox(key=seed, counter=rep << 128)).standard_normal(n)
    s = gz.Stream(seed, rep)
    ours = np.array([gz.standard_normal(s, ki, wi, fi) for _ in range(n)])
    assert np.array_equal(ours.view(np.uint64), ref.view(np.uint64))


def test_host_null_draws_match_reference_streams():
    """mosum.null_draws (the host restatement the GPU test compares with) is the reference's
    per-replication stream, whatever the block it is drawn in."""
    from paper_1807_01751_b200.mosum import CriticalValueRequest, null_draws

    req = CriticalValueRequest(alpha=0.05, h_frac=0.5, horizon=2.0, n_sim=100, reps=1000, seed=3)
    block = null_draws(req, 10, 14, 200)
    for j, rep in enumerate(range(10, 14)):
        ref = np.random.Generator(np.random.Philox(key=3, counter=rep << 128)).standard_normal(200)
        assert np.array_equal(block[:, j], ref)
