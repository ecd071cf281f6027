# masked BIG with X'^T staged in shared memory (3-stage x x^T ring, 2 CTAs/SM): tests + A/B
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_masked.py tests/test_gpu_fuzz.py tests/test_capi.py -x -q -m gpu 2>&1 | tail -2
python -c "
import numpy as np
from paper_1807_01751_b200.device import DevicePlan
from paper_1807_01751_b200.model import TimeAxis
from paper_1807_01751_b200.synth import WORKLOADS, time_axis
w = WORKLOADS['C4']; t = time_axis(w)
print(DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, 'cuda', nan_mode='mask').info())"
WL=C4 NANMODE=mask ROUNDS=2 STEPS=4 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_mx0.so
