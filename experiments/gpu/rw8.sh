# TMEM-ring kernel with 8 warps per CTA (512-px tiles, 2 CTAs/SM) vs 4 warps (256-px, 4 CTAs/SM):
# parity subset for the variant, then interleaved A/B at C2/C5; also the pipeline-only ablation
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
BWM_LIB=experiments/libs/libbwm_rw8.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "not masked and not tensor_core" -x -q -p no:cacheprovider 2>&1 | tail -2
BWM_LIB=experiments/libs/libbwm_rw8.so python -c "
from paper_1807_01751_b200.device import DevicePlan
from paper_1807_01751_b200.model import TimeAxis
from paper_1807_01751_b200.synth import WORKLOADS, time_axis
w = WORKLOADS['C2']; t = time_axis(w)
print(DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, 'cuda').info())"
for wl in C2 C5; do
  WL=$wl ROUNDS=3 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_rw8.so
done
