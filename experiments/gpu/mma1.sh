cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python - <<'PY'
import numpy as np, torch
from paper_1807_01751_b200.device import DevicePlan
from paper_1807_01751_b200.model import TimeAxis
from paper_1807_01751_b200.synth import WORKLOADS, device_stack, time_axis
from oracle import bfast_oracle as bo
w = WORKLOADS["C4"]; t = time_axis(w)
plan = DevicePlan(TimeAxis(t), w.freq, w.harmonics, w.n_hist, w.bandwidth, w.crit, "cuda")
print("plan", plan.info())
y = device_stack(256*64, t, w.freq, w.n_hist, w.nan_frac, seed=5, device="cuda")
res = plan.run_device(y); torch.cuda.synchronize()
ys = y.cpu().numpy()
ref = bo.monitor(ys, t, w.n_hist, w.bandwidth, w.harmonics, w.freq, w.crit, keep_mosum=True)
fi = res.first_idx.cpu().numpy(); mx = res.max_abs.cpu().numpy(); v = res.valid.cpu().numpy().astype(bool)
print("valid eq", np.array_equal(v, ref.valid), "first eq frac", (fi == ref.first_idx).mean())
rel = np.abs(mx[v] - ref.max_abs_mo[v]) / np.maximum(ref.max_abs_mo[v], 1e-30)
print("max rel err", rel.max(), "median", np.median(rel))
PY
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "not C5 and not C2" > gpurun_out/mma1_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/mma1_tests.log
WL=C4 ROUNDS=2 bash experiments/ab_env.sh "BWM_MMA=0" "-"
