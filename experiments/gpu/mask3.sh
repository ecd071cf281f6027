# masked BIG: ring prefetch queue in pass 3; tests + C4 mask A/B + ncu
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_masked.py tests/test_gpu_fuzz.py -x -q -m gpu 2>&1 | tail -2
WL=C4 NANMODE=mask ROUNDS=2 STEPS=4 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so experiments/libs/libbwm_m2.so
timeout 900 bash profiles/run_ncu.sh r02m3 C4 "--nan-mode mask" ; python profiles/stalls.py gpurun_out/prof_r02m3_C4.ncu-rep | head -16; python profiles/source_lines.py gpurun_out/prof_r02m3_C4.ncu-rep 25
