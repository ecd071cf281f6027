# C4: fractional evict_last on re-read rows (createpolicy.fractional), A/B + DRAM bytes per variant
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
L=experiments/libs
WL=C4 ROUNDS=2 bash experiments/ab_libs.sh paper_1807_01751_b200/libbwm.so $L/libbwm_f25.so $L/libbwm_f50.so $L/libbwm_f75.so $L/libbwm_h1f50.so
for lib in paper_1807_01751_b200/libbwm.so $L/libbwm_f25.so $L/libbwm_f50.so $L/libbwm_f75.so $L/libbwm_h1f50.so; do
  BWM_LIB=$lib timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:monitor_kernel_tma -s 3 -c 1 python bench.py --workload C4 --steps 2 --warmup 2 --no-e2e --no-cpu 2>&1 | grep -E "dram__bytes|gpu__time|hit_rate" | sed "s|^|$lib |"
done
