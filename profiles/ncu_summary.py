"""Summarise an ncu --set full capture (raw page) into the numbers the roofline needs.

    python profiles/ncu_summary.py gpurun_out/prof_r01_C2.ncu-rep [bytes_per_launch_algorithmic]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "sm__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.avg.per_cycle_active",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    hdr, units, rows = load(rep)
    for r in rows:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name[:100]}")
        for k in KEYS:
            if k in hdr:
                print(f"  {k:66s} {r[hdr.index(k)]:>18s} {units[hdr.index(k)]}")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h))
                except ValueError:
                    pass
        print("  top stall reasons (warp-cycles per issued instruction):")
        for v, h in sorted(stalls, reverse=True)[:8]:
            print(f"    {h.replace('smsp__average_warp_latency_issue_stalled_', ''):50s} {v:8.3f}")
        if len(sys.argv) > 2:
            alg = float(sys.argv[2])
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
            def val(k):
                return float(r[hdr.index(k)].replace(",", "")) * scale[units[hdr.index(k)]]
            tot = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
            print(f"  dram traffic per launch = {tot:.6e} B; algorithmic = {alg:.6e} B; ratio = {tot / alg:.4f}")


if __name__ == "__main__":
    main()
