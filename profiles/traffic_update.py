"""Record one ncu --set full capture in profiles/traffic.json, the file bench.py reads for
roofline.traffic and roofline.tensor_pipe (per workload key: C2, C4, C5, C2-mask, ...).

    python profiles/traffic_update.py KEY gpurun_out/prof_TAG_WL.ncu-rep ALGORITHMIC_BYTES COMMIT [note]

Per launch: DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and their ratio to the
algorithmic bytes; tensor pipe and FMA pipe activity of the same kernel (the north star asks for
tensor-pipe utilisation of the contraction: fill mode runs it on FFMA2, so its tensor pipe is 0;
masked mode runs the Gram complement on tcgen05.mma kind::tf32).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    key, rep, alg, commit = sys.argv[1], sys.argv[2], float(sys.argv[3]), sys.argv[4]
    note = sys.argv[5] if len(sys.argv) > 5 else None
    hdr, units, rows = raw(rep)
    r = rows[0]

    def val(k):
        i = hdr.index(k)
        return float(r[i].replace(",", "")) * SCALE.get(units[i], 1)

    def pct(k):
        try:
            return float(r[hdr.index(k)].replace(",", "")) if k in hdr else None
        except ValueError:                     # "no data" (a pipe the kernel never used)
            return None

    dram = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    entry = {
        "dram_bytes_per_launch": int(dram),
        "algorithmic_bytes_per_launch": int(alg),
        "ratio": round(dram / alg, 4),
        "kernel": r[hdr.index("Kernel Name")],
        "kernel_ms_ncu": float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
        * {"ms": 1.0, "msecond": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}.get(
            units[hdr.index("gpu__time_duration.sum")], 1.0),
        "tensor_pipe": {
            "tensor_cycles_active_pct": pct("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
            "tensor_inst_pct": pct("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active"),
            "tensor_mem_cycles_active_pct": pct("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_cycles_active_pct": pct("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "source": "ncu --set full, same capture",
        },
        "commit": commit,
        "source": f"ncu --set full capture {rep} (dram__bytes_read + dram__bytes_write)",
    }
    if note:
        entry["note"] = note
    p = Path(__file__).with_name("traffic.json")
    d = json.loads(p.read_text()) if p.exists() else {}
    d[key] = entry
    p.write_text(json.dumps(d, indent=1) + "\n")
    print(key, json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
