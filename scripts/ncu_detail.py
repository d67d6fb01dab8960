"""Detailed counters of every launch in an ncu --set full report (issue, pipes, stalls, DRAM, tensor).
    python scripts/ncu_detail.py gpurun_out/x.ncu-rep [algorithmic_bytes_per_launch]"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
want = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
stalls = [k for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")]
for r in data:
    print(f"## {r[hdr.index('Kernel Name')].split('(')[0]}\n")
    print("| counter | value |\n|---|---|")
    for k in want:
        if k in hdr:
            print(f"| {k} | {r[hdr.index(k)]} {units[hdr.index(k)]} |")
    if alg and "dram__bytes_read.sum" in hdr:
        def mb(k):
            v = float(r[hdr.index(k)].replace(",", ""))
            u = units[hdr.index(k)]
            return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
        t = mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum")
        print(f"| DRAM bytes / algorithmic | {t:.1f} MB / {alg / 1e6:.1f} MB = {t / (alg / 1e6):.2f} |")
    top = sorted(((float(r[hdr.index(k)] or 0), k) for k in stalls), reverse=True)[:8]
    print("\nTop stall reasons (warps per issue-active cycle): " +
          ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} "
                    f"{v:.2f}" for v, k in top) + "\n")
