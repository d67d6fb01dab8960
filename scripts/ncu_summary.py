"""Key counters of an ncu --set full report, one row per profiled launch.
    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = [("Kernel Name", "kernel"), ("Grid Size", "grid"), ("gpu__time_duration.sum", "time"),
        ("dram__bytes_read.sum", "dram rd"), ("dram__bytes_write.sum", "dram wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
        ("lts__t_sectors_srcunit_tex.sum", "L2 sectors (tex)"),
        ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %")]
cols = [(hdr.index(k), lab) for k, lab in want if k in hdr]
print("| " + " | ".join(lab for _, lab in cols) + " |")
print("|" + "---|" * len(cols))
for r in data:
    cells = []
    for i, lab in cols:
        v = r[i]
        if lab == "kernel":
            v = v.split("(")[0].replace("void ", "")
        elif units[i]:
            v = f"{v} {units[i]}"
        cells.append(v)
    print("| " + " | ".join(cells) + " |")
