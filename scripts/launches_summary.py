"""Summarise an ncu launch list (gpu__time_duration.sum) of bench.py: the last complete link step
(kv_link_kernel ... logits_argmax_kernel), per-kernel totals and shares.  Usage:
    python scripts/launches_summary.py gpurun_out/launches_rN.csv > profiles/launches_rN.md"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
hdr, data = rows[h], rows[h + 1:]
K, V, U = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
G, B = hdr.index("Grid Size"), hdr.index("Block Size")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
seq = [(r[K].split("(")[0].replace("void ", ""), float(r[V].replace(",", "")) * scale[r[U]], r[G], r[B]) for r in data]
ends = [i for i, s in enumerate(seq) if s[0].startswith("pic::logits_argmax") or s[0].startswith("logits_argmax")]
# a link step starts at its a2 launch (copy path) or, for the shared-block link (no a2), at its embed
starts = [i for i, s in enumerate(seq) if "kv_link" in s[0] or "embed" in s[0]]
end = ends[-1]
start = max(i for i in starts if i < end)
if "embed" in seq[start][0] and start > 0 and "kv_link" in seq[start - 1][0]:
    start -= 1
step = seq[start:end + 1]
tot = sum(s[1] for s in step)
agg = collections.OrderedDict()
for name, us, g, b in step:
    a = agg.setdefault(name, [0, 0.0, g, b])
    a[0] += 1
    a[1] += us
print(f"# ncu launch list: one link step ({len(step)} launches, serialized cold-cache sum {tot/1e3:.3f} ms)\n")
print("| kernel | launches | total us | share | mean us | grid (last) | block |")
print("|---|---|---|---|---|---|---|")
for name, (n, us, g, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{name}` | {n} | {us:.1f} | {us/tot*100:.1f}% | {us/n:.2f} | {g} | {b} |")
