"""Per-kernel table (time, DRAM bytes, achieved GB/s) from an ncu CSV of
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per, names = collections.defaultdict(dict), {}
for r in rows[hi + 1:]:
    if len(r) > vi:
        per[r[ii]][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
        names[r[ii]] = r[ki]
sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i][:70]]
    a[0] += 1
    a[1] += m["gpu__time_duration.sum"][0] / 1e3
    a[2] += m["dram__bytes_read.sum"][0] * sc[m["dram__bytes_read.sum"][1]]
    a[3] += m["dram__bytes_write.sum"][0] * sc[m["dram__bytes_write.sum"][1]]
tot = sum(a[1] for a in agg.values())
print(f"{'us':>8} {'%':>5} {'n':>3} {'avg us':>8} {'rd MB':>7} {'wr MB':>7} {'GB/s':>7}  kernel")
for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{a[1]:8.1f} {100 * a[1] / tot:5.1f} {a[0]:3d} {a[1] / a[0]:8.1f} {a[2] / a[0] / 1e6:7.1f} {a[3] / a[0] / 1e6:7.1f} "
          f"{(a[2] + a[3]) / (a[1] * 1e-6) / 1e9:7.0f}  {n}")
