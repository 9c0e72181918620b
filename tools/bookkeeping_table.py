"""Bookkeeping-kernel HBM table from an ncu CSV of gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum (bench.py --profile --steps 1):
    python tools/bookkeeping_table.py gpurun_out/prof/step.csv > profiles/round1_bookkeeping_ncu.txt"""
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
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    v, u = m["gpu__time_duration.sum"]
    a[0] += 1
    a[1] += v * scale[u]
    for k, idx in (("dram__bytes_read.sum", 2), ("dram__bytes_write.sum", 3)):
        v, u = m[k]
        a[idx] += v * scale[u] / 1e6
N, q, ldb, kp = 65536, 500, 512, 512
alg = {  # algorithmic MB per launch
    "pack_eps": (N * ldb * 4 + N * ldb * 2 + N * 2 * kp * 2) / 1e6,   # beta + eps read, A hi/lo written
    "rw_center_kernel": (N * ldb * 4 + q * N * 2) / 1e6,                      # beta read, Dt written
    "EpiStoreT<__nv_bfloat16>": (N * 512 * 2 + N * ldb * 2) / 1e6,            # z read, eps written
    "prior_reweight": (N * ldb * 4) / 1e6,                                    # beta read
    # decision scalars of every row + beta/eps read and beta written for the
    # accepted rows, at the C3 acceptance rate of the profiled step (0.256)
    "rw_accept_kernel": (N * 5 * 8 + 0.256 * N * (ldb * 4 + ldb * 2 + ldb * 4)) / 1e6,
    "rw_normals_kernel": (N * 512 * 2) / 1e6,                                 # z written
}
label = {"EpiStoreT<__nv_bfloat16>": "propose GEMM (L z, TMA store)", "pack_eps": "pack_eps_rows",
         "prior_reweight": "prior_reweight_lean"}
peak = 6556.0
print("# Bookkeeping / bandwidth kernels of one C3 lambda step (bench.py --profile --steps 1, ncu")
print("# gpu__time_duration.sum + dram__bytes_read/write.sum, --clock-control none; serialised, cold cache).")
print("# GB/s = DRAM bytes / duration; alg GB/s = algorithmic bytes (DESIGN.md section 3) / duration;")
print("# % of the measured copy peak 6556 GB/s.")
print(f"{'kernel':30s} {'us':>6s} {'DRAM rd MB':>10s} {'DRAM wr MB':>10s} {'DRAM GB/s':>9s} {'alg MB':>7s} "
      f"{'alg GB/s':>8s} {'% peak':>6s}")
for name, (n, t, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    key = [k for k in alg if k in name]
    if not key:
        continue
    k = key[0]
    t, rd, wr = t / n, rd / n, wr / n
    gb = (rd + wr) / t * 1e3
    a = alg[k]
    ag = gb if a is None else a / t * 1e3
    nm = label.get(k, k.replace("_kernel", ""))
    print(f"{nm[:30]:30s} {t:6.1f} {rd:10.1f} {wr:10.1f} {gb:9.0f} {('-' if a is None else f'{a:.1f}'):>7s} "
          f"{ag:8.0f} {ag / peak * 100:6.1f}")
print()
print("# accept: algorithmic bytes are data dependent (decision scalars for all rows, beta/eps read and beta")
print("# written for the accepted rows only, at the step's acceptance rate 0.256); its beta writes stay in L2.")
print("# propose GEMM: also tensor work, the lower triangle of L only: 0.75 * 2*N*kq*kq = 25.8 GFLOP per")
print("# launch at q = 500 (0.55 of the 1385 TFLOP/s peak at 34 us).")
print("# normals: compute-bound (Philox4x32-10 + Box-Muller); its bytes are the 67 MB bf16 output.")
print("# centre pass and propose GEMM outputs stay largely in L2 (read by the next kernel): DRAM writes")
print("# are below the algorithmic bytes.")
