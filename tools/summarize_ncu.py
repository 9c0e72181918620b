"""Summarise ncu captures into profiles/ (run here, on the CPU side).

    python tools/summarize_ncu.py launches <launches.csv> <out.txt>
    python tools/summarize_ncu.py full <rep.ncu-rep> <out.txt> [--traffic-json profiles/k1_traffic.json]
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__ctas_launched.sum",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "smsp__inst_executed.sum",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki]][0] += 1
            agg[r[ki]][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list ({path}); gpu__time_duration.sum, cold-cache serialised: compare shares",
             f"# total {tot / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches", ""]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t / 1e3:10.1f} us {100 * t / tot:5.1f}%  n={n:4d}  avg={t / n / 1e3:8.1f} us  {k[:110]}")
    open(out, "w").write("\n".join(lines) + "\n")


def full(rep, out, traffic_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary of {rep}"]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        lines.append(f"\n## {name[:160]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"  {k} = {v[i]} {units[i]}")
        if traffic_json:
            rd = float(v[h.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(v[h.index("dram__bytes_write.sum")].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = rd * scale[units[h.index("dram__bytes_read.sum")]] + wr * scale[units[h.index("dram__bytes_write.sum")]]
            json.dump({"bytes_per_launch": b, "source": rep, "kernel": name[:160], "workload": "c3", "particles": 65536,
                       "note": "dram__bytes_read.sum + dram__bytes_write.sum of one K1 launch "
                               "(ncu --set full, bench.py --profile)"}, open(traffic_json, "w"), indent=1)
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        full(sys.argv[2], sys.argv[3], tj)
