"""Summarise ncu outputs for profiles/: a launch list CSV (gpu__time_duration per launch) and
`--set full` reports (.ncu-rep), into markdown tables.

  python tools/ncu_summary.py launches <launches.csv>
  python tools/ncu_summary.py full <report.ncu-rep> [<algorithmic bytes per launch> ...]
"""
import collections
import csv
import io
import subprocess
import sys

FULL_METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "ld sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "ld requests"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %peak"),
    ("smsp__inst_executed.sum", "instructions"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"]
        v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)   # -> us
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"launches: {len(data)}, total device time {tot / 1e3:.1f} ms (cold-cache, serialised)\n")
    print("| kernel | launches | total ms | share | mean ms |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k[:80]}` | {v[0]} | {v[1] / 1e3:.1f} | {100 * v[1] / tot:.1f}% | {v[1] / v[0] / 1e3:.3f} |")


def full(path, alg=None):
    out = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    cols = [(m, lab, hdr.index(m)) for m, lab in FULL_METRICS if m in hdr]
    ki = hdr.index("Kernel Name")
    print("| # | kernel | " + " | ".join(f"{lab} ({units[i]})" for _, lab, i in cols) + " | traffic / algorithmic |")
    print("|---|---|" + "---|" * len(cols) + "---|")
    for n, r in enumerate(rows[2:]):
        vals = {m: r[i] for m, _, i in cols}
        try:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(vals["dram__bytes_read.sum"]) * scale[units[hdr.index("dram__bytes_read.sum")]]
            wr = float(vals["dram__bytes_write.sum"]) * scale[units[hdr.index("dram__bytes_write.sum")]]
            ratio = f"{(rd + wr) / float(alg[n]):.3f}" if alg and n < len(alg) else "-"
        except Exception:
            ratio = "-"
        print(f"| {n} | `{r[ki][:60]}` | " + " | ".join(r[i] for _, _, i in cols) + f" | {ratio} |")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3:] or None)
