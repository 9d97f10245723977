"""Summaries of ncu captures for profiles/ (run here, on the .ncu-rep files gpurun brings back).

    python tools/summarize_ncu.py launches gpurun_out/r1_launches.csv
    python tools/summarize_ncu.py kernel gpurun_out/r1_msed64_kernel.ncu-rep [...]
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
KEYS = [
    ("Duration (us)", "gpu__time_duration.sum", 1),
    ("DRAM read+write (MB)", ("dram__bytes_read.sum", "dram__bytes_write.sum"), 1),
    ("DRAM throughput %", "dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("L2 throughput %", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warp instr (M)", "smsp__inst_executed.sum", 1e-6),
    ("FP64 pipe %", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", 1),
    ("ALU pipe %", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("XU pipe %", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    ("tensor (UTC) busy %", "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("registers/thread", "launch__registers_per_thread", 1),
    ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    units = dict(zip(rows[0], rows[1]))
    return [dict(zip(rows[0], r), _units=units) for r in rows[2:]]


def num(d, k):
    try:
        return float(d.get(k, "nan").replace(",", "")) * UNIT.get(d["_units"].get(k, ""), 1.0)
    except ValueError:
        return float("nan")


def kernel(reps):
    print("| kernel | " + " | ".join(k for k, _, _ in KEYS) + " |")
    print("|---|" + "---|" * len(KEYS))
    for rep in reps:
        for d in raw(rep):
            vals = []
            for _, key, sc in KEYS:
                v = sum(num(d, k) for k in key) if isinstance(key, tuple) else num(d, key)
                vals.append(f"{v * sc:.1f}")
            print(f"| {d['Kernel Name'].split('(')[0][:48]} | " + " | ".join(vals) + " |")


def launches(path, steps=10):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        tot[name] += float(r[vi].replace(",", "")) / 1e3
        cnt[name] += 1
    ours = {k: v for k, v in tot.items() if k.startswith("q2::")}
    s = sum(ours.values())
    print(f"| kernel | launches | total us (all {steps} steps incl. warm-up/breakdown) | share of our kernels |")
    print("|---|---|---|---|")
    for k, v in sorted(ours.items(), key=lambda t: -t[1]):
        print(f"| {k} | {cnt[k]} | {v:.0f} | {100 * v / s:.1f}% |")


if __name__ == "__main__":
    if sys.argv[1] == "kernel":
        kernel(sys.argv[2:])
    else:
        launches(sys.argv[2])
