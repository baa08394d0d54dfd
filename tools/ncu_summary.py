"""Summarise ncu output for profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/rNN_launches.md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep        > profiles/rNN_kernels.md

launches: per-kernel count, total and mean device time and share of the
captured launches (cold-cache, serialised by ncu: compare SHARES).
full: per-kernel duration, DRAM bytes, FP64-pipe and issue utilisation,
occupancy, top stall reasons (from `ncu -i ... --page raw --csv`).
"""
import collections
import csv
import io
import subprocess
import sys


def short(name: str) -> str:
    n = name.split("(")[0]
    for pre in ("void ", "fsecu::", "(anonymous namespace)::", "unnamed>::"):
        n = n.replace(pre, "")
    return n.split("::")[-1].lstrip("<")[:60]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                 "ms": 1.0, "second": 1e3, "s": 1e3}.get(unit, 1.0)
        a = agg[short(r[hdr.index("Kernel Name")])]
        a[0] += 1
        a[1] += v * scale
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total ms | mean ms | share |")
    print("|---|---|---|---|---|")
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {c} | {t:.3f} | {t / c:.4f} | {100 * t / tot:.1f}% |")
    print(f"| **all** | {sum(v[0] for v in agg.values())} | {tot:.3f} | | 100% |")


METRICS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("smsp__inst_executed.sum", "warp instr"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
             and h.endswith("_per_issue_active.ratio")]
    print("| kernel | " + " | ".join(m[1] for m in METRICS) + " | top stalls (cycles/issue) |")
    print("|" + "---|" * (len(METRICS) + 2))
    for r in rows[2:]:
        cells = []
        for m, _ in METRICS:
            if m not in hdr:
                cells.append("-")
                continue
            i = hdr.index(m)
            v = r[i].replace(",", "")
            try:
                f = float(v)
                u = units[i]
                if m.startswith("dram__bytes"):
                    f = f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1) / 1e9
                    cells.append(f"{f:.3f} GB")
                elif m == "gpu__time_duration.sum":
                    f = f * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3,
                             "msecond": 1.0, "ms": 1.0}.get(u, 1)
                    cells.append(f"{f:.3f}")
                else:
                    cells.append(f"{f:.3g}")
            except ValueError:
                cells.append(v)
        st = sorted(((float(r[i] or 0), hdr[i].replace("smsp__average_warps_issue_stalled_", "")
                      .replace("_per_issue_active.ratio", "")) for i in stall), reverse=True)[:3]
        cells.append(", ".join(f"{n} {v:.2f}" for v, n in st))
        print(f"| {short(r[ki])} | " + " | ".join(cells) + " |")


STAGE_OF = {"k_spread": "spread", "k_gather_mma": "gather", "k_gather_tma": "gather",
            "k_realspace": "realspace",
            "k_xscale": "kscale", "k_xscale2": "kscale"}


def traffic(path):
    """profiles/traffic.json: dram read+write bytes per launch by bench stage name."""
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    res = {}
    for r in rows[2:]:
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            tot += float(r[i].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                   "Gbyte": 1e9}.get(units[i], 1)
        name = short(r[ki]).split("<")[0]
        if name in STAGE_OF:
            res[STAGE_OF[name]] = tot
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](sys.argv[2])
