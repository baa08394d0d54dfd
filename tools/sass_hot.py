"""Summarise an ncu source page (SASS) export: executed warp instructions by
opcode, FP64 instruction counts, and the hottest instructions by stall
samples (with average active threads).  Diagnostics for DESIGN.md / profiles/.

    ncu -i rep.ncu-rep --page source --csv --print-source sass -k regex:K > k.csv
    python tools/sass_hot.py k.csv [top]
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    col = {k: hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                     "Instructions Executed", "Avg. Threads Executed")}
    ins = []
    for r in rows[hdr_i + 1:]:
        if len(r) != len(hdr):
            continue
        try:
            n = int(r[col["Instructions Executed"]] or 0)
            st = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
            th = float(r[col["Avg. Threads Executed"]] or 0)
        except ValueError:
            continue
        src = r[col["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        ins.append((r[col["Address"]], src, op.split(".")[0], n, st, th))
    tot = sum(i[3] for i in ins)
    stall = sum(i[4] for i in ins)
    by = collections.Counter()
    thr = collections.Counter()
    for a, s, op, n, st, th in ins:
        by[op] += n
        thr[op] += n * th
    print(f"warp instructions executed: {tot:.4g}   stall samples: {stall}")
    fp64 = sum(v for k, v in by.items() if k.startswith("D") and k[:4] in
               ("DFMA", "DMUL", "DADD", "DSET", "DMNM", "DMMA"))
    print(f"FP64 (DFMA/DMUL/DADD/DSETP/DMMA) warp instructions: {fp64:.4g} "
          f"({100 * fp64 / max(tot, 1):.1f} %)")
    print("\nopcode                 warp instr      %   avg threads")
    for op, v in by.most_common(25):
        print(f"{op:20s} {v:12.4g} {100 * v / tot:6.1f} {thr[op] / max(v, 1):8.1f}")
    print(f"\ntop {top} by stall samples")
    for a, s, op, n, st, th in sorted(ins, key=lambda i: -i[4])[:top]:
        print(f"{a[-5:]} {st:7d} {n:10d} {th:5.1f}  {s[:70]}")


if __name__ == "__main__":
    main()
