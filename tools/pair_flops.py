"""Calibrate F_pair (FP64 flops per accepted real-space pair) from an ncu
source-page (SASS) export of k_realspace: thread-level DFMA count x 2 + DMUL +
DADD, over the accepted pairs of that launch (bench line realspace_work.pairs).

    python tools/pair_flops.py k_realspace_src.csv PAIRS
"""
import csv
import sys


def main():
    path, pairs = sys.argv[1], float(sys.argv[2])
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    A, S = h.index("Address"), h.index("Source")
    N, T = h.index("Instructions Executed"), h.index("Avg. Threads Executed")
    seen = set()
    cnt = {"DFMA": 0.0, "DMUL": 0.0, "DADD": 0.0}
    for r in rows[hi + 1:]:
        if len(r) != len(h) or r[A] in seen:
            continue
        seen.add(r[A])
        toks = r[S].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.split(".")[0]
        if op in cnt:
            cnt[op] += float(r[N] or 0) * float(r[T] or 0)
    flops = 2 * cnt["DFMA"] + cnt["DMUL"] + cnt["DADD"]
    print({k: round(v / pairs, 2) for k, v in cnt.items()}, "flops/pair", round(flops / pairs, 1))


if __name__ == "__main__":
    main()
