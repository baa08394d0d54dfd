"""Aggregate ncu SASS-level stall samples and executed instructions by CUDA
source line, using the line table of the same build (nvdisasm -g).

    nvdisasm -g -c k.cubin > k.sass        (cuobjdump -xelf all build/k.o)
    ncu -i rep --page source --csv --print-source sass -k regex:K > k.csv
    python tools/stall_lines.py k.sass FUNCTION_MANGLED k.csv [top]
"""
import collections
import csv
import re
import sys


def line_map(sass_path, fn):
    out, cur, on = {}, None, False
    for ln in open(sass_path):
        if ln.startswith("//---------------------"):
            on = fn in ln
            continue
        if not on:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            out[int(m.group(1), 16)] = cur
    return out


def main():
    sass, fn, csvp = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    lm = line_map(sass, fn)
    rows = list(csv.reader(open(csvp)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    ci = {k: hdr.index(k) for k in ("Address", "Warp Stall Sampling (All Samples)",
                                    "Instructions Executed")}
    recs = []
    for r in rows[hi + 1:]:
        if len(r) != len(hdr):
            continue
        try:
            recs.append((int(r[ci["Address"]], 16), int(r[ci["Warp Stall Sampling (All Samples)"]] or 0),
                         int(r[ci["Instructions Executed"]] or 0)))
        except ValueError:
            pass
    base = min(a for a, _, _ in recs)
    st, ex = collections.Counter(), collections.Counter()
    for a, s, n in recs:
        key = lm.get(a - base, "?")
        st[key] += s
        ex[key] += n
    tot_s, tot_e = sum(st.values()), sum(ex.values())
    print(f"stall samples {tot_s}, warp instructions {tot_e:.3e}")
    print(f"{'line':40s} {'stall%':>7s} {'instr%':>7s}")
    for k, s in st.most_common(top):
        print(f"{k:40s} {100 * s / tot_s:7.2f} {100 * ex[k] / tot_e:7.2f}")


if __name__ == "__main__":
    main()
