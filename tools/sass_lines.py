"""Attribute an ncu SASS source page (CSV) to CUDA source lines.

    nvdisasm -g -c <cubin> > all.txt
    ncu -i rep --page source --csv --print-source sass --launch-count 1 > sass.csv
    python tools/sass_lines.py all.txt <mangled kernel> sass.csv [--outer]

Prints instructions executed per source line (innermost, or with --outer the
line in the kernel body the inlined code was called from), share of total.
"""
import csv
import re
import sys
from collections import Counter


def line_map(dis, fn, outer):
    sec = f".text.{fn}:"
    m, cur, on = {}, None, False
    for ln in open(dis):
        if ln.startswith(sec):
            on = True
            continue
        if on and ln.startswith("//----"):
            break
        if not on:
            continue
        if "//## File" in ln:
            parts = re.findall(r'File "([^"]+)", line (\d+)', ln)
            f, l = parts[-1] if outer else parts[0]
            cur = f"{f.split('/')[-1]}:{l}"
        mm = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if mm:
            m[int(mm.group(1), 16)] = (cur, mm.group(2).strip())
    return m


def main(dis, fn, sass_csv, outer=False):
    lm = line_map(dis, fn, outer)
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    ia, ie = hdr.index("Address"), hdr.index("Instructions Executed")
    data = [r for r in rows[2:] if len(r) > ie and r[ia].startswith("0x")]
    base = int(data[0][ia], 16)
    tot = Counter()
    for r in data:
        off = int(r[ia], 16) - base
        src = lm.get(off, ("?", ""))[0]
        tot[src] += int(r[ie])
    s = sum(tot.values())
    print(f"total warp instructions executed: {s}")
    for k, v in tot.most_common(45):
        print(f"{100 * v / s:6.2f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], "--outer" in sys.argv)
