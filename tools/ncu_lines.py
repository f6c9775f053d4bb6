"""Attribute an ncu SASS source page (CSV) to CUDA source lines via nvdisasm -g.

usage: python tools/ncu_lines.py <sass_page.csv> <all.sass> <mangled-kernel-name> [top]
"""
import collections
import csv
import re
import sys


def line_map(sass_path, kernel):
    lines = open(sass_path).read().split("\n")
    start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{kernel}:"))
    cur = None
    m = {}
    for l in lines[start + 1:]:
        if l.startswith(".text.") or l.startswith("//----"):
            break
        mm = re.search(r'line (\d+)', l)
        if l.strip().startswith("//##") and mm:
            cur = int(mm.group(1))
            continue
        mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
        if mo:
            m[int(mo.group(1), 16)] = cur
    return m


def main():
    page, sass, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(page)))
    h = rows[1]
    data = [r for r in rows[2:] if r and r[0].startswith("0x")]
    # first instance only (the page may repeat per launch)
    base = int(data[0][0], 16)
    seen = set()
    uniq = []
    for r in data:
        a = int(r[0], 16)
        if a in seen:
            break
        seen.add(a)
        uniq.append(r)
    si = h.index("Warp Stall Sampling (All Samples)")
    ie = h.index("Instructions Executed")
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    lm = line_map(sass, kernel)
    st, ins = collections.Counter(), collections.Counter()
    for r in uniq:
        ln = lm.get(int(r[0], 16) - base)
        st[ln] += f(r[si])
        ins[ln] += f(r[ie])
    ts, ti = sum(st.values()), sum(ins.values())
    print(f"samples {ts:.0f} warp-instr {ti:.3e}")
    for ln, v in st.most_common(top):
        print(f"line {ln}: stall {100 * v / ts:5.1f}%  instr {100 * ins[ln] / ti:5.1f}%")


if __name__ == "__main__":
    main()


def by_instr(page, sass, kernel, top=30):
    rows = list(csv.reader(open(page)))
    h = rows[1]
    data = [r for r in rows[2:] if r and r[0].startswith("0x")]
    seen, uniq = set(), []
    for r in data:
        a = int(r[0], 16)
        if a in seen:
            break
        seen.add(a)
        uniq.append(r)
    base = int(uniq[0][0], 16)
    ie = h.index("Instructions Executed")
    f = lambda x: float(x) if x not in ("", "-") else 0.0
    lm = line_map(sass, kernel)
    ins = collections.Counter()
    for r in uniq:
        ins[lm.get(int(r[0], 16) - base)] += f(r[ie])
    tot = sum(ins.values())
    return tot, ins.most_common(top)
