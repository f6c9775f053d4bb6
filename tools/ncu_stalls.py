"""Stall-reason totals of an ncu source page (CSV), optionally per CUDA source line.
usage: python tools/ncu_stalls.py <sass_page.csv> [<all.sass> <mangled-kernel> [top]]"""
import collections, csv, sys
sys.path.insert(0, __file__.rsplit('/', 1)[0])
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if r and r[0].startswith("0x")]
seen, uniq = set(), []
for r in data:
    a = int(r[0], 16)
    if a in seen:
        break
    seen.add(a)
    uniq.append(r)
cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
f = lambda x: float(x) if x not in ("", "-") else 0.0
tot = collections.Counter()
for r in uniq:
    for i in cols:
        tot[h[i]] += f(r[i])
T = sum(tot.values())
print("stall samples by reason:")
for k, v in tot.most_common(12):
    print(f"  {k:24s} {100 * v / T:5.1f}%")
if len(sys.argv) > 3:
    import ncu_lines
    lm = ncu_lines.line_map(sys.argv[2], sys.argv[3])
    base = int(uniq[0][0], 16)
    per = collections.defaultdict(collections.Counter)
    for r in uniq:
        ln = lm.get(int(r[0], 16) - base)
        for i in cols:
            per[ln][h[i]] += f(r[i])
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
    order = sorted(per, key=lambda l: -sum(per[l].values()))[:top]
    for ln in order:
        s = sum(per[ln].values())
        rs = ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in per[ln].most_common(3))
        print(f"line {ln}: {100 * s / T:5.1f}%  ({rs})")
