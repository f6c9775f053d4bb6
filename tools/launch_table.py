"""ncu launch-list CSV (--metrics gpu__time_duration.sum --csv) -> markdown table of kernel shares.
usage: python tools/launch_table.py <csv> <command string> > out.md"""
import collections, csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = [r for r in csv.reader(lines) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    if r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    agg[r[ki]].append(v * scale)
solve = {k: v for k, v in agg.items() if k.startswith(("void msq::pass1", "msq::carry", "void msq::fixup", "msq::strip", "void msq::seed", "void msq::team"))}
tot = sum(sum(v) for v in solve.values())
print("# ncu launch list (cfg4 bench)\n")
print(f"Command: `{sys.argv[2]}`\n(cold-cache, serialised per launch: compare shares, not absolutes)\n")
print("| kernel | launches | mean us | share of the solve kernels |\n|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = f"{100 * sum(v) / tot:.1f}%" if k in solve else "(not a solve kernel)"
    print(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v):.1f} | {share} |")
