"""Summarise `build.py --force -v` ptxas output: kernel -> regs, stack, spills."""
import re, subprocess, sys
out = subprocess.run([sys.executable, "paper_2503_18974_b200/build.py", "--force", "-v"],
                     capture_output=True, text=True, cwd=sys.argv[1] if len(sys.argv) > 1 else ".")
txt = out.stdout + out.stderr
cur = None
rows = {}
for line in txt.splitlines():
    m = re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1); rows.setdefault(cur, {}); continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows[cur].update(stack=int(m.group(1)), st=int(m.group(2)), ld=int(m.group(3)))
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1); rows.setdefault(cur, {})
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows[cur]["regs"] = int(m.group(1))
import subprocess as sp
for k, v in rows.items():
    if "kernel" not in k:
        continue
    name = sp.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    print(f"{v.get('regs','?'):>4} regs {v.get('stack',0):>4} stack {v.get('st',0):>4}/{v.get('ld',0):<4} spill  {name[:110]}")
if out.returncode:
    print(txt[-3000:])
