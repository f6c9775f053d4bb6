"""Attribute LDL/STL in one kernel of libmsq.so to source lines (needs -lineinfo).
usage: python tools/local_mem_lines.py <mangled-kernel-substring>"""
import collections, glob, os, re, subprocess, sys, tempfile
lib = os.path.join(os.path.dirname(__file__), "..", "paper_2503_18974_b200", "_lib", "libmsq.so")
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True, check=True)
cub = glob.glob(os.path.join(d, "*.cubin"))[0]
txt = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
want = sys.argv[1]
cur_fn = None; cur = None; c = collections.Counter(); n = 0
for line in txt.splitlines():
    m = re.match(r"\.text\.(\S+):", line)
    if m:
        cur_fn = m.group(1); continue
    if cur_fn is None or want not in cur_fn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
    if re.search(r"\b(LDL|STL)", line):
        c[cur] += 1; n += 1
print("total LDL/STL:", n)
for k, v in c.most_common(25):
    print(v, k)
