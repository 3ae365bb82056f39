"""ptxas -v summary per kernel: python tools/ptxas_table.py <file.cu> [filter]"""
import re
import subprocess
import sys

src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
       "-Xptxas", "-v", "-c", src, "-o", "/tmp/_ptxas_table.o"]
out = subprocess.run(cmd, capture_output=True, text=True, cwd=None).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"rnnb::|LayerArgs<[^>]*>|CUtensorMap_st|\(.*\)", "", cur)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
for k, v in rows.items():
    if flt in k:
        print(f"{v.get('regs', '?'):>4} regs  spill {v.get('spill', '?'):>8}  {k}")
