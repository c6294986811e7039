"""Registers / spills per K1 variant (ptxas -v of k_tma.cu; development aid)."""
import re
import subprocess
import sys

src = "paper_1912_00695_b200/csrc/k_tma.cu"
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
       "-Xptxas", "-v,-warn-spills", "-c", "-o", "/tmp/_regs.o", src] + sys.argv[1:]
out = subprocess.run(cmd, capture_output=True, text=True).stderr


def targs(line):
    m = re.search(r"k_tmaI((?:Li\d+E)+)", line)
    return tuple(re.findall(r"Li(\d+)E", m.group(1))) if m else None


cur, spill = None, {}
for line in out.splitlines():
    m = re.search(r"Registers are spilled.*?(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and targs(line):
        spill[targs(line)] = m.groups()
    if "Compiling entry function" in line:
        cur = targs(line)
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print("k_tma<" + ",".join(cur) + ">", "regs", m.group(1), "spill st/ld", *spill.get(cur, ("0", "0")))
        cur = None
for line in out.splitlines():
    if "error" in line:
        print(line)
