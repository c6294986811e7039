"""Registers / spills per K1 variant (ptxas -v of k_tma.cu; development aid)."""
import re
import subprocess
import sys

src = "paper_1912_00695_b200/csrc/k_tma.cu"
cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "--expt-relaxed-constexpr",
       "-Xptxas", "-v,-warn-spills", "-c", "-o", "/tmp/_regs.o", src] + sys.argv[1:]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
spill = {}
for line in out.splitlines():
    m = re.search(r"Registers are spilled.*k_tmaILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+).*?(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill[m.groups()[:7]] = (m.group(8), m.group(9))
    m = re.search(r"Compiling entry function '.*k_tmaILi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)ELi(\d+)", line)
    if m:
        cur = m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        sp = spill.get(cur, ("0", "0"))
        print("H=%s R1=%s T1=%s SU=%s SA=%s UNR=%s YW=%s" % cur, "regs", m.group(1), "spill st/ld", *sp)
        cur = None
for line in out.splitlines():
    if "error" in line:
        print(line)
