"""Registers and spills per kernel from `nvcc -Xptxas -v` output (stdin): python tools/ptxas_spills.py < log"""
import re
import subprocess
import sys

txt = sys.stdin.read()
cur = None
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        try:
            cur = subprocess.run(["c++filt"], input=cur, capture_output=True, text=True).stdout.strip()
        except Exception:
            pass
        cur = re.sub(r"tod::\(anonymous namespace\)::", "", cur)
        cur = re.sub(r"\(.*", "", cur)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        st, ld = int(m.group(1)), int(m.group(2))
        spill = (st, ld)
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        flag = "SPILL %d/%d" % spill if spill != (0, 0) else ""
        print("%-60s %4s regs %s" % (cur[:60], m2.group(1), flag))
        cur = None
