"""Registers / spills per kernel from csrc/build.log:
python tools/ptxas_regs.py [substring]"""
import re
import subprocess
import sys

log = open(sys.argv[2] if len(sys.argv) > 2 else "paper_1507_02557_b200/csrc/build.log").read().splitlines()
want = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
for i, l in enumerate(log):
    m = re.search(r"Compiling entry function '([^']+)'", l)
    if m:
        cur = m.group(1)
        continue
    if cur and "Used" in l and "registers" in l:
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        spill = log[i - 1] if "spill" in log[i - 1] else ""
        sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", spill)
        if want in name:
            regs = re.search(r"Used (\d+) registers", l).group(1)
            print(f"{regs:>4} regs  spill {sp.groups() if sp else '-'}  {name.split('(')[0]}")
        cur = None
