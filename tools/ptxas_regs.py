"""Registers / spills per kernel from build/ptxas_*.log:  python tools/ptxas_regs.py [substring]"""
import glob, re, subprocess, sys
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for f in sorted(glob.glob("build/ptxas_*.log")):
    cur = None
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
            spill = ""
        m = re.search(r"(\d+) bytes spill stores", line)
        if m and cur:
            spill = m.group(1)
        m = re.search(r"Used (\d+) registers", line)
        if m and cur and pat in cur:
            print(f"{m.group(1):>4} regs  spill {spill:>5}  {cur.replace('halp::','').replace('(halp::FgParams, int)','')}")
