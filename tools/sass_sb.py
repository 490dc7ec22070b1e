"""Annotate SASS with the scoreboard fields of the control word (sm_70+ encoding):
    cuobjdump -sass obj.o | python tools/sass_sb.py <mangled-name-substring> [addr_lo addr_hi]
prints  addr  stall  wr=<barrier set by this instr>  rd=<read barrier>  wait=<barriers waited>  text"""
import re
import sys

name = sys.argv[1]
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 30
on = False
pend = None
for line in sys.stdin:
    if "Function :" in line:
        on = name in line
        continue
    if not on:
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s+(.*?);\s*/\* 0x([0-9a-f]{16}) \*/", line)
    if m:
        pend = (int(m.group(1), 16), m.group(2).strip())
        continue
    m = re.match(r"\s*/\* 0x([0-9a-f]{16}) \*/", line)
    if m and pend:
        h = int(m.group(1), 16)
        stall = (h >> 41) & 0xF
        wr = (h >> 46) & 7
        rd = (h >> 49) & 7
        wait = (h >> 52) & 0x3F
        a, txt = pend
        pend = None
        if lo <= a <= hi:
            w = ",".join(str(i) for i in range(6) if wait >> i & 1)
            print(f"{a:05x} st={stall:2d} wr={'-' if wr == 7 else wr} rd={'-' if rd == 7 else rd} wait=[{w}]  {txt[:80]}")
