"""Registers / spill stores per fft_line_kernel variant from a ptxas -v log
(development tool)."""
import re, sys

cur = sp = None
for l in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '_ZN[^']*?(\w+?kernel)I([^']*)'", l)
    if m:
        cur = m.group(1) + "<" + m.group(2)[:40] + ">"
        continue
    if cur and "spill" in l:
        sp = re.search(r"(\d+) bytes spill stores", l).group(1)
    if cur and "Used" in l:
        r = re.search(r"Used (\d+) registers", l).group(1)
        print(f"{cur:60s} regs {r:>4s} spill {sp}")
        cur = None
