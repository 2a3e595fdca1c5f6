#!/usr/bin/env python
"""Print SASS with the control fields decoded (stall cycles, yield, write/read barrier, wait mask)
for a line range of `cuobjdump -sass` output.  Usage: sass_ctrl.py file.sass first_line last_line"""
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
lo, hi = int(sys.argv[2]), int(sys.argv[3])
i = lo
while i < hi:
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?)\s*/\* 0x([0-9a-f]{16}) \*/', lines[i])
    if m and i + 1 < len(lines):
        m2 = re.search(r'/\* 0x([0-9a-f]{16}) \*/', lines[i + 1])
        if m2:
            hi64 = int(m2.group(1), 16)
            ctrl = hi64 >> 41          # bits 105.. of the 128-bit word
            stall = ctrl & 0xf
            yld = (ctrl >> 4) & 1
            wbar = (ctrl >> 5) & 7
            rbar = (ctrl >> 8) & 7
            wmask = (ctrl >> 11) & 0x3f
            print(f"{m.group(1)} s{stall:2d} y{yld} w{wbar if wbar < 7 else '-'} r{rbar if rbar < 7 else '-'} "
                  f"m{wmask:06b}  {m.group(2)[:70]}")
            i += 2
            continue
    i += 1
