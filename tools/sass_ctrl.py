#!/usr/bin/env python3
"""Decode the scheduling control fields of cuobjdump -sass output (sm_70+ 128-bit encoding):
stall count, yield, write/read barrier index, wait mask. usage: cuobjdump -sass x.o | tools/sass_ctrl.py [regex]"""
import re, sys
pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
lines = sys.stdin.read().split('\n')
i = 0
out = []
while i < len(lines):
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]{16}) \*/', lines[i])
    if m and i + 1 < len(lines):
        m2 = re.match(r'\s*/\* (0x[0-9a-f]{16}) \*/', lines[i + 1])
        if m2:
            hi = int(m2.group(1), 16)
            ctrl = hi >> 41
            stall = ctrl & 0xf
            yld = (ctrl >> 4) & 1
            wbar = (ctrl >> 5) & 7
            rbar = (ctrl >> 8) & 7
            wait = (ctrl >> 11) & 0x3f
            out.append((m.group(1), m.group(2).strip(), stall, yld, wbar, rbar, wait))
            i += 2
            continue
    i += 1
for a, ins, stall, yld, wbar, rbar, wait in out:
    if pat and not pat.search(ins):
        continue
    wb = '-' if wbar == 7 else str(wbar)
    rb = '-' if rbar == 7 else str(rbar)
    print(f'{a} st{stall:2d} y{yld} W{wb} R{rb} wait{wait:06b}  {ins[:80]}')
