#!/usr/bin/env python3
"""Static issue spacing between consecutive DMMAs (sum of stall counts) from tools/sass_ctrl.py output."""
import re, collections, sys
gaps = collections.Counter(); cur = None; n = 0; tot = 0; ninst = 0
for l in open(sys.argv[1]).read().split('\n'):
    m = re.match(r'(\w+) st\s*(\d+) y(\d) W(.) R(.) wait(\d+)\s+(.*)', l)
    if not m: continue
    st = int(m.group(2)); ins = m.group(7)
    if 'DMMA' in ins:
        if cur is not None:
            gaps[cur] += 1; n += 1; tot += cur
        cur = st
    elif cur is not None:
        cur += st; ninst += 1
print('DMMA gaps', n, 'mean', round(tot / n, 2), 'other instrs per DMMA', round(ninst / n, 2), sorted(gaps.items()))
