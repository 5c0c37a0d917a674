#!/usr/bin/env python3
"""From tools/sass_ctrl.py output: for every non-DMMA instruction that waits on a scoreboard last set
by a DMMA, the distance (in DMMAs issued) to that DMMA — small distances are warps waiting out the
DMMA latency. usage: tools/sass_sbdist.py ctrl.txt"""
import re, collections, sys
recs = []
for l in open(sys.argv[1]).read().split('\n'):
    m = re.match(r'(\w+) st\s*(\d+) y(\d) W(.) R(.) wait(\d+)\s+(.*)', l)
    if m:
        recs.append((m.group(1), int(m.group(2)), m.group(4), m.group(5), m.group(6), m.group(7)))
idx = [i for i, r in enumerate(recs) if 'DMMA' in r[5]]
lo, hi = idx[0], idx[-1]
last_set, dcount = {}, 0
dist = collections.Counter()
for i in range(lo, hi + 1):
    a, st, w, rb, wait, ins = recs[i]
    if 'DMMA' in ins:
        dcount += 1
    for b in range(6):
        if wait[5 - b] == '1' and b in last_set and 'DMMA' not in ins and 'DMMA' in last_set[b][1]:
            dist[(ins.split()[0].split('.')[0] + last_set[b][1][-4:], min(dcount - last_set[b][0], 20))] += 1
    if w != '-':
        last_set[int(w)] = (dcount, ins + ' [W]')
    if rb != '-':
        last_set[int(rb)] = (dcount, ins + ' [R]')
ops = sorted({k[0] for k in dist})
for op in ops:
    print(op, {d: c for (o, d), c in sorted(dist.items()) if o == op})
