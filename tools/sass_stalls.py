#!/usr/bin/env python3
"""Summarise an ncu source-page CSV (gzip): stall samples and executed counts by SASS opcode,
and the hottest instructions. usage: tools/sass_stalls.py file.csv.gz [top]"""
import csv, gzip, collections, sys
rows = list(csv.reader(gzip.open(sys.argv[1], 'rt')))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = rows[1]
cols = {h: i for i, h in enumerate(hdr)}
si, ei, so = cols['# Samples'], cols['Instructions Executed'], cols['Source']
by, ex = collections.Counter(), collections.Counter()
tot = 0
data = []
for r in rows[2:]:
    try:
        s = int(r[si])
    except Exception:
        continue
    toks = r[so].split()
    op = toks[1] if toks and toks[0].startswith('@') else (toks[0] if toks else '')
    by[op] += s
    tot += s
    try:
        ex[op] += int(r[ei])
    except Exception:
        pass
    data.append((s, r[cols['Address']][-5:], r[so].strip(), r[ei]))
print('total samples', tot)
for op, s in by.most_common(18):
    print(f'{op:30s} {100 * s / tot:5.1f}%  executed {ex[op] / 1e6:9.2f} M')
print('--- hottest instructions')
for s, ad, src, e in sorted(data, reverse=True)[:top]:
    print(f'{100 * s / tot:5.2f}% {ad} {src[:70]:70s} {e}')
