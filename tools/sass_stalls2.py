#!/usr/bin/env python3
"""Per-opcode stall-reason matrix from an ncu source-page CSV (gzip), consumer code only if a
address range is given. usage: tools/sass_stalls2.py file.csv.gz"""
import csv, gzip, collections, sys
rows = list(csv.reader(gzip.open(sys.argv[1], 'rt')))
hdr = rows[1]
cols = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
mat = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in rows[2:]:
    toks = r[cols['Source']].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    op = op.split('.')[0]
    for h in reasons:
        try: v = int(r[cols[h]])
        except Exception: v = 0
        mat[op][h] += v; tot[h] += v
allt = sum(tot.values())
top_reasons = [h for h, _ in tot.most_common(8)]
print('reason totals:', {h[6:]: round(100 * tot[h] / allt, 1) for h in top_reasons})
print(f"{'op':10s}" + ''.join(f'{h[6:]:>13s}' for h in top_reasons) + '   total%')
for op, c in sorted(mat.items(), key=lambda kv: -sum(kv[1].values()))[:12]:
    print(f'{op:10s}' + ''.join(f'{100 * c[h] / allt:13.2f}' for h in top_reasons) + f'{100 * sum(c.values()) / allt:9.2f}')
