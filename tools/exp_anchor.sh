show() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['roofline']['kernel'], d['roofline']['kernel_ms'], d['roofline']['frac'], round(d['value']/1e12,2), d.get('checksum_c'))"; }
QG_SMALL=0 python tools/exp_anchor.py
for bk in 12 36; do
echo -n "config5 anchored kb12 bk$bk: "; QG_ANCHOR_BK=$bk python bench.py --config config5 --steps 3 --warmup 3 --no-cpu --no-e2e --kblock 12 --anchored 1 2>&1 | show
done
echo -n "config2 anchored kb28: "; python bench.py --config config2 --steps 20 --warmup 3 --no-cpu --no-e2e --kblock 28 --anchored 1 2>&1 | show
echo -n "config5 anchored kb20 (not exact in the conservative model; timing only): "; python bench.py --config config5 --steps 3 --warmup 3 --no-cpu --no-e2e --kblock 20 --anchored 1 2>&1 | show
