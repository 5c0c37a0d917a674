short() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['kernel'], d['ms'], d['frac'], d['checksum'])"; }
echo -n "c3 default: "; python tools/k4_micro.py --p 3 --k 256 --m 8192 --reps 9 | short
echo -n "c3 nomem (compute on stale smem): "; QG_DEBUG_MODE=1 python tools/k4_micro.py --p 3 --k 256 --m 8192 --reps 9 | short
for s in 0 2000 3000 5000; do echo -n "c3 skew $s: "; QG_SKEW_NS=$s python tools/k4_micro.py --p 3 --k 256 --m 8192 --reps 9 | short; done
echo -n "c3 nomem skew 0: "; QG_SKEW_NS=0 QG_DEBUG_MODE=1 python tools/k4_micro.py --p 3 --k 256 --m 8192 --reps 9 | short
echo -n "c3 bk28: "; QG_TILED_SINGLE_BK=28 python tools/k4_micro.py --p 3 --k 256 --m 8192 --reps 9 | short
echo -n "c3 dyn: "; QG_DYN=1 python tools/k4_micro.py --p 3 --k 256 --m 8192 --reps 9 | short
