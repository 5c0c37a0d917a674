# Start-skew sweep (clock spin vs nanosleep) on the contraction alone (tools/k4_micro.py).
short() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['kernel'], d['ms'], d['frac'])"; }
for rep in 1 2; do
for s in 0 2000 3000 3400 4000 5000 6800; do
  echo -n "c3 spin $s: "; QG_SKEW_NS=$s python tools/k4_micro.py --p 3 --k 256 --m 8192 --reps 9 | short
done
echo -n "c3 sleep 4000: "; QG_SKEW_SLEEP=1 python tools/k4_micro.py --p 3 --k 256 --m 8192 --reps 9 | short
done
for s in 0 4000; do
  echo -n "c5 spin $s: "; QG_SKEW_NS=$s python tools/k4_micro.py --p 3 --k 32768 | short
  echo -n "c2 spin $s: "; QG_SKEW_NS=$s python tools/k4_micro.py --p 7 --k 4096 | short
done
echo -n "c5 sleep 4000: "; QG_SKEW_SLEEP=1 python tools/k4_micro.py --p 3 --k 32768 | short
echo -n "c2 sleep 4000: "; QG_SKEW_SLEEP=1 python tools/k4_micro.py --p 7 --k 4096 | short
