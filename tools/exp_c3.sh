short() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['kernel'], d['t'], d['e'], d['kblock'], d['ms'], d['frac'], d['eff_T'], d['checksum'])"; }
echo -n "c3 default: "; python tools/k4_micro.py --p 3 --k 256 --m 8192 --reps 9 | short
echo -n "c3 anchored t8 e6 kb12: "; python tools/k4_micro.py --p 3 --k 256 --m 8192 --t 8 --e 6 --kblock 12 --anchored 1 --reps 9 | short
echo -n "c3 anchored t10 e5 kb20: "; python tools/k4_micro.py --p 3 --k 256 --m 8192 --t 10 --e 5 --kblock 20 --anchored 1 --reps 9 | short
echo -n "c3 t8 e6 kb20 fp64 flush: "; python tools/k4_micro.py --p 3 --k 256 --m 8192 --t 8 --e 6 --kblock 20 --anchored 0 --reps 9 | short
