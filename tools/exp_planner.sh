# Planner check: the chosen plan (anchored where picked) against the best FP64-flush plan, contraction alone.
short() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['kernel'], 't',d['t'],'e',d['e'],'kb',d['kblock'], d['ms'], 'eff_T', d['eff_T'])"; }
for pk in "5 20000" "11 20000" "13 20000" "31 20000" "2 32768" "7 20000" "3 6000" "17 50000"; do
  set -- $pk
  echo -n "p=$1 k=$2 planner: "; timeout 120 python tools/k4_micro.py --p $1 --k $2 | short
  echo -n "p=$1 k=$2 no-anchor: "; timeout 120 python tools/k4_micro.py --p $1 --k $2 --anchored 0 --plain 1 | short
done
