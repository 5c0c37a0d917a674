short() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['kernel'], d['ms'], d['frac'], d['checksum'])"; }
for v in $VARIANTS; do
  export QG_LIB_PATH=$PWD/paper_0803_1975_b200/_lib/var_$v/libqgemm_b200.so
  echo -n "$v c5 kb12 bk36: "; python tools/k4_micro.py --p 3 --k 32768 --kblock 12 --anchored 1 | short
  echo -n "$v c5 kb12 bk12: "; QG_ANCHOR_BK=12 python tools/k4_micro.py --p 3 --k 32768 --kblock 12 --anchored 1 | short
  echo -n "$v c2 kb28: "; python tools/k4_micro.py --p 7 --k 4096 --kblock 28 --anchored 1 | short
done
