short() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().split('\n')[-1]); print(d['kernel'], d['kblock'], d['ms'], d['frac'], d['checksum'])"; }
for v in $VARIANTS; do
  export QG_LIB_PATH=$PWD/paper_0803_1975_b200/_lib/var_$v/libqgemm_b200.so
  echo -n "$v c5: "; python tools/k4_micro.py --p 3 --k 32768 | short
  echo -n "$v c2: "; python tools/k4_micro.py --p 7 --k 4096 | short
  echo -n "$v p5 k=20000: "; python tools/k4_micro.py --p 5 --k 20000 | short
done
