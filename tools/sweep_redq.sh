# timing sweep of the blocked REDQ contraction (config 4 shape); debug bit 3 skips the in-place REDQ
run() { echo "== $*"; env "$@" python bench.py --config ${CFG:-config4} --steps 10 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['checksum_c'])"; }
run QG_DEBUG_MODE=0
run QG_DEBUG_MODE=8
run QG_SKEW_NS=0
run QG_SKEW_NS=8000
CFG=config4_left run QG_DEBUG_MODE=0
CFG=config4_full run QG_DEBUG_MODE=0
