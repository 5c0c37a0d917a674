# One bench line per BASELINE config (and the config-4 left/full variants)
# into gpurun_out/bench_<config>.json; config 5 runs the full 32768^3 product.
set -u
mkdir -p gpurun_out
for c in config1 config2 config3 config4 config4_left config4_full; do
  python bench.py --config $c --steps 20 --warmup 5 --cpu-s 4 2>/dev/null | tail -1 > gpurun_out/bench_$c.json
done
python bench.py --config config2 --output cc --steps 20 --warmup 5 --no-cpu 2>/dev/null | tail -1 > gpurun_out/bench_config2_cc.json
python bench.py --config config5 --steps 20 --warmup 5 --cpu-s 4 2>/dev/null | tail -1 > gpurun_out/bench_config5.json
for c in config1 config2 config2_cc config3 config4 config4_left config4_full config5; do
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/bench_{c}.json"))
except Exception as ex:
    print(c, "FAILED", ex); sys.exit(0)
e2e = d.get("e2e", {}).get("value")
cpu = d.get("cpu_baseline", {}).get("value")
print(c, round(d["ms_per_step"], 4), "ms", round(d["value"] / 1e12, 2), "T/s", "frac", d["roofline"]["frac"],
      "e2e", e2e and round(e2e / 1e12, 2), "cpu", cpu and round(cpu / 1e9, 2), d.get("clocks", {}).get("reasons"))
PY
done
