"""bench.py keeps the driver's contract: one JSON line with the metric keys,
roofline / cpu_baseline / e2e / gpu_launches / clocks for our arm, and the
reference arm's line (CPU only, runs here)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().split("\n") if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "config1", "--steps", "1", "--warmup", "3", "--ref-step-s", "0.3")
    if "unavailable" in d:
        pytest.skip(d["unavailable"])
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["warmup"] >= 3


@pytest.mark.gpu
def test_our_arm_line():
    d = run_bench("--config", "config1", "--steps", "3", "--warmup", "3", "--cpu-s", "0.5", "--cpu1-s", "0.3",
                  "--e2e-steps", "2")
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] <= 1.05
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["one_thread"]["value"] > 0 and d["cpu_baseline"]["rows_bit_exact_vs_gpu"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["matches_device"] and e["pageable"]["matches_pinned"]
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["checksum_c"] == 262622  # README.md:97-99


@pytest.mark.gpu
def test_redq_arm_line():
    d = run_bench("--config", "config4", "--steps", "2", "--warmup", "3", "--no-cpu", "--e2e-steps", "1")
    assert BASE_KEYS <= set(d) and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["frac"] > 0.5 and d["e2e"]["value"] > 0


def test_default_workload_is_config5():
    """The headline is config 5 (p=3, 32768^3), the config BASELINE's
    1/2/4/8-GPU metric is quoted on."""
    sys.path.insert(0, ROOT)
    import bench

    args = bench.make_parser().parse_args([])
    assert args.config == "config5" and args.gpus == 1 and args.impl == "ours"
    assert bench.CONFIGS["config5"][:4] == (3, 32768, 32768, 32768)


@pytest.mark.gpu
def test_multi_rank_strong_scaling_functional():
    """Two ranks on one GPU over gloo (a functional check of the strong-scaling
    path: row shards of the fixed m, slot pack + all-gather of packed B, own
    slot first): C's checksum equals the single-GPU one (README.md:97-99)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29541", os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "config1",
           "--steps", "2", "--warmup", "3", "--dist-backend", "gloo", "--no-cpu", "--e2e-steps", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().split("\n") if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["config"]["m"] == 512
    assert d["checksum_c"] == 262622
    assert d["e2e"]["matches_device"] and d["e2e"]["value"] > 0  # the all-gather host path on rank 0's shard
