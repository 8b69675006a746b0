"""The committed bench lines (profiles/r1_bench*.json, produced by bench.py on a
B200) carry every key of the driver's contract with consistent values; and
bench.py's static metric/config agree with BASELINE.json's north star."""

import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(path):
    with open(path) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_bench_line_contract():
    d = _last_json(os.path.join(ROOT, "profiles", "r1_bench.json"))
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "roofline", "cpu_baseline",
                "e2e", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["warmup"] >= 3 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert "workload" in d["config"] and "l2" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert abs(r["achieved"] - d["value"]) < 1e-6
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < d["value"] * 1.01  # end to end cannot beat the device-only number
    assert d["clocks"]["sm_mhz"] > 0 and not set(d["clocks"]["reasons"]) & {
        "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert d["gpu_launches"] == d["steps"] * d["config"]["launches_per_step"]


def test_reference_line_contract():
    d = _last_json(os.path.join(ROOT, "profiles", "r1_bench_reference.json"))
    assert d["impl"] == "reference"
    if "unavailable" in d:
        return
    assert d["metric"] == _last_json(os.path.join(ROOT, "profiles", "r1_bench.json"))["metric"]
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_metric_matches_baseline_json():
    import bench

    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        base = json.load(f)
    assert bench.METRIC == base["metric"]


def test_gpus_flag_spawns_ranks_gloo():
    """`bench.py --gpus 2` with no launcher re-executes itself under
    torch.distributed.run with 2 ranks (here the --dry-run plumbing: gloo
    all-reduce of the ranks, rank 0 prints the line)."""
    import subprocess
    import sys

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["rank_sum"] == 1 and d["gpus_arg"] == 2


def test_gpus_flag_mismatch_refused():
    import subprocess
    import sys

    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_gpus_flag_refused_without_devices():
    """A box with fewer GPUs than --gpus refuses loudly instead of running one
    rank and reporting n_gpus 1."""
    import subprocess
    import sys

    import torch

    if torch.cuda.device_count() >= 2:
        return
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 3 and "refusing" in out.stderr


def test_l2_clean_rotation():
    """The headline's copy rotation: within a step no launch group reads the
    same weight copy twice, and every copy is used."""
    import bench

    seen = {}
    for ki in range(len(bench.BITS)):
        for gi in range(len(bench.GROUPS)):
            c = bench.copy_index(ki, gi)
            assert (gi, c) not in seen
            seen[(gi, c)] = ki
    assert {c for _, c in seen} == set(range(bench.N_COPIES))
