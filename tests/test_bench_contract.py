"""bench.py JSON-line contract: the reference arm on CPU (small bounded
sample) and, on a GPU, our arm at a small size (the keys the driver reads)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config"}


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("workload", ["m4", "m5"])
def test_reference_arm_line(workload):
    extra = ["--size", "32"] if workload == "m4" else []
    d = run_bench("--impl", "reference", "--workload", workload, *extra, "--steps", "1", "--warmup", "0")
    assert BASE <= set(d)
    assert d["scaling"] == ("weak" if workload == "m4" else "strong")
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["dtype"] == "f64" and d["config"]["workload"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line(gpu_available):
    d = run_bench("--size", "64", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert BASE <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0 < r["frac"] < 1 and r["achieved"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] < d["value"]  # host copies inside the timed region
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_weak_scaling_rank_grid():
    """bench.py's M4 decomposition is SURVEY.md §8d's (p1,p2,p3) rank grid,
    one n^3 block per rank; M5 splits its 64 blocks into equal bricks."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_1905_04341_b200.parallel import plan_for
    for ranks, grid in [(1, [1, 1, 1]), (2, [2, 1, 1]), (4, [2, 2, 1]), (8, [2, 2, 2])]:
        assert bench.rank_grid(ranks) == grid
        cfg = bench.make_config(64, ranks)
        assert list(cfg.desc.nx) == [64 * g for g in grid] and cfg.nblocks == ranks
        plan = plan_for(cfg, ranks)
        assert sorted(g for r in range(ranks) for g in plan.local_gids(r)) == list(range(ranks))
        assert all(len(plan.local_gids(r)) == 1 for r in range(ranks))
        m5 = bench.make_m5_config()
        p5 = plan_for(m5, ranks)
        assert all(len(p5.local_gids(r)) == 64 // ranks for r in range(ranks))
