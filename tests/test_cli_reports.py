"""CLI perf reports on the GPU: `pmhd report` -- the Fig. 3
analogue (acceptance 11: named regions cover >= 90 % of the
cycle and include reconstruct, riemann, ct_emf, integrate, boundary) -- and
`pmhd roofline` (cmd_roofline: self-consistent Eq. 1-3
reports)."""
import csv
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_1905_04341_b200" / "bin" / "pmhd"
pytestmark = pytest.mark.gpu


def _run(args, tmp_path):
    if not CLI.exists():
        pytest.fail("bin/pmhd missing (run __graft_entry__.build())")
    r = subprocess.run([str(CLI), *args, "--out", str(tmp_path)], cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    return r.stdout


def test_report_regions(gpu_available, tmp_path):
    out = _run(["report", "--config", "examples/linear_wave_256.in", "--cycles", "10", "--warmup", "3"],
               tmp_path)
    rows = list(csv.DictReader(open(tmp_path / "profile.csv")))
    names = [r["region"] for r in rows]
    for need in ("reconstruct", "riemann", "ct_emf", "integrate", "boundary"):
        assert need in names
    cov = float(re.search(r"regions cover ([0-9.]+) %", out).group(1))
    assert cov >= 90.0, out
    by = {r["region"]: r for r in rows}
    rie = float(by["riemann"]["time_s"])
    for r in rows:  # self-consistent derived columns
        assert float(r["time_normalized"]) == pytest.approx(float(r["time_s"]) / rie, rel=1e-5)
        if float(r["bytes"]) > 0:
            assert float(r["intensity"]) == pytest.approx(float(r["flops"]) / float(r["bytes"]), rel=1e-5)
        assert float(r["time_s"]) > 0.0
    assert float(by["riemann"]["flops"]) > float(by["reconstruct"]["flops"]) > 0


def test_roofline_report(gpu_available, tmp_path):
    out = _run(["roofline", "--config", "examples/linear_wave_64.in", "--cycles", "20",
                "--platform", "profiles/platforms.csv", "--platform-id", "b200"], tmp_path)
    lines = (tmp_path / "portability.csv").read_text().splitlines()
    assert lines[0] == "platform,space,epsilon_gflops,cap_gflops,efficiency"
    plat, space, eps, cap, e = lines[1].split(",")
    assert plat == "b200" and space == "dram"
    assert float(e) == pytest.approx(float(eps) / float(cap), rel=1e-5)  # e recomputable
    assert 0.0 < float(e) <= 1.2
    assert lines[2].split(",")[0] == "pp_metric_dram" and float(lines[2].split(",")[1]) == pytest.approx(float(e))
    roof = list(csv.DictReader(open(tmp_path / "roofline.csv")))
    ceil = [r for r in roof if r["series"] == "ceiling"]
    assert max(float(r["gflops"]) for r in ceil) == pytest.approx(36985.0)
    assert any(r["series"] == "achieved" for r in roof)
    assert "e = " in out
