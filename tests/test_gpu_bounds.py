"""Bounds-checked debug build (lib/test/libpmhd_gpu_check.so, -DPMHD_BOUNDS_CHECK):
every element index the fused kernels, the x1 ghost push and the exchange
form must lie inside its block array, else the kernel traps (the GPU pool has
no compute-sanitizer).  Runs the edge-case meshes through it in a subprocess
and checks the results against the oracle as well."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1905_04341_b200", "lib", "test", "libpmhd_gpu_check.so")

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np
from paper_1905_04341_b200 import RunConfig
from paper_1905_04341_b200.solver import GpuSolver
from oracle.binding import OracleSolver
sys.path.insert(0, {root!r} + '/tests')
from test_gpu_parity import CASES
names = ["wave3d_tiny_blocks", "wave3d_ng3_ragged", "wave3d_ng4_8blk", "ot2d_ragged", "blast3d_8blk_floor",
         "turb3d"]
for name in names:
    kw, ncyc = CASES[name]
    cfg = RunConfig(**kw)
    o, g = OracleSolver(cfg, workers=4), GpuSolver(cfg)
    assert g.build_info.endswith("+bounds-check"), g.build_info
    o.load_pgen(); g.load_pgen()
    dt = o.new_dt()
    for _ in range(min(ncyc, 3)):
        dn, _ = o.vl2_step(dt)
        g.vl2_step(dt)
        dt = dn
    ks, js, is_ = cfg.active_slices()
    for gid in range(cfg.nblocks):
        a, b = o.get_block(gid).u, g.get_block(gid).u
        s = np.maximum(np.abs(a).max(axis=(1, 2, 3), keepdims=True), 1e-300)
        assert np.max(np.abs(a - b) / s) <= 1e-11, (name, gid)
    print("ok", name, flush=True)
"""


# the default kernel selection, then the round-2 alternatives forced on these
# small meshes: column / row march flux kernels, the x1 + x2 kernel, and the
# TMA-staged, warp-specialised and two-kernel update forms
VARIANTS = {
    "default": {},
    "march": {"PMHD_FLUX_MARCH": "2", "PMHD_FLUX_MARCH_X1": "1", "PMHD_FLUX_MARCH_STAGES": "3"},
    "xy_tma": {"PMHD_FLUX_XY": "1", "PMHD_UPDATE": "tma"},
    "march_ws": {"PMHD_FLUX_MARCH": "2", "PMHD_FLUX_MARCH_STAGES": "3", "PMHD_UPDATE": "ws"},
    # the two-kernel update (edge EMFs + cell update), the default on meshes
    # that fill the GPU, forced here
    "march_emf": {"PMHD_FLUX_MARCH": "2", "PMHD_FLUX_MARCH_STAGES": "3", "PMHD_UPDATE": "emf"},
}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", list(VARIANTS))
def test_bounds_checked_build(gpu_available, variant):
    assert os.path.exists(LIB), "build it: make testlib"
    env = dict(os.environ, PMHD_GPU_LIB=LIB, **VARIANTS[variant])
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert r.stdout.count("ok ") == 6
