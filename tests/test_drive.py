"""Turbulence driving (BASELINE config 5 "driven") on the
CPU oracle: solenoidal deterministic modes, exact energy injection, zero net
momentum, decomposition independence, and a driven run staying physical.
The GPU side is checked against this in tests/test_gpu_parity.py."""
import numpy as np
import pytest

from paper_1905_04341_b200 import RunConfig
from paper_1905_04341_b200.drive import TurbulenceDriver, run_driven
from oracle.binding import OracleSolver

KW = dict(nx1=16, nx2=16, nx3=16, mb1=8, mb2=8, mb3=8, pgen="turbulence", turb_drive=1, turb_dedt=0.5,
          turb_every=2)


def totals(o, cfg):
    ks, js, is_ = cfg.active_slices()
    E, M, KE = 0.0, np.zeros(3), 0.0
    for g in range(cfg.nblocks):
        u = o.get_block(g).u[:, ks, js, is_]
        E += u[4].sum()
        M += u[1:4].reshape(3, -1).sum(1)
        KE += (0.5 * (u[1] ** 2 + u[2] ** 2 + u[3] ** 2) / u[0]).sum()
    return E, M, KE


def test_modes_solenoidal_and_deterministic():
    cfg = RunConfig(**KW)
    d = TurbulenceDriver(cfg)
    k, c, s = d.modes(3)
    assert len(k) == 16  # half space of 1 <= |k|^2 <= 4
    assert np.abs((k * c).sum(1)).max() < 1e-15 and np.abs((k * s).sum(1)).max() < 1e-15
    k2, c2, s2 = TurbulenceDriver(RunConfig(**KW)).modes(3)
    assert np.array_equal(c, c2) and np.array_equal(s, s2)
    assert not np.array_equal(c, d.modes(4)[1])  # new draw per event
    k2d, _, _ = TurbulenceDriver(RunConfig(**dict(KW, nx3=1, mb3=1))).modes(0)
    assert len(k2d) == 6 and not k2d[:, 2].any()


def test_kick_injects_energy_without_momentum():
    cfg = RunConfig(**KW)
    o = OracleSolver(cfg, workers=4)
    o.load_pgen()
    E0, M0, K0 = totals(o, cfg)
    d = TurbulenceDriver(cfg)
    de = d.energy(0.02)
    scale = d.kick(o, 0, de)
    assert scale > 0
    E1, M1, K1 = totals(o, cfg)
    assert abs((E1 - E0) - de) <= 1e-11 * de  # all of it kinetic, exactly de
    assert abs((K1 - K0) - de) <= 1e-11 * de
    # zero mean momentum up to summation rounding: ~ n_cells * eps * |m|
    assert np.abs(M1 - M0).max() <= 16**3 * 2.2e-16 * max(1.0, np.abs(M0).max())
    # ghosts were refreshed: another exchange changes nothing
    before = [o.get_block(g).u.copy() for g in range(cfg.nblocks)]
    o.exchange()
    assert all(np.array_equal(b, o.get_block(g).u) for g, b in enumerate(before))


def test_decomposition_independent():  # SPEC.md:95 (<= 1e-13 relative)
    out = []
    for mb in (16, 8):
        cfg = RunConfig(**dict(KW, mb1=mb, mb2=mb, mb3=mb))
        o = OracleSolver(cfg, workers=4)
        o.load_pgen()
        run_driven(o, cfg, 4)
        ks, js, is_ = cfg.active_slices()
        full = np.zeros((5, 16, 16, 16))
        for g in range(cfg.nblocks):
            c = cfg.block_coords(g)
            full[:, c[2] * mb:(c[2] + 1) * mb, c[1] * mb:(c[1] + 1) * mb, c[0] * mb:(c[0] + 1) * mb] = \
                o.get_block(g).u[:5, ks, js, is_]
        out.append(full)
    scale = np.abs(out[0]).reshape(5, -1).max(1)[:, None, None, None]
    assert np.abs(out[0] - out[1]).max() / 1.0 <= 1e-13 * scale.max()


def test_driven_run_grows_kinetic_energy():
    cfg = RunConfig(**dict(KW, turb_dedt=5.0))
    o = OracleSolver(cfg, workers=4)
    o.load_pgen()
    _, _, K0 = totals(o, cfg)
    t, dt, events = run_driven(o, cfg, 8)
    assert events == 4 and dt > 0
    E, M, K = totals(o, cfg)
    assert K > K0 and np.isfinite(E)
