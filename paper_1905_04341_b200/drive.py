"""Turbulence driving (BASELINE config 5 "driven-decaying"):
the host orchestration of one impulsive forcing event over an engine's
drive_begin / drive_energy / drive_apply (pmhd_gpu.h; the CPU oracle has the
same three calls).  Definition: include/pmhd_host.h.

Global sums are combined per block in gid order (all-gathered across ranks
when ``allgather`` is given), so one process and any decomposition produce
the same bits.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native as N


class TurbulenceDriver:
    """Impulsive solenoidal forcing: every ``cfg.turb_every`` cycles, raise
    the mean energy density by ``turb_dedt`` x (time since the last event),
    all of it kinetic, with zero net momentum.  ``kick(engine, e, de)`` takes
    de as the sum over cells of the per-cell energy change, i.e.
    turb_dedt x dt x (number of cells) (``energy(dt)``)."""

    def __init__(self, cfg):
        self.cfg = cfg
        lib = N.host_lib()
        self.ct, self.st = [], []
        for a in range(3):
            n = cfg.desc.nx[a]
            c, s = np.zeros(5 * n), np.zeros(5 * n)
            lib.pmhd_host_drive_tables(C.byref(cfg.c), a, N.dptr(c), N.dptr(s))
            self.ct.append(c)
            self.st.append(s)

    def energy(self, elapsed: float) -> float:
        """de of a kick after ``elapsed`` time: mean energy density rises by
        turb_dedt x elapsed."""
        return self.cfg.c.turb_dedt * elapsed * float(self.cfg.active_cells)

    def modes(self, event: int):
        """(k, c, s): nmode x 3 arrays of event ``event``."""
        m = N.DriveModesC()
        rc = N.host_lib().pmhd_host_drive_modes(C.byref(self.cfg.c), int(event), C.byref(m))
        if rc != N.PMHD_OK:
            raise ValueError(f"drive modes: error {rc}")
        n = m.n
        k = np.array([[m.k[q][a] for a in range(3)] for q in range(n)], dtype=np.int32)
        c = np.array([[m.c[q][a] for a in range(3)] for q in range(n)])
        s = np.array([[m.s[q][a] for a in range(3)] for q in range(n)])
        return k, c, s

    @staticmethod
    def _combine(gids, sums, allgather=None):
        rows = {g: sums[b] for b, g in enumerate(gids)}
        if allgather is not None:
            merged = {}
            for part in allgather(rows):
                merged.update(part)
            rows = merged
        tot = [0.0, 0.0, 0.0, 0.0]
        for g in sorted(rows):
            for q in range(4):
                tot[q] = tot[q] + float(rows[g][q])
        return tot

    def kick(self, engine, event: int, de: float, allgather=None):
        """One forcing event on ``engine`` (GpuSolver or OracleSolver) with
        energy ``de``.  Returns the impulse amplitude."""
        k, c, s = self.modes(event)
        tot = self._combine(engine.gids, engine.drive_begin(k, c, s, self.ct, self.st), allgather)
        mean = np.array([tot[1] / tot[0], tot[2] / tot[0], tot[3] / tot[0]])
        te = self._combine(engine.gids, engine.drive_energy(mean), allgather)
        scale = N.host_lib().pmhd_host_drive_scale(te[0], te[1], float(de))
        engine.drive_apply(mean, scale)
        return scale


def run_driven(engine, cfg, ncycles: int, dt: float = None, t: float = 0.0):
    """cmd_run loop with driving (single process): VL2 cycles, a kick every
    ``turb_every`` cycles with de = turb_dedt x elapsed time, dt recomputed
    after each kick.  Returns (t, dt, events)."""
    drv = TurbulenceDriver(cfg)
    if dt is None or dt <= 0:
        dt = engine.new_dt()
    acc, event = 0.0, 0
    for n in range(ncycles):
        dt_next, _ = engine.vl2_step(dt)
        t += dt
        acc += dt
        dt = dt_next
        if cfg.c.turb_drive and (n + 1) % cfg.c.turb_every == 0:
            drv.kick(engine, event, drv.energy(acc))
            acc = 0.0
            event += 1
            dt = engine.new_dt()
    return t, dt, event
