"""Host-side Mesh / MeshBlock model and input-file API (Python view of the C++
host library ``libpmhd_host.so``).

Mirrors the reference's core_mesh / bench_cli host types:
  MeshConfig, build_mesh
  RunConfig, parse_config
  WaveSetup / init_linear_wave SPEC.md:126-129, :218-226
  l1_error
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import native as N


class ConfigError(RuntimeError):
    """defs.hpp:36-39"""


class ParseError(RuntimeError):
    """defs.hpp:64-70: carries the 1-based line number."""

    def __init__(self, line: int, msg: str):
        super().__init__(f"parse error at line {line}: {msg}")
        self.line_number = line


class UnphysicalStateError(RuntimeError):
    """defs.hpp:51-62: stage tag and global (k, j, i) of the failing cell."""

    def __init__(self, stage: str, k: int, j: int, i: int):
        super().__init__(f"unphysical state in stage '{stage}' at cell (k={k}, j={j}, i={i})")
        self.stage_tag, self.kk, self.jj, self.ii = stage, k, j, i


def _fmt(v) -> str:
    if isinstance(v, bool):
        return "1" if v else "0"
    if isinstance(v, float):
        return repr(v)
    return str(v)


class RunConfig:
    """RunConfig parsed from ``key = value`` text; keyword
    overrides are appended as later lines (later keys override)."""

    def __init__(self, text: str = "", **overrides):
        lib = N.host_lib()
        self.c = N.RunConfigC()
        lib.pmhd_host_config_defaults(C.byref(self.c))
        lines = [text] + [f"{k} = {_fmt(v)}" for k, v in overrides.items()]
        full = "\n".join(lines)
        err_line = C.c_int(0)
        buf = C.create_string_buffer(256)
        rc = lib.pmhd_host_config_parse(full.encode(), C.byref(self.c), C.byref(err_line), buf, 256)
        if rc != N.PMHD_OK:
            raise ParseError(err_line.value, buf.value.decode())
        self.text = full

    # ---- geometry -----------------------------------------------------------
    def validate(self):
        buf = C.create_string_buffer(256)
        rc = N.host_lib().pmhd_host_validate(C.byref(self.c), buf, 256)
        if rc != N.PMHD_OK:
            raise ConfigError(buf.value.decode())

    @property
    def desc(self) -> N.MeshDesc:
        return self.c.mesh

    @property
    def dim(self) -> int:
        return 2 if self.c.mesh.nx[2] == 1 else 3

    @property
    def nblocks(self) -> int:
        return N.host_lib().pmhd_host_nblocks(C.byref(self.c))

    @property
    def block_dims(self):
        n = (C.c_int * 3)()
        N.host_lib().pmhd_host_block_dims(C.byref(self.c), n)
        return (n[0], n[1], n[2])

    @property
    def active_cells(self) -> int:
        m = self.c.mesh
        return m.nx[0] * m.nx[1] * m.nx[2]

    def block_coords(self, gid: int):
        c = (C.c_int * 3)()
        N.host_lib().pmhd_host_block_coords(C.byref(self.c), gid, c)
        return (c[0], c[1], c[2])

    def active_slices(self):
        ng = self.c.mesh.ng
        m = self.c.mesh
        ks = slice(ng, ng + m.mb[2]) if self.dim == 3 else slice(0, 1)
        return ks, slice(ng, ng + m.mb[1]), slice(ng, ng + m.mb[0])

    # ---- problem generators --------------------------------------------------
    def new_block(self) -> "BlockState":
        return BlockState.zeros(self.block_dims)

    def pgen_block(self, gid: int) -> "BlockState":
        b = self.new_block()
        rc = N.host_lib().pmhd_host_pgen_block(C.byref(self.c), gid, N.dptr(b.u), N.dptr(b.b1f),
                                               N.dptr(b.b2f), N.dptr(b.b3f))
        if rc != N.PMHD_OK:
            raise ConfigError(f"problem generator failed (code {rc})")
        return b

    def exact_block(self, gid: int, t: float) -> np.ndarray:
        n1, n2, n3 = self.block_dims
        u = np.zeros((8, n3, n2, n1))
        rc = N.host_lib().pmhd_host_exact_block(C.byref(self.c), gid, t, N.dptr(u))
        if rc != N.PMHD_OK:
            raise ConfigError("exact solution only exists for linear waves")
        return u

    def wave_eigen(self):
        lam = C.c_double()
        r = (C.c_double * 7)()
        res = C.c_double()
        rc = N.host_lib().pmhd_host_wave_eigen(C.byref(self.c), C.byref(lam), r, C.byref(res))
        if rc != N.PMHD_OK:
            raise ConfigError("no eigenmode")
        return lam.value, np.array(list(r)), res.value

    # ---- PMHD1 snapshot / restart -------------------------------
    @staticmethod
    def _ptrs(blocks, field):
        arr = (N._dp * len(blocks))(*[N.dptr(getattr(b, field)) for b in blocks])
        return arr

    def snapshot_write(self, path, blocks, t):
        """blocks: one BlockState per gid (all blocks of the mesh)."""
        rc = N.host_lib().pmhd_host_snapshot_write(
            str(path).encode(), C.byref(self.c), float(t), *[self._ptrs(blocks, f) for f in
                                                          ("u", "b1f", "b2f", "b3f")])
        if rc != N.PMHD_OK:
            raise OSError(f"snapshot write failed: {path}")

    def snapshot_read(self, path):
        """Returns (blocks, t): the active cells and faces of every block
        (ghosts zero; run exchange_ghosts after loading)."""
        blocks = [self.new_block() for _ in range(self.nblocks)]
        t = C.c_double()
        rc = N.host_lib().pmhd_host_snapshot_read(
            str(path).encode(), C.byref(self.c), C.byref(t), *[self._ptrs(blocks, f) for f in
                                                             ("u", "b1f", "b2f", "b3f")])
        if rc != N.PMHD_OK:
            raise ParseError(0, f"not a PMHD1 snapshot of this mesh: {path}")
        return blocks, t.value

    def default_tlim(self) -> float:
        return N.host_lib().pmhd_host_default_tlim(C.byref(self.c))


@dataclass
class BlockState:
    """Host copy of one MeshBlock: u (8 x n3 x n2 x n1, Array4 layout,
    array.hpp:50-80) and the staggered face arrays (array.hpp:19-48)."""

    u: np.ndarray
    b1f: np.ndarray
    b2f: np.ndarray
    b3f: np.ndarray

    @classmethod
    def zeros(cls, dims):
        n1, n2, n3 = dims
        return cls(np.zeros((8, n3, n2, n1)), np.zeros((n3, n2, n1 + 1)),
                   np.zeros((n3, n2 + 1, n1)), np.zeros((n3 + 1, n2, n1)))

    def copy(self) -> "BlockState":
        return BlockState(self.u.copy(), self.b1f.copy(), self.b2f.copy(), self.b3f.copy())


def l1_error(cfg: RunConfig, blocks, t: float):
    """l1_error: per conserved variable L1 over active cells
    against the exact linear-wave solution, plus sqrt(sum L1_q^2)."""
    ks, js, is_ = cfg.active_slices()
    tot = np.zeros(8)
    for gid, b in enumerate(blocks):
        ex = cfg.exact_block(gid, t)
        tot += np.abs(b.u[:, ks, js, is_] - ex[:, ks, js, is_]).reshape(8, -1).sum(axis=1)
    l1 = tot / cfg.active_cells
    return l1, math.sqrt(float(np.sum(l1 * l1)))
