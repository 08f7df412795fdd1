"""oracle/binding.py -- TEST INFRASTRUCTURE (ctypes binding of liboracle.so).

Exposes the CPU oracle with the same solver interface as the product's
``paper_1905_04341_b200.solver.GpuSolver`` so parity tests read alike.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_1905_04341_b200 import native as N
from paper_1905_04341_b200.mesh import BlockState, UnphysicalStateError, ConfigError

HERE = Path(__file__).resolve().parent
_libs = {}
_dp = C.POINTER(C.c_double)


def lib(ref: bool = False) -> C.CDLL:
    """liboracle.so, or oracle/_ref/liboracle_ref.so (the same restatement run
    through the reference's own par_for / ThreadPool) when ref=True."""
    if ref not in _libs:
        path = HERE / ("_ref/liboracle_ref.so" if ref else "liboracle.so")
        L = C.CDLL(str(path))
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_mesh_create.argtypes = [C.POINTER(N.MeshDesc), C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_mesh_create_local.argtypes = [C.POINTER(N.MeshDesc), C.c_int, C.c_int,
                                               C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)]
        L.oracle_stage_compute.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, C.POINTER(N.Status)]
        L.oracle_exchange_dir.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.oracle_halo_count.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.oracle_halo_count.restype = C.c_longlong
        L.oracle_halo_pack.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        L.oracle_halo_unpack.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, _dp]
        _ip = C.POINTER(C.c_int)
        L.oracle_drive_begin.argtypes = [C.c_void_p, C.c_int, _ip, _dp, _dp, C.POINTER(_dp), C.POINTER(_dp), _dp]
        L.oracle_drive_energy.argtypes = [C.c_void_p, _dp, _dp]
        L.oracle_drive_apply.argtypes = [C.c_void_p, _dp, C.c_double]
        L.oracle_mesh_destroy.argtypes = [C.c_void_p]
        L.oracle_mesh_destroy.restype = None
        L.oracle_set_workers.argtypes = [C.c_int]
        L.oracle_set_workers.restype = None
        L.oracle_block_dims.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
        L.oracle_nblocks.argtypes = [C.c_void_p]
        L.oracle_set_block.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp]
        L.oracle_get_block.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.oracle_exchange.argtypes = [C.c_void_p]
        L.oracle_new_dt.argtypes = [C.c_void_p, _dp, C.POINTER(N.Status)]
        L.oracle_stage.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, C.POINTER(N.Status)]
        L.oracle_vl2_step.argtypes = [C.c_void_p, C.c_double, _dp, C.POINTER(N.Status)]
        L.oracle_diag.argtypes = [C.c_void_p, C.c_int, _dp]
        L.oracle_face_data.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.oracle_emf_data.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.oracle_flops.argtypes = [_dp]
        L.oracle_flops.restype = None
        L.oracle_flops_reset.restype = None
        L.oracle_region_flops.argtypes = [_dp]
        L.oracle_region_flops.restype = None
        L.oracle_cons_to_prim.argtypes = [_dp, C.c_double, _dp]
        L.oracle_prim_to_cons.argtypes = [_dp, C.c_double, _dp]
        L.oracle_prim_to_cons.restype = None
        L.oracle_fast_speed.argtypes = [_dp, C.c_double, C.c_int]
        L.oracle_fast_speed.restype = C.c_double
        L.oracle_riemann.argtypes = [C.c_int, _dp, _dp, C.c_double, C.c_double, _dp]
        L.oracle_riemann.restype = C.c_int
        L.oracle_phys_flux.argtypes = [_dp, C.c_double, C.c_double, _dp]
        L.oracle_phys_flux.restype = None
        L.oracle_plm_slope.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int]
        L.oracle_plm_slope.restype = C.c_double
        _libs[ref] = L
    return _libs[ref]


def _arr(x):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return a, a.ctypes.data_as(_dp)


# ---- pointwise ops (golden-vector tests) ------------------------------------
def cons_to_prim(u8, gamma):
    u, pu = _arr(u8)
    w = np.zeros(8)
    rc = lib().oracle_cons_to_prim(pu, gamma, w.ctypes.data_as(_dp))
    if rc != N.PMHD_OK:
        raise UnphysicalStateError("eos", -1, -1, -1)
    return w


def prim_to_cons(w8, gamma):
    w, pw = _arr(w8)
    u = np.zeros(8)
    lib().oracle_prim_to_cons(pw, gamma, u.ctypes.data_as(_dp))
    return u


def fast_speed(w8, gamma, dim):
    w, pw = _arr(w8)
    return lib().oracle_fast_speed(pw, gamma, dim)


def riemann(solver, wl7, wr7, bx, gamma, with_fallback=False):
    a, pa = _arr(wl7)
    b, pb = _arr(wr7)
    out = np.zeros(7)
    fb = lib().oracle_riemann(N.RIEMANN[solver], pa, pb, bx, gamma, out.ctypes.data_as(_dp))
    return (out, bool(fb)) if with_fallback else out


def phys_flux(w7, bx, gamma):
    a, pa = _arr(w7)
    out = np.zeros(7)
    lib().oracle_phys_flux(pa, bx, gamma, out.ctypes.data_as(_dp))
    return out


def plm_slope(qm, q0, qp, limiter="mc"):
    return lib().oracle_plm_slope(qm, q0, qp, N.LIMITER[limiter])


def flops():
    out = np.zeros(4)
    lib().oracle_flops(out.ctypes.data_as(_dp))
    return out


def flops_reset():
    lib().oracle_flops_reset()


REGIONS = ("c2p", "reconstruct", "riemann", "ct_emf", "integrate")


def region_flops():
    """Flops per region (REGIONS order) tallied by counting meshes since the
    last flops_reset()."""
    out = np.zeros(5)
    lib().oracle_region_flops(out.ctypes.data_as(_dp))
    return out


# ---- mesh-level solver --------------------------------------------------------
class OracleSolver:
    """CPU restatement of the reference solver."""

    def __init__(self, cfg, workers: int = 1, counting: bool = False, ref: bool = False, gids=None):
        self.cfg = cfg
        self.L = lib(ref)
        self.h = C.c_void_p()
        if gids is None:
            rc = self.L.oracle_mesh_create(C.byref(cfg.desc), int(counting), int(workers), C.byref(self.h))
        else:
            arr = (C.c_int * len(gids))(*gids)
            rc = self.L.oracle_mesh_create_local(C.byref(cfg.desc), int(counting), int(workers), arr,
                                                 len(gids), C.byref(self.h))
        if rc != N.PMHD_OK:
            raise ConfigError(self.L.oracle_last_error().decode())
        self.nblocks = self.L.oracle_nblocks(self.h)
        self.gids = sorted(gids) if gids is not None else list(range(self.nblocks))

    # ---- multi-rank pieces (paper_1905_04341_b200/parallel.py) ------------------
    def stage_compute(self, s, dt):
        dn = C.c_double()
        st = N.Status()
        self._check(self.L.oracle_stage_compute(self.h, s, dt, C.byref(dn), C.byref(st)), st)
        return dn.value, st

    def stage_prefetch(self, s, dt):
        """(GPU overlap hook; nothing to do on the CPU.)"""

    def exchange_dir(self, d, half):
        self.L.oracle_exchange_dir(self.h, d, int(half))

    def halo_count(self, d, side):
        return int(self.L.oracle_halo_count(self.h, d, side))

    def alloc_halo(self, n):
        import torch
        return torch.empty(n, dtype=torch.float64)

    def halo_pack(self, gid, d, side, half, buf):
        self.L.oracle_halo_pack(self.h, gid, d, side, int(half), C.cast(buf.data_ptr(), _dp))

    def halo_unpack(self, gid, d, side, half, buf):
        self.L.oracle_halo_unpack(self.h, gid, d, side, int(half), C.cast(buf.data_ptr(), _dp))

    # ---- turbulence driving (pmhd_gpu.h drive_* semantics) -------------------
    def drive_begin(self, k, c, s, ct, st):
        sums = np.zeros((len(self.gids), 4))
        cp = (_dp * 3)(*[t.ctypes.data_as(_dp) for t in ct])
        sp = (_dp * 3)(*[t.ctypes.data_as(_dp) for t in st])
        self.L.oracle_drive_begin(self.h, len(k), k.ctypes.data_as(C.POINTER(C.c_int)), c.ctypes.data_as(_dp),
                                  s.ctypes.data_as(_dp), cp, sp, sums.ctypes.data_as(_dp))
        return sums

    def drive_energy(self, mean):
        sums = np.zeros((len(self.gids), 4))
        m = np.asarray(mean, dtype=np.float64)
        self.L.oracle_drive_energy(self.h, m.ctypes.data_as(_dp), sums.ctypes.data_as(_dp))
        return sums

    def drive_apply(self, mean, scale):
        m = np.asarray(mean, dtype=np.float64)
        self.L.oracle_drive_apply(self.h, m.ctypes.data_as(_dp), float(scale))

    def close(self):
        if self.h:
            self.L.oracle_mesh_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_block(self, gid, b: BlockState):
        self.L.oracle_set_block(self.h, gid, N.dptr(b.u), N.dptr(b.b1f), N.dptr(b.b2f), N.dptr(b.b3f))

    def get_block(self, gid, with_w=False):
        b = BlockState.zeros(self.cfg.block_dims)
        w = np.zeros_like(b.u) if with_w else None
        self.L.oracle_get_block(self.h, gid, N.dptr(b.u), N.dptr(w), N.dptr(b.b1f), N.dptr(b.b2f),
                                N.dptr(b.b3f))
        return (b, w) if with_w else b

    def load_pgen(self, exchange=True):
        for gid in self.gids:
            self.set_block(gid, self.cfg.pgen_block(gid))
        if exchange:
            self.exchange()

    def exchange(self):
        self.L.oracle_exchange(self.h)

    @staticmethod
    def _check(rc, st):
        if rc == N.PMHD_ERR_UNPHYSICAL:
            tag = {0: "init", 1: "stage1", 2: "stage2"}.get(st.stage, str(st.stage))
            raise UnphysicalStateError(tag, st.k, st.j, st.i)
        if rc != N.PMHD_OK:
            raise RuntimeError(f"oracle error {rc}")

    def new_dt(self):
        dt = C.c_double()
        st = N.Status()
        self._check(self.L.oracle_new_dt(self.h, C.byref(dt), C.byref(st)), st)
        return dt.value

    def stage(self, s, dt):
        dn = C.c_double()
        st = N.Status()
        self._check(self.L.oracle_stage(self.h, s, dt, C.byref(dn), C.byref(st)), st)
        return dn.value, st

    def vl2_step(self, dt):
        dn = C.c_double()
        st = N.Status()
        self._check(self.L.oracle_vl2_step(self.h, dt, C.byref(dn), C.byref(st)), st)
        return dn.value, st

    def diag(self, kind):
        out = np.zeros(5)
        self.L.oracle_diag(self.h, kind, out.ctypes.data_as(_dp))
        return out

    def divb_max(self):
        return float(self.diag(N.DIAG_DIVB_MAX)[0])

    def sums(self):
        return self.diag(N.DIAG_SUMS)

    def face_data(self, gid, direction):
        n1, n2, n3 = self.cfg.block_dims
        shp = [(8, n3, n2, n1 + 1), (8, n3, n2 + 1, n1), (8, n3 + 1, n2, n1)][direction]
        out = np.zeros(shp)
        self.L.oracle_face_data(self.h, gid, direction, out.ctypes.data_as(_dp))
        return out

    def emf_data(self, gid, comp):
        n1, n2, n3 = self.cfg.block_dims
        shp = [(n3 + 1, n2 + 1, n1), (n3 + 1, n2, n1 + 1), (n3, n2 + 1, n1 + 1)][comp]
        out = np.zeros(shp)
        self.L.oracle_emf_data(self.h, gid, comp, out.ctypes.data_as(_dp))
        return out

    def run(self, ncycles=None, tlim=None, dt=None):
        """cmd_run loop with the dt cap of SPEC.md:256."""
        t = 0.0
        if dt is None or dt <= 0:
            dt = self.new_dt()
        n = 0
        floors = 0
        while (ncycles is None or n < ncycles) and (tlim is None or t < tlim):
            last = False
            if tlim is not None and t + dt >= tlim:
                dt = tlim - t
                last = True
            dn, st = self.vl2_step(dt)
            floors += st.floor_count
            t = tlim if last else t + dt
            dt = dn
            n += 1
        return t, n, dt, floors
