"""GpuSolver -- the reference's solver ops over the CUDA C-ABI.

Same method set as the reference's CPU solver that cmd_run / cmd_bench /
cmd_scale drive: vl2_step, exchange_ghosts, compute_dt,
max_divergence_b, conservation sums.  Every call goes through
``libpmhd_gpu.so`` (include/pmhd_gpu.h); there is no CPU fallback -- a
missing library or device raises.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import native as N
from .mesh import BlockState, ConfigError, UnphysicalStateError

_TAG = {0: "init", 1: "stage1", 2: "stage2"}


class CudaError(RuntimeError):
    pass


class GpuSolver:
    def __init__(self, cfg, device: int = 0, parity: bool = False, gids=None):
        self.cfg = cfg
        self.device = device
        self.L = N.gpu_lib(parity)
        if self.L.pmhd_gpu_abi_version() != 1:
            raise CudaError("ABI version mismatch")
        self.ctx = C.c_void_p()
        rc = self.L.pmhd_gpu_ctx_create(device, C.byref(self.ctx))
        if rc != N.PMHD_OK:
            raise CudaError(f"pmhd_gpu_ctx_create failed (code {rc}): no usable sm_100 device")
        self.mesh = C.c_void_p()
        if gids is None:
            rc = self.L.pmhd_gpu_mesh_create(self.ctx, C.byref(cfg.desc), None, 0, C.byref(self.mesh))
            self.gids = list(range(cfg.nblocks))
        else:
            arr = (C.c_int * len(gids))(*gids)
            rc = self.L.pmhd_gpu_mesh_create(self.ctx, C.byref(cfg.desc), arr, len(gids), C.byref(self.mesh))
            self.gids = list(gids)
        self._check(rc)

    @property
    def stream_handle(self) -> int:
        """cudaStream_t of the context (for torch.cuda.ExternalStream events)."""
        return int(self.L.pmhd_gpu_stream(self.ctx) or 0)

    @property
    def build_info(self) -> str:
        return self.L.pmhd_gpu_build_info().decode()

    def _err(self) -> str:
        return self.L.pmhd_gpu_last_error(self.ctx).decode()

    def _check(self, rc, st=None):
        if rc == N.PMHD_OK:
            return
        if rc == N.PMHD_ERR_UNPHYSICAL and st is not None:
            raise UnphysicalStateError(_TAG.get(st.stage, str(st.stage)), st.k, st.j, st.i)
        if rc == N.PMHD_ERR_CONFIG:
            raise ConfigError(self._err())
        raise CudaError(f"pmhd_gpu error {rc}: {self._err()}")

    def close(self):
        if getattr(self, "mesh", None):
            self.L.pmhd_gpu_mesh_destroy(self.mesh)
            self.mesh = C.c_void_p()
        if getattr(self, "ctx", None):
            self.L.pmhd_gpu_ctx_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state -------------------------------------------------------------------
    def set_block(self, gid, b: BlockState):
        self._check(self.L.pmhd_gpu_upload_block(self.mesh, gid, N.dptr(b.u), N.dptr(b.b1f),
                                                 N.dptr(b.b2f), N.dptr(b.b3f)))

    def get_block(self, gid, with_w=False, out: BlockState = None):
        """Download block gid (Bcc re-derived from the faces).  out: an
        existing BlockState to fill (e.g. pinned host buffers)."""
        b = BlockState.zeros(self.cfg.block_dims) if out is None else out
        w = np.zeros_like(b.u) if with_w else None
        self._check(self.L.pmhd_gpu_download_block(self.mesh, gid, N.dptr(b.u), N.dptr(w),
                                                   N.dptr(b.b1f), N.dptr(b.b2f), N.dptr(b.b3f)))
        return (b, w) if with_w else b

    def load_pgen(self, exchange=True):
        for gid in self.gids:
            self.set_block(gid, self.cfg.pgen_block(gid))
        if exchange:
            self.exchange()

    # ---- reference ops -------------------------------------------------------------
    def exchange(self):
        self._check(self.L.pmhd_gpu_exchange(self.mesh))

    def new_dt(self):
        dt = C.c_double()
        st = N.Status()
        self._check(self.L.pmhd_gpu_new_dt(self.mesh, C.byref(dt), C.byref(st)), st)
        return dt.value

    def stage(self, s, dt):
        dn = C.c_double()
        st = N.Status()
        self._check(self.L.pmhd_gpu_stage(self.mesh, s, dt, C.byref(dn), C.byref(st)), st)
        return dn.value, st

    def vl2_step(self, dt):
        dn = C.c_double()
        st = N.Status()
        self._check(self.L.pmhd_gpu_vl2_step(self.mesh, dt, C.byref(dn), C.byref(st)), st)
        return dn.value, st

    def run(self, ncycles=None, tlim=None, dt=None):
        t = C.c_double(0.0)
        d = C.c_double(dt if dt else 0.0)
        n = C.c_int(0)
        st = N.Status()
        rc = self.L.pmhd_gpu_run(self.mesh, -1 if ncycles is None else int(ncycles),
                                 0.0 if tlim is None else float(tlim), C.byref(t), C.byref(d),
                                 C.byref(n), C.byref(st))
        self._check(rc, st)
        return t.value, n.value, d.value, st.floor_count

    def divb_max(self):
        out = np.zeros(5)
        self._check(self.L.pmhd_gpu_diag(self.mesh, N.DIAG_DIVB_MAX, N.dptr(out)))
        return float(out[0])

    def sums(self):
        out = np.zeros(5)
        self._check(self.L.pmhd_gpu_diag(self.mesh, N.DIAG_SUMS, N.dptr(out)))
        return out

    # ---- multi-rank pieces (parallel.py) ---------------------------------------
    def stage_compute(self, s, dt):
        dn = C.c_double()
        st = N.Status()
        self._check(self.L.pmhd_gpu_stage_compute(self.mesh, s, dt, C.byref(dn), C.byref(st)), st)
        return dn.value, st

    # ---- peer-memory halo (pmhd_gpu.h peer_attach) ---------------------------
    def slab(self):
        """(device base address, 64-byte CUDA IPC handle) of this mesh's state slab."""
        base = C.c_void_p()
        h = C.create_string_buffer(64)
        self._check(self.L.pmhd_gpu_slab(self.mesh, C.byref(base), h))
        return base.value, h.raw

    def ipc_open(self, handle: bytes) -> int:
        base = C.c_void_p()
        self._check(self.L.pmhd_gpu_ipc_open(self.ctx, C.create_string_buffer(handle, 64), C.byref(base)))
        return base.value

    def ipc_close(self, base: int):
        self._check(self.L.pmhd_gpu_ipc_close(self.ctx, C.c_void_p(base)))

    def peer_attach(self, owners, bases):
        """owners[gid] = rank; bases[rank] = that rank's slab as mapped here (None: unmapped)."""
        own = (C.c_int * len(owners))(*owners)
        arr = (C.c_void_p * len(bases))(*[C.c_void_p(b) if b else None for b in bases])
        self._check(self.L.pmhd_gpu_peer_attach(self.mesh, len(bases), own, arr))

    def stage_prefetch(self, s, dt):
        """Stage s's interior flux tiles, overlapping the coming exchange."""
        self._check(self.L.pmhd_gpu_stage_prefetch(self.mesh, s, dt))

    def exchange_dir(self, d, half):
        self._check(self.L.pmhd_gpu_exchange_dir(self.mesh, d, int(half)))

    def halo_count(self, d, side):
        n = C.c_longlong()
        self._check(self.L.pmhd_gpu_halo_count(self.mesh, d, side, C.byref(n)))
        return n.value

    def alloc_halo(self, n):
        import torch
        return torch.empty(n, dtype=torch.float64, device=f"cuda:{self.device}")

    def halo_pack(self, gid, d, side, half, buf):
        self._check(self.L.pmhd_gpu_halo_pack(self.mesh, gid, d, side, int(half), C.c_void_p(buf.data_ptr())))

    # ---- turbulence driving (pmhd_gpu.h drive_*; orchestration in drive.py) ----
    def drive_begin(self, k, c, s, ct, st):
        import numpy as np
        sums = np.zeros((len(self.gids), 4))
        cp = (N._dp * 3)(*[N.dptr(t) for t in ct])
        sp = (N._dp * 3)(*[N.dptr(t) for t in st])
        self._check(self.L.pmhd_gpu_drive_begin(self.mesh, len(k), k.ctypes.data_as(N._ip), N.dptr(c),
                                                N.dptr(s), cp, sp, N.dptr(sums)))
        return sums

    def drive_energy(self, mean):
        import numpy as np
        sums = np.zeros((len(self.gids), 4))
        self._check(self.L.pmhd_gpu_drive_energy(self.mesh, N.dptr(np.asarray(mean, dtype=np.float64)),
                                                 N.dptr(sums)))
        return sums

    def drive_apply(self, mean, scale):
        import numpy as np
        self._check(self.L.pmhd_gpu_drive_apply(self.mesh, N.dptr(np.asarray(mean, dtype=np.float64)),
                                                float(scale)))

    def set_async(self, on=True):
        """Stream-ordered multi-rank mode (pmhd_gpu_set_async)."""
        self._check(self.L.pmhd_gpu_set_async(self.mesh, int(on)))

    def torch_stream(self):
        """The context's stream as a torch.cuda.ExternalStream."""
        import torch
        return torch.cuda.ExternalStream(self.stream_handle, device=torch.device("cuda", self.device))

    def halo_unpack(self, gid, d, side, half, buf):
        self._check(self.L.pmhd_gpu_halo_unpack(self.mesh, gid, d, side, int(half), C.c_void_p(buf.data_ptr())))

    def set_profiling(self, on=True):
        self._check(self.L.pmhd_gpu_set_profiling(self.mesh, int(on)))

    def region_times(self, reset=False):
        rt = N.RegionTimes()
        self._check(self.L.pmhd_gpu_region_times(self.mesh, C.byref(rt), int(reset)))
        return {f: getattr(rt, f) for f, _ in N.RegionTimes._fields_}
