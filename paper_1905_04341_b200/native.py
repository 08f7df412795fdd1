"""ctypes bindings of the two native libraries of the product.

* ``libpmhd_host.so``  -- host C++ layer (input files, mesh geometry, problem
  generators), ``include/pmhd_host.h``.
* ``libpmhd_gpu.so``   -- the sm_100a CUDA path behind the C-ABI
  ``include/pmhd_gpu.h`` (``libpmhd_gpu_parity.so`` is the same source built
  with ``--fmad=false`` for bitwise parity runs).

The structures below mirror the C headers field for field.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_DIR = PKG_DIR / "lib"
REPO_DIR = PKG_DIR.parent

# --- enums (include/pmhd_gpu.h) ---------------------------------------------
PMHD_OK = 0
PMHD_ERR_CONFIG = 1
PMHD_ERR_BUFFER = 2
PMHD_ERR_INPUT = 3
PMHD_ERR_UNPHYSICAL = 4
PMHD_ERR_CUDA = 5
PMHD_ERR_UNSUPPORTED = 6

RIEMANN = {"hlld": 0, "hlle": 1, "roe": 2}
LIMITER = {"mc": 0, "vanleer": 1}
EOS = {"error": 0, "floor": 1}
EMF = {"upwind": 0, "arith": 1}
DIAG_DIVB_MAX = 0
DIAG_SUMS = 1

PGEN = {"linear_wave": 0, "orszag_tang": 1, "blast": 2, "turbulence": 3, "uniform": 4}


class MeshDesc(C.Structure):
    _fields_ = [
        ("nx", C.c_int * 3),
        ("mb", C.c_int * 3),
        ("ng", C.c_int),
        ("xmin", C.c_double * 3),
        ("xmax", C.c_double * 3),
        ("gamma", C.c_double),
        ("cfl", C.c_double),
        ("riemann", C.c_int),
        ("limiter", C.c_int),
        ("eos_mode", C.c_int),
        ("emf_mode", C.c_int),
        ("dfloor", C.c_double),
        ("pfloor", C.c_double),
    ]


class Status(C.Structure):
    _fields_ = [
        ("code", C.c_int),
        ("stage", C.c_int),
        ("k", C.c_int),
        ("j", C.c_int),
        ("i", C.c_int),
        ("floor_count", C.c_longlong),
        ("fallback_count", C.c_longlong),
    ]


class RegionTimes(C.Structure):
    _fields_ = [
        ("c2p_ms", C.c_double),
        ("riemann_ms", C.c_double),
        ("ct_emf_ms", C.c_double),
        ("integrate_ms", C.c_double),
        ("boundary_ms", C.c_double),
        ("dt_ms", C.c_double),
        ("calls", C.c_longlong),
        ("kernel_launches", C.c_longlong),
        ("reconstruct_ms", C.c_double),
    ]


class RunConfigC(C.Structure):
    _fields_ = [
        ("mesh", MeshDesc),
        ("pgen", C.c_int),
        ("wave_amp", C.c_double),
        ("wave_n", C.c_int * 3),
        ("wave_mode", C.c_int),
        ("wave_rho", C.c_double),
        ("wave_p", C.c_double),
        ("wave_v", C.c_double * 3),
        ("wave_b", C.c_double * 3),
        ("blast_pin", C.c_double),
        ("blast_pout", C.c_double),
        ("blast_r", C.c_double),
        ("blast_rho", C.c_double),
        ("blast_b", C.c_double * 3),
        ("turb_mach", C.c_double),
        ("turb_seed", C.c_uint64),
        ("uniform_w", C.c_double * 8),
        ("nlim", C.c_int),
        ("tlim", C.c_double),
        ("workers", C.c_int),
        ("gpus", C.c_int),
        ("turb_drive", C.c_int),
        ("turb_dedt", C.c_double),
        ("turb_every", C.c_int),
    ]


class DriveModesC(C.Structure):
    _fields_ = [
        ("n", C.c_int),
        ("k", (C.c_int * 3) * 64),
        ("c", (C.c_double * 3) * 64),
        ("s", (C.c_double * 3) * 64),
    ]


class PlatformC(C.Structure):
    _fields_ = [
        ("id", C.c_char * 32),
        ("t_peak", C.c_double),
        ("nspace", C.c_int),
        ("space", (C.c_char * 16) * 8),
        ("bw", C.c_double * 8),
    ]


_P = C.POINTER
_dp = _P(C.c_double)
_ip = _P(C.c_int)


def _load(path: Path) -> C.CDLL:
    if not path.exists():
        raise OSError(f"native library missing: {path} (run __graft_entry__.build())")
    return C.CDLL(str(path), mode=C.RTLD_GLOBAL)


_host = None
_gpu = {}


def host_lib() -> C.CDLL:
    global _host
    if _host is None:
        L = _load(LIB_DIR / "libpmhd_host.so")
        L.pmhd_host_config_defaults.argtypes = [_P(RunConfigC)]
        L.pmhd_host_config_parse.argtypes = [C.c_char_p, _P(RunConfigC), _ip, C.c_char_p, C.c_int]
        L.pmhd_host_validate.argtypes = [_P(RunConfigC), C.c_char_p, C.c_int]
        L.pmhd_host_nblocks.argtypes = [_P(RunConfigC)]
        L.pmhd_host_block_dims.argtypes = [_P(RunConfigC), _ip]
        L.pmhd_host_block_dims.restype = None
        L.pmhd_host_block_coords.argtypes = [_P(RunConfigC), C.c_int, _ip]
        L.pmhd_host_block_coords.restype = None
        L.pmhd_host_pgen_block.argtypes = [_P(RunConfigC), C.c_int, _dp, _dp, _dp, _dp]
        L.pmhd_host_exact_block.argtypes = [_P(RunConfigC), C.c_int, C.c_double, _dp]
        L.pmhd_host_wave_eigen.argtypes = [_P(RunConfigC), _dp, _dp, _dp]
        L.pmhd_host_default_tlim.argtypes = [_P(RunConfigC)]
        L.pmhd_host_default_tlim.restype = C.c_double
        _pp = _P(_dp)
        L.pmhd_host_snapshot_write.argtypes = [C.c_char_p, _P(RunConfigC), C.c_double, _pp, _pp, _pp, _pp]
        L.pmhd_host_snapshot_read.argtypes = [C.c_char_p, _P(RunConfigC), _dp, _pp, _pp, _pp, _pp]
        L.pmhd_host_drive_modes.argtypes = [_P(RunConfigC), C.c_longlong, _P(DriveModesC)]
        L.pmhd_host_drive_tables.argtypes = [_P(RunConfigC), C.c_int, _dp, _dp]
        L.pmhd_host_drive_scale.argtypes = [C.c_double, C.c_double, C.c_double]
        L.pmhd_host_drive_scale.restype = C.c_double
        L.pmhd_perf_load_platforms.argtypes = [C.c_char_p, _P(PlatformC), C.c_int, _ip, _ip, C.c_char_p,
                                               C.c_int]
        L.pmhd_perf_format_platforms.argtypes = [_P(PlatformC), C.c_int, C.c_char_p, C.c_int]
        L.pmhd_perf_roofline_cap.argtypes = [_P(PlatformC), _P(C.c_char_p), _dp, C.c_int, _dp, _ip]
        L.pmhd_perf_arch_efficiency.argtypes = [C.c_double, C.c_double, _dp, _ip]
        L.pmhd_perf_pp_metric.argtypes = [_dp, _ip, C.c_int, _dp]
        _host = L
    return _host


GPU_SYMBOLS = [
    "pmhd_gpu_abi_version", "pmhd_gpu_ctx_create", "pmhd_gpu_ctx_destroy",
    "pmhd_gpu_last_error", "pmhd_gpu_mesh_create", "pmhd_gpu_mesh_destroy",
    "pmhd_gpu_block_dims", "pmhd_gpu_upload_block", "pmhd_gpu_download_block",
    "pmhd_gpu_exchange", "pmhd_gpu_new_dt", "pmhd_gpu_stage", "pmhd_gpu_vl2_step",
    "pmhd_gpu_run", "pmhd_gpu_diag", "pmhd_gpu_set_profiling", "pmhd_gpu_region_times",
    "pmhd_gpu_build_info", "pmhd_gpu_stream", "pmhd_gpu_stage_compute", "pmhd_gpu_exchange_dir",
    "pmhd_gpu_halo_count", "pmhd_gpu_halo_pack", "pmhd_gpu_halo_unpack", "pmhd_gpu_set_async",
    "pmhd_gpu_drive_begin", "pmhd_gpu_drive_energy", "pmhd_gpu_drive_apply", "pmhd_gpu_stage_prefetch",
    "pmhd_gpu_slab", "pmhd_gpu_ipc_open", "pmhd_gpu_ipc_close", "pmhd_gpu_peer_attach",
]


def gpu_lib_path(parity: bool = False) -> Path:
    # PMHD_GPU_LIB: A/B experiments with an alternative in-tree build of the
    # same sources (e.g. lib/exp/*.so); never a CPU substitute.
    if not parity and os.environ.get("PMHD_GPU_LIB"):
        return Path(os.environ["PMHD_GPU_LIB"]).resolve()
    return LIB_DIR / ("libpmhd_gpu_parity.so" if parity else "libpmhd_gpu.so")


def gpu_lib(parity: bool = False) -> C.CDLL:
    """Load the CUDA C-ABI library.  There is no fallback: a missing library
    raises OSError."""
    if parity not in _gpu:
        # RTLD_LOCAL (+ -Bsymbolic at link time): the FMA and the parity build
        # export the same names and must never interpose on each other.
        path = gpu_lib_path(parity)
        if not path.exists():
            raise OSError(f"native library missing: {path} (run __graft_entry__.build())")
        L = C.CDLL(str(path), mode=C.RTLD_LOCAL)
        L.pmhd_gpu_abi_version.argtypes = []
        L.pmhd_gpu_ctx_create.argtypes = [C.c_int, _P(C.c_void_p)]
        L.pmhd_gpu_ctx_destroy.argtypes = [C.c_void_p]
        L.pmhd_gpu_last_error.argtypes = [C.c_void_p]
        L.pmhd_gpu_last_error.restype = C.c_char_p
        L.pmhd_gpu_mesh_create.argtypes = [C.c_void_p, _P(MeshDesc), _ip, C.c_int, _P(C.c_void_p)]
        L.pmhd_gpu_mesh_destroy.argtypes = [C.c_void_p]
        L.pmhd_gpu_block_dims.argtypes = [C.c_void_p, _ip]
        L.pmhd_gpu_upload_block.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp]
        L.pmhd_gpu_download_block.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.pmhd_gpu_exchange.argtypes = [C.c_void_p]
        L.pmhd_gpu_new_dt.argtypes = [C.c_void_p, _dp, _P(Status)]
        L.pmhd_gpu_stage.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, _P(Status)]
        L.pmhd_gpu_vl2_step.argtypes = [C.c_void_p, C.c_double, _dp, _P(Status)]
        L.pmhd_gpu_run.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, _dp, _ip, _P(Status)]
        L.pmhd_gpu_diag.argtypes = [C.c_void_p, C.c_int, _dp]
        L.pmhd_gpu_set_profiling.argtypes = [C.c_void_p, C.c_int]
        L.pmhd_gpu_region_times.argtypes = [C.c_void_p, _P(RegionTimes), C.c_int]
        L.pmhd_gpu_stage_compute.argtypes = [C.c_void_p, C.c_int, C.c_double, _dp, _P(Status)]
        L.pmhd_gpu_exchange_dir.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.pmhd_gpu_halo_count.argtypes = [C.c_void_p, C.c_int, C.c_int, _P(C.c_longlong)]
        L.pmhd_gpu_halo_pack.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.pmhd_gpu_halo_unpack.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.pmhd_gpu_set_async.argtypes = [C.c_void_p, C.c_int]
        L.pmhd_gpu_stage_prefetch.argtypes = [C.c_void_p, C.c_int, C.c_double]
        L.pmhd_gpu_slab.argtypes = [C.c_void_p, _P(C.c_void_p), C.c_void_p]
        L.pmhd_gpu_ipc_open.argtypes = [C.c_void_p, C.c_void_p, _P(C.c_void_p)]
        L.pmhd_gpu_ipc_close.argtypes = [C.c_void_p, C.c_void_p]
        L.pmhd_gpu_peer_attach.argtypes = [C.c_void_p, C.c_int, _ip, _P(C.c_void_p)]
        L.pmhd_gpu_drive_begin.argtypes = [C.c_void_p, C.c_int, _ip, _dp, _dp, _P(_dp), _P(_dp), _dp]
        L.pmhd_gpu_drive_energy.argtypes = [C.c_void_p, _dp, _dp]
        L.pmhd_gpu_drive_apply.argtypes = [C.c_void_p, _dp, C.c_double]
        L.pmhd_gpu_stream.argtypes = [C.c_void_p]
        L.pmhd_gpu_stream.restype = C.c_void_p
        L.pmhd_gpu_build_info.argtypes = []
        L.pmhd_gpu_build_info.restype = C.c_char_p
        _gpu[parity] = L
    return _gpu[parity]


def dptr(a):
    """double* of a C-contiguous float64 numpy array (or NULL for None)."""
    if a is None:
        return C.cast(None, _dp)
    assert a.dtype.name == "float64" and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def cpu_count() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
