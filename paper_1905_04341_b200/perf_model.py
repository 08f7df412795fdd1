"""perf_model: Eq. 1 roofline cap, Eq. 2 architectural
efficiency, Eq. 3 performance-portability metric and the Table 2 platform
CSV, over the C implementation in libpmhd_host.so (csrc/host/perf_model.cpp;
the CLI's `pmhd roofline` / `pmhd report` use the same functions)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

from . import native as N
from .mesh import ParseError


@dataclass
class RooflinePlatform:
    """RooflinePlatform: T_peak in FLOP/s, bandwidths B/s."""
    id: str
    t_peak: float
    bw: dict = field(default_factory=dict)

    def _c(self) -> N.PlatformC:
        p = N.PlatformC()
        p.id = self.id.encode()
        p.t_peak = self.t_peak
        p.nspace = len(self.bw)
        for q, (k, v) in enumerate(self.bw.items()):
            p.space[q].value = k.encode()
            p.bw[q] = v
        return p


def _from_c(p: N.PlatformC) -> RooflinePlatform:
    return RooflinePlatform(p.id.decode(), p.t_peak,
                            {p.space[q].value.decode(): p.bw[q] for q in range(p.nspace)})


def load_platform_table(text: str):
    """load_platform_table: list of RooflinePlatform;
    ParseError(line) on a malformed row."""
    arr = (N.PlatformC * 64)()
    n, line = C.c_int(0), C.c_int(0)
    buf = C.create_string_buffer(256)
    rc = N.host_lib().pmhd_perf_load_platforms(text.encode(), arr, 64, C.byref(n), C.byref(line), buf, 256)
    if rc != N.PMHD_OK:
        raise ParseError(line.value, buf.value.decode())
    return [_from_c(arr[q]) for q in range(n.value)]


def format_platform_table(plats) -> str:
    arr = (N.PlatformC * max(1, len(plats)))(*[p._c() for p in plats])
    need = N.host_lib().pmhd_perf_format_platforms(arr, len(plats), None, 0)
    buf = C.create_string_buffer(need)
    N.host_lib().pmhd_perf_format_platforms(arr, len(plats), buf, need)
    return buf.value.decode()


def roofline_cap(plat: RooflinePlatform, intensities: dict):
    """roofline_cap (Eq. 1): (P_max, binding) with binding 'compute' or the
    memory space whose B*I binds."""
    names = list(intensities)
    sp = (C.c_char_p * max(1, len(names)))(*[k.encode() for k in names])
    iv = (C.c_double * max(1, len(names)))(*[float(intensities[k]) for k in names])
    cap, bind = C.c_double(), C.c_int()
    p = plat._c()
    if N.host_lib().pmhd_perf_roofline_cap(C.byref(p), sp, iv, len(names), C.byref(cap), C.byref(bind)):
        raise ValueError(f"unknown memory space in {names} for platform {plat.id}")
    return cap.value, ("compute" if bind.value < 0 else names[bind.value])


def arch_efficiency(eps: float, cap: float):
    """arch_efficiency (Eq. 2): (e, flagged) with flagged = e > 1."""
    e, flag = C.c_double(), C.c_int()
    if N.host_lib().pmhd_perf_arch_efficiency(float(eps), float(cap), C.byref(e), C.byref(flag)):
        raise ValueError("zero or negative roofline cap")
    return e.value, bool(flag.value)


def pp_metric(effs, supported=None) -> float:
    """pp_metric (Eq. 3): harmonic mean of the efficiencies, 0 if any
    platform is unsupported."""
    n = len(effs)
    e = (C.c_double * n)(*effs)
    sup = (C.c_int * n)(*([1] * n if supported is None else [int(bool(x)) for x in supported]))
    P = C.c_double()
    if N.host_lib().pmhd_perf_pp_metric(e, sup, n, C.byref(P)):
        raise ValueError("supported platform with zero efficiency")
    return P.value
