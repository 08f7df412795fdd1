"""CPU-only checks of the drop-in boundary: the C-ABI libraries load and
export every symbol declared in include/*.h (no compute calls without a GPU),
plus the host C++ layer (input-file API, MeshConfig, problem generators)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1905_04341_b200 import RunConfig, ParseError, ConfigError
from paper_1905_04341_b200 import native as N

ROOT = Path(__file__).resolve().parents[1]


def declared(header):
    txt = (ROOT / "include" / header).read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\**\s+\**(pmhd_\w+)\s*\(", txt, re.M)))


@pytest.mark.parametrize("parity", [False, True])
def test_gpu_library_exports_header(parity):
    names = declared("pmhd_gpu.h")
    assert len(names) >= 17
    lib = ctypes.CDLL(str(N.gpu_lib_path(parity)), mode=ctypes.RTLD_LOCAL)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(N.GPU_SYMBOLS)


@pytest.mark.parametrize("parity", [False, True])
def test_build_info_is_one_csv_field(parity):
    """pmhd_gpu_build_info() (host-only, no device needed) is the policy
    column of `pmhd bench`'s CSV row: no commas or newlines."""
    lib = ctypes.CDLL(str(N.gpu_lib_path(parity)), mode=ctypes.RTLD_LOCAL)
    lib.pmhd_gpu_build_info.restype = ctypes.c_char_p
    info = lib.pmhd_gpu_build_info().decode()
    assert info and "," not in info and "\n" not in info, info
    assert info.endswith("+parity(fmad=false)") == parity


def test_gpu_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.gpu_lib_path(False))],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_host_library_exports_header():
    names = declared("pmhd_host.h")
    lib = N.host_lib()
    for n in names:
        assert hasattr(lib, n), n


def test_parse_config_spec_examples():
    c = RunConfig("nx1 = 64\npolicy = flat1d")
    assert c.desc.nx[0] == 64
    d = RunConfig("")
    assert tuple(d.desc.nx) == (16, 16, 16) and d.nblocks == 1
    with pytest.raises(ParseError) as ei:
        RunConfig("nx1 = banana")
    assert ei.value.line_number == 1
    with pytest.raises(ParseError) as ei:
        RunConfig("# comment\nnx1 = 8\nfoo = 3")
    assert ei.value.line_number == 3
    e = RunConfig("nx1 = 8\nnx1 = 32  # later wins")
    assert e.desc.nx[0] == 32
    f = RunConfig("<mesh>\nnx1 = 24\n<problem>\nriemann = hlle")
    assert f.desc.nx[0] == 24 and f.desc.riemann == 1


def test_mesh_invariants():
    with pytest.raises(ConfigError):
        RunConfig(nx1=48, nx2=32, nx3=32, mb1=32, mb2=32, mb3=32).validate()
    with pytest.raises(ConfigError):
        RunConfig(ng=1).validate()
    c = RunConfig(nx1=64, nx2=64, nx3=64, mb1=32, mb2=32, mb3=32)
    c.validate()
    assert c.nblocks == 8 and c.block_dims == (36, 36, 36)
    c2 = RunConfig(nx1=64, nx2=32, nx3=1, mb1=32, mb2=32, mb3=1)
    assert c2.dim == 2 and c2.block_dims == (36, 36, 1)


@pytest.mark.parametrize("pgen", ["linear_wave", "orszag_tang", "blast", "turbulence", "uniform"])
def test_pgen_divergence_free(pgen):
    kw = dict(nx1=16, nx2=16, nx3=16, mb1=16, mb2=16, mb3=16, pgen=pgen, wave_n1=1, wave_n2=1,
              wave_n3=1)
    if pgen == "orszag_tang":
        kw.update(nx3=1, mb3=1)
    cfg = RunConfig(**kw)
    b = cfg.pgen_block(0)
    ks, js, is_ = cfg.active_slices()
    dx = 1.0 / 16
    div = (np.diff(b.b1f, axis=2)[ks, js, is_] + np.diff(b.b2f, axis=1)[ks, js, is_]) / dx
    if cfg.dim == 3:
        div += np.diff(b.b3f, axis=0)[ks, js, is_] / dx
    assert np.max(np.abs(div)) <= 1e-13
    assert np.all(b.u[0, ks, js, is_] > 0)


def test_wave_eigenvector_residual():
    for mode in range(7):
        cfg = RunConfig(wave_mode=mode)
        lam, r, res = cfg.wave_eigen()
        assert res <= 1e-12, (mode, res)
        assert abs(np.linalg.norm(r) - 1.0) <= 1e-12
    # fast speed of the default background is 2 (a^2=1, B^2=3.25, Bx^2=1)
    lam, _, _ = RunConfig(wave_mode=6).wave_eigen()
    assert abs(lam - 2.0) <= 1e-12


def test_wave_eigenvector_numpy_oracle():
    """Cross-check against numpy.linalg.eig of a centred finite-difference
    Jacobian (the SPEC's eigen oracle)."""
    g = 5.0 / 3.0
    bn = 1.0

    def flux(U):
        d, mn, mt1, mt2, E, bt1, bt2 = U
        vn, vt1, vt2 = mn / d, mt1 / d, mt2 / d
        pb = 0.5 * (bn * bn + bt1 * bt1 + bt2 * bt2)
        p = (g - 1) * (E - 0.5 * (mn * vn + mt1 * vt1 + mt2 * vt2) - pb)
        pt = p + pb
        return np.array([mn, mn * vn + pt - bn * bn, mt1 * vn - bn * bt1, mt2 * vn - bn * bt2,
                         (E + pt) * vn - bn * (vn * bn + vt1 * bt1 + vt2 * bt2), bt1 * vn - bn * vt1,
                         bt2 * vn - bn * vt2])
    U0 = np.array([1.0, 0, 0, 0, 0.6 / (g - 1) + 0.5 * (1 + 2 + 0.25), np.sqrt(2), 0.5])
    J = np.zeros((7, 7))
    for c in range(7):
        h = 1e-6
        e = np.zeros(7)
        e[c] = h
        J[:, c] = (flux(U0 + e) - flux(U0 - e)) / (2 * h)
    vals, vecs = np.linalg.eig(J)
    for mode in (5, 6):
        lam, r, _ = RunConfig(wave_mode=mode).wave_eigen()
        k = np.argmin(np.abs(vals.real - lam))
        assert abs(vals[k].real - lam) <= 1e-7
        v = vecs[:, k].real
        v = v / np.linalg.norm(v)
        assert min(np.linalg.norm(v - r), np.linalg.norm(v + r)) <= 1e-6
