"""The product build's branch-free division / square root (physics.cuh) against
the IEEE operators over operands spanning the ranges the physics produces (and
well beyond): 1e-30 .. 1e30, both signs, exact squares, powers of two, and
sqrt(0).

* product variant (PMHD_DIVSQRT_1ULP, the Makefile's FASTDS): MUFU seed + one
  cubic Newton step, no rounding correction -- every result within 1 ulp;
  its reciprocal square root drsqrt (HLLD's |Bx| / sqrt(rho*)) within 2 ulp
  of the IEEE expression it replaces, 1 / sqrt(x) (which rounds twice and is
  itself up to 1 ulp from the exact root; drsqrt rounds once);
* PMHD_FAST_DIVSQRT alone: the IEEE fast-path sequence -- bit for bit."""
import ctypes as C

import numpy as np
import pytest

from paper_1905_04341_b200.native import LIB_DIR

pytestmark = pytest.mark.gpu


def _run(name):
    path = LIB_DIR / "test" / name
    if not path.exists():
        pytest.fail(f"missing {path} (run __graft_entry__.build())")
    L = C.CDLL(str(path))
    L.pmhd_test_divsqrt.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]
    rng = np.random.default_rng(1905)
    n = 1 << 22
    a = rng.choice([-1.0, 1.0], n) * 10.0 ** rng.uniform(-30, 30, n)
    b = rng.choice([-1.0, 1.0], n) * 10.0 ** rng.uniform(-30, 30, n)
    # physics-like magnitudes, exact cases and perfect squares
    a[: n // 4] = rng.uniform(1e-3, 1e3, n // 4)
    b[: n // 4] = rng.uniform(1e-3, 1e3, n // 4)
    a[n // 4: n // 4 + 1000] = np.arange(1000, dtype=np.float64) ** 2
    b[n // 4: n // 4 + 1000] = 2.0 ** rng.integers(-60, 60, 1000)
    a[n // 4] = 0.0
    out = np.zeros(6, dtype=np.uint64)
    rc = L.pmhd_test_divsqrt(a.ctypes.data, b.ctypes.data, n, out.ctypes.data)
    assert rc == 0
    return out


def test_product_divsqrt_within_one_ulp(gpu_available):
    out = _run("libpmhd_divsqrt_check.so")
    assert out[2] <= 1, f"division off by {out[2]} ulp"
    assert out[3] <= 1, f"sqrt off by {out[3]} ulp"
    assert out[5] <= 2, f"rsqrt off by {out[5]} ulp from 1/sqrt(x)"
    assert out[4] > 0 or out[5] == 0
    print(f"product variant: {out[0]} divisions, {out[1]} square roots and {out[4]} reciprocal roots "
          "differ from IEEE (max {out[2]}, {out[3]}, {out[5]} ulp)")


def test_exact_divsqrt_bitwise_ieee(gpu_available):
    out = _run("libpmhd_divsqrt_exact_check.so")
    assert out[0] == 0, f"{out[0]} divisions differ from IEEE"
    assert out[1] == 0, f"{out[1]} square roots differ from IEEE"
    assert out[4] == 0 and out[5] == 0  # no drsqrt in this build
