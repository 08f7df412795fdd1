"""perf_model and its acceptance criteria 6 and 7
(SPEC.md:541-542): Eq. 1 cap, Eq. 2 efficiency, Eq. 3 portability metric,
the Table 2 platform CSV."""
import math

import pytest

from paper_1905_04341_b200 import ParseError
from paper_1905_04341_b200.perf_model import (RooflinePlatform, arch_efficiency, format_platform_table,
                                             load_platform_table, pp_metric, roofline_cap)

V100 = "id,t_peak_gflops,bw_dram_gbs\nv100,7000,782\n"


def test_v100_fixture_dram_bound():
    (v,) = load_platform_table(V100)
    assert v.id == "v100" and v.t_peak == 7000e9 and v.bw == {"dram": 782e9}
    cap, bind = roofline_cap(v, {"dram": 1.0})
    assert cap == 782e9 and bind == "dram"


def test_cap_saturates_and_knee():
    (v,) = load_platform_table(V100)
    cap, bind = roofline_cap(v, {"dram": 1e9})
    assert cap == 7000e9 and bind == "compute"
    knee = 7000.0 / 782.0
    assert roofline_cap(v, {"dram": knee * 0.999})[1] == "dram"
    assert roofline_cap(v, {"dram": knee * 1.001})[1] == "compute"


def test_multi_space_min_and_unknown_space():
    p = RooflinePlatform("x", 1e12, {"dram": 1e11, "l2": 5e11})
    assert roofline_cap(p, {"dram": 2.0, "l2": 1.0}) == (2e11, "dram")
    assert roofline_cap(p, {"dram": 10.0, "l2": 0.1}) == (5e10, "l2")
    with pytest.raises(ValueError):
        roofline_cap(p, {"hbm": 1.0})


def test_eq2_fixture_72_5_percent():  # acceptance 6
    e, flag = arch_efficiency(0.82e12, 1.13e12)
    assert abs(e - 0.7257) <= 5e-4 and not flag
    assert arch_efficiency(5.0, 5.0) == (1.0, False)
    assert arch_efficiency(6.0, 5.0)[1] is True  # flagged, not clamped
    assert math.isclose(arch_efficiency(3 * 0.82e12, 1.13e12)[0], 3 * e, rel_tol=1e-15)  # linearity
    with pytest.raises(ValueError):
        arch_efficiency(1.0, 0.0)


def test_eq3_properties():  # acceptance 7
    assert abs(pp_metric([0.725, 0.5]) - 0.5918) <= 1e-4
    assert pp_metric([0.63]) == 0.63
    assert pp_metric([0.4, 0.4, 0.4]) == pytest.approx(0.4, abs=0, rel=1e-15)
    assert pp_metric([0.9, 0.5], supported=[1, 0]) == 0.0
    effs = [0.9, 0.3, 0.6]
    assert pp_metric(effs) == pp_metric(effs[::-1])  # permutation invariant
    # harmonic-mean bounds.  (SPEC.md:422 words this as "<= min efficiency",
    # which no mean of unequal efficiencies satisfies; the harmonic mean lies
    # in [min, max] and is <= the arithmetic mean.)
    assert min(effs) <= pp_metric(effs) <= sum(effs) / len(effs)
    with pytest.raises(ValueError):
        pp_metric([0.5, 0.0])


def test_platform_table_parse_errors_and_round_trip():
    assert load_platform_table("") == []
    text = "id,t_peak_gflops,bw_dram_gbs,bw_l2_gbs\nb200,36985,6451.2,20000\nv100,7000,782,3000\n"
    plats = load_platform_table(text)
    again = load_platform_table(format_platform_table(plats))
    assert again == plats
    with pytest.raises(ParseError) as ei:
        load_platform_table("id,t_peak_gflops,bw_dram_gbs\nv100,banana,782\n")
    assert ei.value.line_number == 2
    with pytest.raises(ParseError) as ei:
        load_platform_table("id,t_peak_gflops,bw_dram_gbs\nv100,7000\n")
    assert ei.value.line_number == 2
    with pytest.raises(ParseError):
        load_platform_table("id,peak\n")


def test_shipped_platform_file():
    import pathlib
    plats = {p.id: p for p in load_platform_table(
        (pathlib.Path(__file__).resolve().parent.parent / "profiles" / "platforms.csv").read_text())}
    assert plats["v100"].bw["dram"] == 782e9
    assert plats["b200"].t_peak == 36985e9
