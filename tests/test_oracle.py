"""CPU tests of the oracle (test infrastructure) against the reference's own
known answers (tests/golden/spec_known_answers.json, transcribed from
/root/reference/SPEC.md) and the SPEC properties, plus an independent
textbook HLLD and the reference exec layer (oracle/_ref) cross-checks."""
import json
import math
import os

import numpy as np
import pytest

from paper_1905_04341_b200 import RunConfig, l1_error, ConfigError
from paper_1905_04341_b200 import native as N
from oracle import binding as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_known_answers.json")))
TOL = GOLD["tolerances"]
G53 = 5.0 / 3.0


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# ---------------------------------------------------------------- known answers
@pytest.mark.parametrize("v", GOLD["cons_to_prim"], ids=lambda v: v["ref"])
def test_cons_to_prim_known(v):
    if v.get("error"):
        with pytest.raises(Exception):
            O.cons_to_prim(v["u"], v["gamma"])
        return
    w = O.cons_to_prim(v["u"], v["gamma"])
    assert np.allclose(w, v["w"], rtol=TOL["known_answer_rel"], atol=0)


@pytest.mark.parametrize("v", GOLD["prim_to_cons"], ids=lambda v: v["ref"])
def test_prim_to_cons_known(v):
    u = O.prim_to_cons(v["w"], v["gamma"])
    assert rel(u[4], v["E"]) <= TOL["known_answer_rel"]


@pytest.mark.parametrize("v", GOLD["fast_speed"], ids=lambda v: v["ref"])
def test_fast_speed_known(v):
    cf = O.fast_speed(v["w"], v["gamma"], v["dim"])
    assert rel(cf, v["cf"]) <= 2 * TOL["fast_speed_rel"]


def test_prim_cons_roundtrip_random():
    rng = np.random.default_rng(1)
    for _ in range(500):
        w = np.array([rng.uniform(0.1, 10), *rng.normal(0, 2, 3), rng.uniform(0.1, 10), *rng.normal(0, 2, 3)])
        w2 = O.cons_to_prim(O.prim_to_cons(w, G53), G53)
        scale = np.maximum(np.abs(w), 1e-3)
        assert np.all(np.abs(w2 - w) / scale <= 1e-13)


def test_fast_speed_bounds_random():
    rng = np.random.default_rng(2)
    for _ in range(500):
        w = np.array([rng.uniform(0.1, 10), 0, 0, 0, rng.uniform(0.1, 10), *rng.normal(0, 2, 3)])
        for d in range(3):
            cf = O.fast_speed(w, G53, d)
            cs = math.sqrt(G53 * w[4] / w[0])
            ca = abs(w[5 + d]) / math.sqrt(w[0])
            assert cf >= max(cs, ca) * (1 - 1e-14)


@pytest.mark.parametrize("v", GOLD["compute_dt"], ids=lambda v: v["ref"])
def test_compute_dt_known(v):
    cfg = RunConfig(**v["config"])
    s = O.OracleSolver(cfg)
    s.load_pgen()
    assert rel(s.new_dt(), v["dt"]) <= 1e-14
    # doubling resolution halves dt
    c2 = dict(v["config"], nx1=32, nx2=32, nx3=32, mb1=32, mb2=32, mb3=32)
    s2 = O.OracleSolver(RunConfig(**c2))
    s2.load_pgen()
    assert rel(s2.new_dt(), v["dt"] / 2) <= 1e-14


@pytest.mark.parametrize("v", GOLD["build_mesh"], ids=lambda v: v["ref"])
def test_build_mesh_known(v):
    cfg = RunConfig(nx1=v["nx"][0], nx2=v["nx"][1], nx3=v["nx"][2], mb1=v["mb"][0],
                    mb2=v["mb"][1], mb3=v["mb"][2])
    if v.get("error"):
        with pytest.raises(ConfigError):
            cfg.validate()
        with pytest.raises(ConfigError):
            O.OracleSolver(cfg)
        return
    cfg.validate()
    assert cfg.nblocks == v["nblocks"]
    assert O.OracleSolver(cfg).nblocks == v["nblocks"]


def test_arch_efficiency_fixture():
    v = GOLD["arch_efficiency"][0]
    assert abs(v["eps"] / v["cap"] - v["e"]) <= v["tol"]


# ---------------------------------------------------------------- PLM
def test_plm_limiter_properties():
    for lim in ("mc", "vanleer"):
        assert O.plm_slope(2.0, 2.0, 2.0, lim) == 0.0
        s = O.plm_slope(1.0, 1.5, 2.0, lim)
        assert abs(s - 0.5) <= 1e-16
        assert O.plm_slope(1.0, 3.0, 2.0, lim) == 0.0  # extremum
    rng = np.random.default_rng(3)
    for _ in range(2000):
        qm, q0, qp = rng.normal(size=3)
        for lim in ("mc", "vanleer"):
            s = O.plm_slope(qm, q0, qp, lim)
            lo, hi = min(qm, q0, qp), max(qm, q0, qp)
            if (q0 - qm) * (qp - q0) <= 0:
                assert s == 0.0
            assert lo - 1e-15 <= q0 + 0.5 * s <= hi + 1e-15
            assert lo - 1e-15 <= q0 - 0.5 * s <= hi + 1e-15


# ---------------------------------------------------------------- Riemann
def phys_flux(w, bx, g):
    d, u, v, ww, p, by, bz = w
    pt = p + 0.5 * (bx * bx + by * by + bz * bz)
    e = p / (g - 1) + 0.5 * d * (u * u + v * v + ww * ww) + 0.5 * (bx * bx + by * by + bz * bz)
    return np.array([d * u, d * u * u + pt - bx * bx, d * v * u - bx * by, d * ww * u - bx * bz,
                     (e + pt) * u - bx * (u * bx + v * by + ww * bz), by * u - bx * v, bz * u - bx * ww])


def rand_state(rng):
    return np.array([rng.uniform(0.2, 5), *rng.normal(0, 1, 3), rng.uniform(0.2, 5), *rng.normal(0, 1, 2)])


def test_riemann_consistency():
    rng = np.random.default_rng(4)
    for _ in range(1000):
        w = rand_state(rng)
        bx = rng.normal()
        F = O.phys_flux(w, bx, G53)
        assert np.max(np.abs(F - phys_flux(w, bx, G53))) <= 1e-14 * (np.max(np.abs(F)) + 1)
        fe = O.riemann("hlle", w, w, bx, G53)
        assert np.array_equal(fe, F)  # exactly F(W)
        scale = np.max(np.abs(F)) + 1.0
        fd = O.riemann("hlld", w, w, bx, G53)
        assert np.max(np.abs(fd - F)) / scale <= 1e-13


def test_hlle_supersonic_branch():
    wl = np.array([1.0, 10.0, 0.1, 0.2, 0.6, 0.3, 0.1])
    wr = np.array([0.5, 9.0, -0.1, 0.0, 0.4, -0.2, 0.5])
    f = O.riemann("hlle", wl, wr, 0.7, G53)
    assert np.array_equal(f, O.phys_flux(wl, 0.7, G53))  # S_L > 0 -> F(U_L) exactly
    f = O.riemann("hlld", wl, wr, 0.7, G53)
    assert np.array_equal(f, O.phys_flux(wl, 0.7, G53))


def test_hlld_stationary_contact():
    for bx in (0.0, 0.8):
        wl = np.array([1.0, 0, 0, 0, 1.0, 0.3, 0.2])
        wr = np.array([0.125, 0, 0, 0, 1.0, 0.3, 0.2])
        f = O.riemann("hlld", wl, wr, bx, G53)
        assert abs(f[0]) <= 1e-15


def hlld_textbook(wl, wr, bx, g):
    """Independent Miyoshi & Kusano (2005) HLLD, written from the paper with
    a different algebraic arrangement (pt* from Eq. 23-form, direct divides)."""
    def cons(W):
        d, u, v, w, p, by, bz = W
        e = p / (g - 1) + 0.5 * d * (u * u + v * v + w * w) + 0.5 * (bx * bx + by * by + bz * bz)
        return np.array([d, d * u, d * v, d * w, e, by, bz])

    def cfast(W):
        d, u, v, w, p, by, bz = W
        a2, b2, bx2 = g * p / d, (bx * bx + by * by + bz * bz) / d, bx * bx / d
        return math.sqrt(0.5 * (a2 + b2 + math.sqrt((a2 + b2) ** 2 - 4 * a2 * bx2)))

    UL, UR = cons(wl), cons(wr)
    FL, FR = phys_flux(wl, bx, g), phys_flux(wr, bx, g)
    SL = min(wl[1] - cfast(wl), wr[1] - cfast(wr))
    SR = max(wl[1] + cfast(wl), wr[1] + cfast(wr))
    if SL >= 0:
        return FL
    if SR <= 0:
        return FR
    ptL = wl[4] + 0.5 * (bx * bx + wl[5] ** 2 + wl[6] ** 2)
    ptR = wr[4] + 0.5 * (bx * bx + wr[5] ** 2 + wr[6] ** 2)
    SM = ((SR - wr[1]) * wr[0] * wr[1] - (SL - wl[1]) * wl[0] * wl[1] - ptR + ptL) / \
         ((SR - wr[1]) * wr[0] - (SL - wl[1]) * wl[0])
    pst = ptL + wl[0] * (SL - wl[1]) * (SM - wl[1])

    def star(W, U, S):
        d, u, v, w, p, by, bz = W
        dst = d * (S - u) / (S - SM)
        den = d * (S - u) * (S - SM) - bx * bx
        if abs(den) < 1e-8 * pst:
            vs, ws, bys, bzs = v, w, by, bz
        else:
            vs = v - bx * by * (SM - u) / den
            ws = w - bx * bz * (SM - u) / den
            bys = by * (d * (S - u) ** 2 - bx * bx) / den
            bzs = bz * (d * (S - u) ** 2 - bx * bx) / den
        pt = p + 0.5 * (bx * bx + by * by + bz * bz)
        es = ((S - u) * U[4] - pt * u + pst * SM + bx * ((u * bx + v * by + w * bz) - (SM * bx + vs * bys + ws * bzs))) / (S - SM)
        return dst, vs, ws, bys, bzs, es

    dL, vL, wL_, byL, bzL, eL = star(wl, UL, SL)
    dR, vR, wR_, byR, bzR, eR = star(wr, UR, SR)
    ULs = np.array([dL, dL * SM, dL * vL, dL * wL_, eL, byL, bzL])
    URs = np.array([dR, dR * SM, dR * vR, dR * wR_, eR, byR, bzR])
    SLs, SRs = SM - abs(bx) / math.sqrt(dL), SM + abs(bx) / math.sqrt(dR)
    if SLs >= 0:
        return FL + SL * (ULs - UL)
    if SRs <= 0:
        return FR + SR * (URs - UR)
    if 0.5 * bx * bx < 1e-8 * pst:
        ULss, URss = ULs, URs
    else:
        sg = math.copysign(1.0, bx)
        sl, sr = math.sqrt(dL), math.sqrt(dR)
        vss = (sl * vL + sr * vR + sg * (byR - byL)) / (sl + sr)
        wss = (sl * wL_ + sr * wR_ + sg * (bzR - bzL)) / (sl + sr)
        byss = (sl * byR + sr * byL + sg * sl * sr * (vR - vL)) / (sl + sr)
        bzss = (sl * bzR + sr * bzL + sg * sl * sr * (wR_ - wL_)) / (sl + sr)
        vbss = SM * bx + vss * byss + wss * bzss
        eLss = eL - sl * sg * ((SM * bx + vL * byL + wL_ * bzL) - vbss)
        eRss = eR + sr * sg * ((SM * bx + vR * byR + wR_ * bzR) - vbss)
        ULss = np.array([dL, dL * SM, dL * vss, dL * wss, eLss, byss, bzss])
        URss = np.array([dR, dR * SM, dR * vss, dR * wss, eRss, byss, bzss])
    if SM >= 0:
        return FL + SL * (ULs - UL) + SLs * (ULss - ULs)
    return FR + SR * (URs - UR) + SRs * (URss - URs)


def test_hlld_matches_textbook():
    rng = np.random.default_rng(5)
    worst = 0.0
    for _ in range(2000):
        wl, wr = rand_state(rng), rand_state(rng)
        bx = rng.normal()
        a = O.riemann("hlld", wl, wr, bx, G53)
        b = hlld_textbook(wl, wr, bx, G53)
        scale = np.max(np.abs(phys_flux(wl, bx, G53))) + np.max(np.abs(phys_flux(wr, bx, G53)))
        worst = max(worst, np.max(np.abs(a - b)) / scale)
    assert worst <= 1e-12, worst


def test_hlld_between_hlle_and_exact_for_shocktube():
    # Brio-Wu left/right states: HLLD and HLLE give the same supersonic-free
    # mass-flux sign and HLLD is less diffusive on the contact (|F_d| smaller)
    wl = np.array([1.0, 0, 0, 0, 1.0, 1.0, 0])
    wr = np.array([0.125, 0, 0, 0, 0.1, -1.0, 0])
    fd = O.riemann("hlld", wl, wr, 0.75, 2.0)
    fe = O.riemann("hlle", wl, wr, 0.75, 2.0)
    assert np.sign(fd[0]) == np.sign(fe[0])
    assert np.all(np.isfinite(fd))


# ---------------------------------------------------------------- mesh level
def small_wave(n=16, blocks=1, **kw):
    mb = n // blocks
    return RunConfig(nx1=n, nx2=n // 2, nx3=n // 2, mb1=mb, mb2=n // 2, mb3=n // 2, x2max=0.5,
                     x3max=0.5, **kw)


def test_uniform_state_unchanged():
    cfg = RunConfig(nx1=12, nx2=12, nx3=12, mb1=12, mb2=12, mb3=12, pgen="uniform", rho=1.3,
                    v1=0.4, v2=-0.2, v3=0.1, p=0.7, b1=0.3, b2=-0.5, b3=0.2)
    s = O.OracleSolver(cfg)
    s.load_pgen()
    b0 = s.get_block(0)
    for _ in range(5):
        dt = s.new_dt()
        s.vl2_step(dt)
    b1 = s.get_block(0)
    ks, js, is_ = cfg.active_slices()
    d = np.abs(b1.u[:, ks, js, is_] - b0.u[:, ks, js, is_]) / np.maximum(np.abs(b0.u[:, ks, js, is_]), 1)
    assert d.max() <= TOL["uniform_state"]


def test_emf_zero_and_uniform():
    cfg = RunConfig(nx1=8, nx2=8, nx3=8, mb1=8, mb2=8, mb3=8, pgen="uniform", rho=1, p=1, b1=0.3,
                    b2=0.2, b3=0.1)
    s = O.OracleSolver(cfg)
    s.load_pgen()
    s.vl2_step(s.new_dt())
    for c in range(3):
        e = s.emf_data(0, c)
        # v = 0 -> E = 0 up to HLLD star-state round-off (face E ~ 1e-17)
        assert np.max(np.abs(e)) <= 1e-16
    cfg_e = RunConfig(nx1=8, nx2=8, nx3=8, mb1=8, mb2=8, mb3=8, pgen="uniform", rho=1, p=1, b1=0.3,
                      b2=0.2, b3=0.1, riemann="hlle")
    s = O.OracleSolver(cfg_e)
    s.load_pgen()
    s.vl2_step(s.new_dt())
    for c in range(3):
        assert np.max(np.abs(s.emf_data(0, c))) == 0.0  # HLLE(W,W) = F(W) exactly -> exactly 0
    cfg = RunConfig(nx1=8, nx2=8, nx3=8, mb1=8, mb2=8, mb3=8, pgen="uniform", rho=1, p=1, v1=0.2,
                    v2=0.1, v3=-0.3, b1=0.3, b2=0.2, b3=0.1)
    s = O.OracleSolver(cfg)
    s.load_pgen()
    s.vl2_step(s.new_dt())
    ks = slice(2, 11)
    for c in range(3):
        e = s.emf_data(0, c)[2:10, 2:10, 2:10]
        assert np.ptp(e) <= 1e-16 * max(1, np.max(np.abs(e)))


def test_divb_ramp():
    cfg = RunConfig(nx1=8, nx2=8, nx3=8, mb1=8, mb2=8, mb3=8, pgen="uniform")
    s = O.OracleSolver(cfg)
    b = cfg.new_block()
    n1 = b.b1f.shape[2]
    sl = 3.0
    dx = 1.0 / 8
    b.b1f[:] = sl * dx * np.arange(n1)[None, None, :]
    b.u[0] = 1
    b.u[4] = 1
    s.set_block(0, b)
    assert abs(s.divb_max() - sl) <= 1e-13


@pytest.mark.parametrize("blocks", [1, 2])
def test_linear_wave_divb_and_conservation(blocks):
    cfg = RunConfig(nx1=16, nx2=16, nx3=16, mb1=16 // blocks, mb2=16, mb3=16, wave_n1=1, wave_n2=1,
                    wave_n3=1, wave_mode=6, wave_amp=1e-4)
    s = O.OracleSolver(cfg, workers=4)
    s.load_pgen()
    assert s.divb_max() <= TOL["divb_vecpot"]
    s0 = s.sums()
    s.run(ncycles=10)
    s1 = s.sums()
    for v in (0, 4):  # mass and energy
        assert abs(s1[v] - s0[v]) / abs(s0[v]) <= TOL["conservation_rel"]
    assert s.divb_max() <= TOL["divb_period"]


def test_decomposition_independence_bitwise():
    res = []
    for blocks in [(1, 1, 1), (2, 2, 2)]:
        cfg = RunConfig(nx1=16, nx2=16, nx3=16, mb1=16 // blocks[0], mb2=16 // blocks[1],
                        mb3=16 // blocks[2], wave_n1=1, wave_n2=1, wave_n3=0, wave_amp=1e-3)
        s = O.OracleSolver(cfg, workers=4)
        s.load_pgen()
        s.run(ncycles=4)
        # assemble global active arrays
        glob = np.zeros((5, 16, 16, 16))
        ks, js, is_ = cfg.active_slices()
        for gid in range(cfg.nblocks):
            c = cfg.block_coords(gid)
            mb = (16 // blocks[0], 16 // blocks[1], 16 // blocks[2])
            glob[:, c[2] * mb[2]:(c[2] + 1) * mb[2], c[1] * mb[1]:(c[1] + 1) * mb[1],
                 c[0] * mb[0]:(c[0] + 1) * mb[0]] = s.get_block(gid).u[:5, ks, js, is_]
        res.append(glob)
    assert np.array_equal(res[0], res[1])


def test_linear_wave_convergence_order():  # SPEC.md:244, acceptance 1
    errs = []
    for n in (32, 64):
        cfg = RunConfig(nx1=n, nx2=8, nx3=8, mb1=n, mb2=8, mb3=8, x2max=8.0 / n, x3max=8.0 / n,
                        wave_mode=6)
        s = O.OracleSolver(cfg, workers=8)
        s.load_pgen()
        tl = cfg.default_tlim()
        t, _, _, _ = s.run(tlim=tl)
        blocks = [s.get_block(g) for g in range(cfg.nblocks)]
        errs.append(l1_error(cfg, blocks, t)[1])
    order = math.log2(errs[0] / errs[1])
    assert order >= TOL["order_min"], (errs, order)


def test_l1_error_fixture():
    cfg = small_wave(16)
    b = cfg.pgen_block(0)
    ex = cfg.exact_block(0, 0.0)
    b.u[:] = ex
    ks, js, is_ = cfg.active_slices()
    b.u[0, ks, js, is_] += 1e-3
    l1, comb = l1_error(cfg, [b], 0.0)
    assert abs(l1[0] - 1e-3) <= 1e-15 and np.all(l1[1:] == 0)


def test_unphysical_state_error_location():  # SPEC.md:136,213 ; defs.hpp:51-62
    cfg = RunConfig(nx1=8, nx2=8, nx3=8, mb1=8, mb2=8, mb3=8, pgen="uniform", rho=1, p=1e-3,
                    b1=0.0, b2=0.0, b3=0.0)
    s = O.OracleSolver(cfg)
    b = cfg.pgen_block(0)
    b.u[4, 2 + 3, 2 + 1, 2 + 6] = -1.0  # negative energy at global (k=3, j=1, i=6)
    s.set_block(0, b)
    s.exchange()
    from paper_1905_04341_b200 import UnphysicalStateError
    with pytest.raises(UnphysicalStateError) as ei:
        s.vl2_step(1e-3)
    assert (ei.value.stage_tag, ei.value.kk, ei.value.jj, ei.value.ii) == ("stage1", 3, 1, 6)


def test_floors_activate_and_count():
    cfg = RunConfig(nx1=8, nx2=8, nx3=8, mb1=8, mb2=8, mb3=8, pgen="uniform", rho=1, p=1e-3,
                    eos_mode="floor", pfloor=1e-2, dfloor=1e-3)
    s = O.OracleSolver(cfg)
    s.load_pgen()
    _, st = s.vl2_step(1e-4)
    assert st.floor_count == 2 * 512  # every active cell floored in both stages


def test_reference_exec_layer_bitwise():
    """The same restatement dispatched through the reference's own par_for /
    ThreadPool (/root/reference/proj/include/pmhd/exec/dispatch.hpp,
    src/thread_pool.cpp, compiled into oracle/_ref) gives bitwise-identical
    fields: the policy-equivalence contract SPEC.md:338,520."""
    ref_so = os.path.join(os.path.dirname(O.__file__), "_ref", "liboracle_ref.so")
    if not os.path.exists(ref_so):
        pytest.skip("oracle/_ref not built (reference absent)")
    out = []
    for ref, workers in ((False, 1), (True, 1), (True, 4)):
        cfg = small_wave(16, wave_n2=1, wave_amp=1e-3)
        s = O.OracleSolver(cfg, workers=workers, ref=ref)
        s.load_pgen()
        s.run(ncycles=3)
        out.append(s.get_block(0).u)
    assert np.array_equal(out[0], out[1]) and np.array_equal(out[0], out[2])


def test_counting_mode_bitwise_and_counts():
    cfg = small_wave(8, wave_amp=1e-3)
    a = O.OracleSolver(cfg)
    a.load_pgen()
    a.vl2_step(1e-3)
    O.flops_reset()
    c = O.OracleSolver(cfg, counting=True)
    c.load_pgen()
    c.vl2_step(1e-3)
    f = O.flops()
    assert np.array_equal(a.get_block(0).u, c.get_block(0).u)
    assert f.sum() > 1000 * cfg.active_cells


@pytest.mark.parametrize("riemann", ["hlld", "hlle"])
def test_orszag_tang_runs_to_half_time(riemann):
    """Nonlinear 2D robustness (BASELINE config 2): the standard Orszag-Tang
    vortex runs to t = 0.5 in error mode (no negative pressure), keeps div B at
    round-off and conserves mass.  (A wrong sign in the GS05 corner-EMF
    gradient terms makes this blow up at t ~ 0.07 while linear waves still
    converge.)"""
    cfg = RunConfig(nx1=64, nx2=64, nx3=1, mb1=32, mb2=32, mb3=1, pgen="orszag_tang", cfl=0.4,
                    riemann=riemann)
    s = O.OracleSolver(cfg, workers=8)
    s.load_pgen()
    m0 = s.sums()[0]
    t, n, _, _ = s.run(tlim=0.5)
    assert t == 0.5 and n > 100
    assert s.divb_max() <= 1e-12
    assert abs(s.sums()[0] - m0) <= 1e-13 * abs(m0)
    rho = np.concatenate([s.get_block(g).u[0].ravel() for g in range(cfg.nblocks)])
    assert rho.min() > 0.05


def test_blast_with_floors_long_run():
    cfg = RunConfig(nx1=24, nx2=24, nx3=24, mb1=12, mb2=12, mb3=12, x1min=-0.5, x1max=0.5,
                    x2min=-0.5, x2max=0.5, x3min=-0.5, x3max=0.5, pgen="blast", eos_mode="floor",
                    blast_r=0.2)
    s = O.OracleSolver(cfg, workers=8)
    s.load_pgen()
    e0 = s.sums()[4]
    _, _, _, floors = s.run(ncycles=40)
    e1 = s.sums()[4]
    assert np.isfinite(e1)
    if floors == 0:
        assert abs(e1 - e0) <= 1e-12 * abs(e0)
    else:  # pressure floors only ever add internal energy
        assert e1 >= e0 * (1 - 1e-12)
    assert s.divb_max() <= 1e-11
