"""GPU parity tests: the CUDA path (through the C-ABI, include/pmhd_gpu.h)
against the CPU oracle on the same seeded inputs.

* parity build (libpmhd_gpu_parity.so, --fmad=false): bit-identical fields,
  dt, floor counts and error locations;
* product build (libpmhd_gpu.so, FMA): per-cell scaled difference
  |a-b| <= 1e-11 * max(|b|, max_domain|b_q|) after N cycles (north_star
  tolerance), identical floor counts.
"""
import numpy as np
import pytest

from paper_1905_04341_b200 import RunConfig, UnphysicalStateError, ConfigError, l1_error
from paper_1905_04341_b200.solver import GpuSolver
from oracle.binding import OracleSolver

pytestmark = pytest.mark.gpu
TOL = 1e-11

CASES = {
    # name: (config kwargs, cycles)
    "wave3d_1blk": (dict(nx1=32, nx2=16, nx3=16, mb1=32, mb2=16, mb3=16, x2max=0.5, x3max=0.5,
                         wave_n1=1, wave_n2=1, wave_amp=1e-3), 5),
    "wave3d_4blk": (dict(nx1=32, nx2=16, nx3=16, mb1=16, mb2=16, mb3=8, x2max=0.5, x3max=0.5,
                         wave_n1=1, wave_n3=1, wave_mode=5, wave_amp=1e-3), 4),
    "ot2d_4blk": (dict(nx1=64, nx2=64, nx3=1, mb1=32, mb2=32, mb3=1, pgen="orszag_tang", cfl=0.4), 20),
    "blast3d_8blk_floor": (dict(nx1=32, nx2=32, nx3=32, mb1=16, mb2=16, mb3=16, x1min=-0.5, x1max=0.5,
                                x2min=-0.5, x2max=0.5, x3min=-0.5, x3max=0.5, pgen="blast",
                                eos_mode="floor", blast_r=0.2), 8),
    "wave3d_hlle_vl_arith": (dict(nx1=16, nx2=16, nx3=16, mb1=16, mb2=16, mb3=16, wave_n1=1,
                                  wave_n2=1, wave_n3=1, wave_amp=1e-2, riemann="hlle",
                                  limiter="vanleer", emf="arith"), 4),
    "turb3d": (dict(nx1=24, nx2=24, nx3=24, mb1=12, mb2=24, mb3=12, pgen="turbulence"), 4),
    "wave3d_roe": (dict(nx1=32, nx2=16, nx3=16, mb1=16, mb2=16, mb3=16, x2max=0.5, x3max=0.5,
                        wave_n1=1, wave_n2=1, wave_amp=1e-3, riemann="roe"), 4),
    "ot2d_roe": (dict(nx1=64, nx2=64, nx3=1, mb1=32, mb2=64, mb3=1, pgen="orszag_tang", cfl=0.4,
                      riemann="roe"), 20),
    # edge cases: ragged blocks (no tile divides them), ng = 3 / 4, tiny blocks
    # (4 cells: the x1 ghost push ranges of both sides cover the whole block)
    "wave3d_ng3_ragged": (dict(nx1=40, nx2=12, nx3=10, mb1=20, mb2=12, mb3=10, ng=3, x2max=0.3, x3max=0.25,
                               wave_n1=1, wave_amp=1e-3), 3),
    "wave3d_ng4_8blk": (dict(nx1=16, nx2=16, nx3=16, mb1=8, mb2=8, mb3=8, ng=4, wave_n1=1, wave_n2=1,
                             wave_n3=1, wave_amp=1e-3), 3),
    "wave3d_tiny_blocks": (dict(nx1=16, nx2=8, nx3=8, mb1=4, mb2=8, mb3=4, x2max=0.5, x3max=0.5, wave_n1=1,
                                wave_amp=1e-3), 3),
    "ot2d_ragged": (dict(nx1=48, nx2=40, nx3=1, mb1=24, mb2=20, mb3=1, x2max=40 / 48, pgen="orszag_tang",
                         cfl=0.4), 6),
    # a larger shock problem: 64^3 blast in 8 blocks, floors active
    "blast3d_64_floor": (dict(nx1=64, nx2=64, nx3=64, mb1=32, mb2=32, mb3=32, x1min=-0.5, x1max=0.5,
                              x2min=-0.5, x2max=0.5, x3min=-0.5, x3max=0.5, pgen="blast",
                              eos_mode="floor", blast_r=0.1), 5),
}


def run_pair(cfg, ncyc, parity):
    o = OracleSolver(cfg, workers=8)
    g = GpuSolver(cfg, parity=parity)
    o.load_pgen()
    g.load_pgen()
    dto, dtg = o.new_dt(), g.new_dt()
    init = (dto, dtg)
    fo = fg = 0
    dts = []
    for _ in range(ncyc):
        dno, sto = o.vl2_step(dto)
        dng, stg = g.vl2_step(dto)  # same dt sequence on both sides
        fo += sto.floor_count
        fg += stg.floor_count
        dts.append((dno, dng))
        dto = dno
    return o, g, init, (fo, fg), dts


def blocks(s, cfg):
    return [s.get_block(gid) for gid in range(cfg.nblocks)]


GROUPS = [(0,), (1, 2, 3), (4,), (5, 6, 7)]  # rho, momentum, energy, B


def scaled_diff(cfg, ref_blocks, gpu_blocks):
    """max over active cells of |a-b| / max(|a|, s_g): s_g = max over the
    domain of the variable's physical group (|m| for momenta, |B| for the
    field components), so a component that is zero up to round-off (e.g. Bz
    of the blast) is measured against the field scale, not its own noise."""
    ks, js, is_ = cfg.active_slices()
    A = np.stack([b.u[:, ks, js, is_] for b in ref_blocks])
    Bg = np.stack([b.u[:, ks, js, is_] for b in gpu_blocks])
    worst = 0.0
    for grp in GROUPS:
        s = max(float(np.max(np.abs(A[:, list(grp)]))), 1e-300)
        for q in grp:
            d = np.abs(A[:, q] - Bg[:, q]) / np.maximum(np.abs(A[:, q]), s)
            worst = max(worst, float(d.max()))
    return worst


@pytest.mark.parametrize("name", list(CASES))
def test_parity_build_bitwise(gpu_available, name):
    kw, ncyc = CASES[name]
    cfg = RunConfig(**kw)
    o, g, (d0o, d0g), (fo, fg), dts = run_pair(cfg, ncyc, parity=True)
    assert d0o == d0g
    for a, b in dts:
        assert a == b
    assert fo == fg
    for gid in range(cfg.nblocks):
        bo, bg = o.get_block(gid), g.get_block(gid)
        for f in ("u", "b1f", "b2f", "b3f"):
            x, y = getattr(bo, f), getattr(bg, f)
            if not np.array_equal(x, y):
                bad = np.argwhere(x != y)
                pytest.fail(f"{name} block {gid} field {f}: {len(bad)} mismatches, first {bad[:3].tolist()}"
                            f" oracle={x[tuple(bad[0])]!r} gpu={y[tuple(bad[0])]!r}")
    assert o.divb_max() == g.divb_max()
    assert np.array_equal(o.sums(), g.sums())


@pytest.mark.parametrize("name", list(CASES))
def test_fma_build_within_tolerance(gpu_available, name):
    kw, ncyc = CASES[name]
    cfg = RunConfig(**kw)
    o, g, _, (fo, fg), dts = run_pair(cfg, ncyc, parity=False)
    assert fo == fg
    for a, b in dts:
        assert abs(a - b) <= TOL * a
    worst = scaled_diff(cfg, blocks(o, cfg), blocks(g, cfg))
    assert worst <= TOL, worst
    assert g.divb_max() <= max(1e-11, 10 * o.divb_max())


@pytest.mark.parametrize("name", list(CASES))
def test_fma_build_fused_update_within_tolerance(gpu_available, name, monkeypatch):
    """The fused update kernel (PMHD_UPDATE=ldg; the two-kernel update is the
    default in 2D and 3D) in the FMA build stays within the oracle tolerance,
    as the default does."""
    monkeypatch.setenv("PMHD_UPDATE", "ldg")
    test_fma_build_within_tolerance(gpu_available, name)


@pytest.mark.parametrize("parity", [True, False])
def test_linear_wave_l1_and_order_on_gpu(gpu_available, parity):
    """Identical linear-wave L1 error and convergence order as the oracle
    (north_star): bitwise-identical L1 for the parity build; for the FMA build
    the L1 norms (~1e-8, of O(1) fields) agree to 1e-13 absolute."""
    errs_o, errs_g = [], []
    for n in (32, 64):
        cfg = RunConfig(nx1=n, nx2=8, nx3=8, mb1=n, mb2=8, mb3=8, x2max=8.0 / n, x3max=8.0 / n)
        tl = cfg.default_tlim()
        o = OracleSolver(cfg, workers=8)
        o.load_pgen()
        to, no, *_ = o.run(tlim=tl)
        g = GpuSolver(cfg, parity=parity)
        g.load_pgen()
        tg, ng_, *_ = g.run(tlim=tl)
        assert to == tg == tl and no == ng_
        errs_o.append(l1_error(cfg, blocks(o, cfg), to)[1])
        errs_g.append(l1_error(cfg, blocks(g, cfg), tg)[1])
    for a, b in zip(errs_o, errs_g):
        if parity:
            assert a == b
        else:
            assert abs(a - b) <= 1e-13
    order_o = np.log2(errs_o[0] / errs_o[1])
    order_g = np.log2(errs_g[0] / errs_g[1])
    assert order_g >= 1.9 and abs(order_o - order_g) <= 1e-3


def test_upload_download_roundtrip(gpu_available):
    cfg = RunConfig(nx1=16, nx2=12, nx3=8, mb1=8, mb2=12, mb3=8, pgen="turbulence")
    g = GpuSolver(cfg)
    rng = np.random.default_rng(0)
    for gid in range(cfg.nblocks):
        b = cfg.new_block()
        for f in ("u", "b1f", "b2f", "b3f"):
            getattr(b, f)[:] = rng.normal(size=getattr(b, f).shape)
        g.set_block(gid, b)
        r = g.get_block(gid)
        for f in ("b1f", "b2f", "b3f"):
            assert np.array_equal(getattr(b, f), getattr(r, f))
        assert np.array_equal(b.u[:5], r.u[:5])
        bcc1 = 0.5 * (b.b1f[:, :, :-1] + b.b1f[:, :, 1:])
        assert np.array_equal(r.u[5], bcc1)


def test_config_errors(gpu_available):
    with pytest.raises(ConfigError):
        GpuSolver(RunConfig(nx1=48, nx2=32, nx3=32, mb1=32, mb2=32, mb3=32))
    with pytest.raises(ConfigError):
        GpuSolver(RunConfig(nx1=16, nx2=16, nx3=16, mb1=16, mb2=16, mb3=16, ng=1))
    # maximum size: a block array must stay below 2^31 doubles (32-bit kernel
    # indexing) -- rejected before any device allocation
    with pytest.raises(ConfigError, match="too large"):
        GpuSolver(RunConfig(nx1=1300, nx2=1300, nx3=1300, mb1=1300, mb2=1300, mb3=1300))
    # launch-grid limit: every kernel folds the block index into gridDim.z
    # (<= 65535) with up to n+1 planes of a block; 256^3 in 16^3 blocks is
    # 4096 blocks x 21 -- rejected up front, not at the first launch
    with pytest.raises(ConfigError, match="too many MeshBlocks"):
        GpuSolver(RunConfig(nx1=256, nx2=256, nx3=256, mb1=16, mb2=16, mb3=16))


def test_upload_drops_pending_prefetch(gpu_available, monkeypatch):
    """A stage-2 prefetch (interior flux tiles on the second stream) that is
    followed by an upload instead of its stage: the upload waits for it and
    voids it, so the next cycle recomputes every tile and stays bit-identical
    to the oracle."""
    monkeypatch.setenv("PMHD_OVERLAP", "1")
    kw, _ = CASES["wave3d_4blk"]
    cfg = RunConfig(**kw)
    o = OracleSolver(cfg, workers=8)
    g = GpuSolver(cfg, parity=True)
    o.load_pgen()
    g.load_pgen()
    dt = o.new_dt()
    assert g.new_dt() == dt
    g.stage_compute(1, dt)
    g.stage_prefetch(2, dt)
    for gid in range(cfg.nblocks):  # overwrite the state: the prefetched fluxes are stale
        g.set_block(gid, o.get_block(gid))
    g.exchange()
    o.vl2_step(dt)
    g.vl2_step(dt)
    for gid in range(cfg.nblocks):
        assert np.array_equal(o.get_block(gid).u, g.get_block(gid).u)


def test_unphysical_error_matches_oracle(gpu_available):
    cfg = RunConfig(nx1=8, nx2=8, nx3=8, mb1=8, mb2=8, mb3=8, pgen="uniform", rho=1, p=1e-3,
                    b1=0.0, b2=0.0, b3=0.0)
    b = cfg.pgen_block(0)
    b.u[4, 2 + 3, 2 + 1, 2 + 6] = -1.0
    b.u[4, 2 + 5, 2 + 0, 2 + 2] = -1.0
    errs = []
    for s in (OracleSolver(cfg), GpuSolver(cfg, parity=True), GpuSolver(cfg)):
        s.set_block(0, b)
        s.exchange()
        with pytest.raises(UnphysicalStateError) as ei:
            s.vl2_step(1e-3)
        errs.append((ei.value.stage_tag, ei.value.kk, ei.value.jj, ei.value.ii))
    assert errs[0] == ("stage1", 3, 1, 6)
    assert errs[0] == errs[1] == errs[2]


def test_run_loop_lands_on_tlim(gpu_available):
    cfg = RunConfig(nx1=16, nx2=16, nx3=16, mb1=16, mb2=16, mb3=16)
    tl = 0.05
    o = OracleSolver(cfg)
    o.load_pgen()
    to, no, *_ = o.run(tlim=tl)
    g = GpuSolver(cfg, parity=True)
    g.load_pgen()
    tg, ng_, *_ = g.run(tlim=tl)
    assert to == tg == tl and no == ng_
    assert np.array_equal(o.get_block(0).u, g.get_block(0).u)


@pytest.mark.parametrize("variant", ["split", "fused"])
def test_kernel_variants_bitwise(gpu_available, variant, monkeypatch):
    """Both kernel organisations (one kernel per reference op, and the fused
    flux / fused update kernels) are bit-identical to the oracle."""
    monkeypatch.setenv("PMHD_KERNELS", variant)
    kw, ncyc = CASES["wave3d_4blk"]
    cfg = RunConfig(**kw)
    o, g, _, _, _ = run_pair(cfg, 3, parity=True)
    for gid in range(cfg.nblocks):
        assert np.array_equal(o.get_block(gid).u, g.get_block(gid).u)


@pytest.mark.parametrize("alt", ["tma", "ws", "emf", "emf_norim"])
@pytest.mark.parametrize("case", ["wave3d_4blk", "blast3d_8blk_floor", "wave3d_tiny_blocks", "wave3d_ng3_ragged",
                                  "wave3d_ng4_8blk", "turb3d", "blast3d_64_floor", "ot2d_ragged", "ot2d_4blk"])
def test_update_kernels_bitwise(gpu_available, case, alt, monkeypatch):
    """The TMA-staged (PMHD_UPDATE=tma), warp-specialised (PMHD_UPDATE=ws) and
    two-kernel (PMHD_UPDATE=emf: corner EMFs, then the cell update) forms and
    the default LDG update kernel compute the same
    expressions on the same operands: the
    parity build gives the same bits with either (the FMA build may contract
    a multiply-add differently in the two kernels; it is held to the oracle
    tolerance by test_fma_build_within_tolerance)."""
    kw, ncyc = CASES[case]
    cfg = RunConfig(**kw)
    out = []
    for kern in ("ldg", alt):
        # emf_norim: the edge-EMF kernel forms its upper-rim edges itself
        monkeypatch.setenv("PMHD_EMF_RIM", "0" if kern == "emf_norim" else "1")
        monkeypatch.setenv("PMHD_UPDATE", kern.split("_")[0])
        g = GpuSolver(cfg, parity=True)
        g.load_pgen()
        dt = g.new_dt()
        dts, floors = [], 0
        for _ in range(ncyc):
            dt, st = g.vl2_step(dt)
            dts.append(dt)
            floors += st.floor_count
        out.append((dts, floors, [g.get_block(gid) for gid in range(cfg.nblocks)]))
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    for b0, b1 in zip(out[0][2], out[1][2]):
        for f in ("u", "b1f", "b2f", "b3f"):
            assert np.array_equal(getattr(b0, f), getattr(b1, f)), (case, f)


@pytest.mark.parametrize("case", ["wave3d_4blk", "blast3d_8blk_floor", "ot2d_ragged", "ot2d_4blk",
                                  "wave3d_tiny_blocks", "wave3d_ng3_ragged", "wave3d_ng4_8blk", "wave3d_roe",
                                  "ot2d_roe", "wave3d_hlle_vl_arith", "turb3d"])
def test_flux_xy_bitwise(gpu_available, case, monkeypatch):
    """The x1 + x2 flux kernel (PMHD_FLUX_XY=1, owned-face ranges) and the
    default one launch per direction give the same bits in the parity build,
    2D (where it also writes the cell-centred E) and 3D."""
    kw, ncyc = CASES[case]
    cfg = RunConfig(**kw)
    out = []
    for xy in ("0", "1"):
        monkeypatch.setenv("PMHD_FLUX_XY", xy)
        g = GpuSolver(cfg, parity=True)
        g.load_pgen()
        dt = g.new_dt()
        dts = []
        for _ in range(ncyc):
            dt, _st = g.vl2_step(dt)
            dts.append(dt)
        out.append((dts, [g.get_block(gid) for gid in range(cfg.nblocks)]))
    assert out[0][0] == out[1][0]
    for b0, b1 in zip(out[0][1], out[1][1]):
        for f in ("u", "b1f", "b2f", "b3f"):
            assert np.array_equal(getattr(b0, f), getattr(b1, f)), (case, f)


@pytest.mark.parametrize("reuse", ["0", "1"])
@pytest.mark.parametrize("case", ["wave3d_4blk", "blast3d_8blk_floor", "ot2d_ragged", "wave3d_tiny_blocks",
                                  "wave3d_ng3_ragged", "wave3d_roe", "wave3d_hlle_vl_arith"])
def test_flux_kernels_bitwise(gpu_available, case, reuse, monkeypatch):
    """The column-march x2 / x3 and row-march x1 flux kernels (the stage-2
    default; forced here in both stages) and the tile kernels
    (PMHD_FLUX_MARCH=0) give the same bits in the parity build, with the
    owned-face ranges and with the extended ones."""
    kw, ncyc = CASES[case]
    cfg = RunConfig(**kw)
    monkeypatch.setenv("PMHD_FACE_REUSE", reuse)
    monkeypatch.setenv("PMHD_FLUX_MARCH_X1", "1")  # the x1 row march too
    monkeypatch.setenv("PMHD_FLUX_MARCH_STAGES", "3")  # in both stages (default: stage 2)
    out = []
    for march in ("0", "2"):  # 2: the march kernels even on these small meshes
        monkeypatch.setenv("PMHD_FLUX_MARCH", march)
        g = GpuSolver(cfg, parity=True)
        g.load_pgen()
        dt = g.new_dt()
        dts = []
        for _ in range(ncyc):
            dt, _st = g.vl2_step(dt)
            dts.append(dt)
        out.append((dts, [g.get_block(gid) for gid in range(cfg.nblocks)]))
    assert out[0][0] == out[1][0]
    for b0, b1 in zip(out[0][1], out[1][1]):
        for f in ("u", "b1f", "b2f", "b3f"):
            assert np.array_equal(getattr(b0, f), getattr(b1, f)), (case, f)


@pytest.mark.parametrize("case", ["wave3d_4blk", "blast3d_8blk_floor", "ot2d_ragged", "wave3d_tiny_blocks",
                                  "wave3d_ng3_ragged", "turb3d"])
def test_face_reuse_bitwise(gpu_available, case, monkeypatch):
    """Owned-face reuse (flux tiles over [s, e) only, halo faces and cell E
    stored as rim images by their owners) leaves the product (FMA) build's
    results unchanged bit for bit: the images are the values the extended
    face ranges computed from the exact ghost copies."""
    kw, ncyc = CASES[case]
    cfg = RunConfig(**kw)
    out = []
    for reuse in ("0", "1"):
        monkeypatch.setenv("PMHD_FACE_REUSE", reuse)
        g = GpuSolver(cfg)
        g.load_pgen()
        dt = g.new_dt()
        dts = []
        for _ in range(ncyc):
            dt, _st = g.vl2_step(dt)
            dts.append(dt)
        out.append((dts, [g.get_block(gid) for gid in range(cfg.nblocks)]))
    assert out[0][0] == out[1][0]
    for b0, b1 in zip(out[0][1], out[1][1]):
        for f in ("u", "b1f", "b2f", "b3f"):
            assert np.array_equal(getattr(b0, f), getattr(b1, f)), (case, f)


@pytest.mark.parametrize("conc", ["2", "3"])
@pytest.mark.parametrize("case", ["wave3d_4blk", "blast3d_8blk_floor", "ot2d_ragged", "turb3d"])
def test_flux_streams_bitwise(gpu_available, case, conc, monkeypatch):
    """Flux launches of a stage on two or three streams (PMHD_FLUX_CONC; 1,
    x2 beside x1 -> x3, is the default) give the serial order's results bit
    for bit in the product build: the launches write disjoint arrays and the
    update waits for all of them."""
    kw, ncyc = CASES[case]
    cfg = RunConfig(**kw)
    out = []
    for c in ("0", "1", conc):
        monkeypatch.setenv("PMHD_FLUX_CONC", c)
        g = GpuSolver(cfg)
        g.load_pgen()
        dt = g.new_dt()
        dts = []
        for _ in range(ncyc):
            dt, _st = g.vl2_step(dt)
            dts.append(dt)
        out.append((dts, [g.get_block(gid) for gid in range(cfg.nblocks)]))
    for o in out[1:]:
        assert o[0] == out[0][0]
        for b0, b1 in zip(out[0][1], o[1]):
            for f in ("u", "b1f", "b2f", "b3f"):
                assert np.array_equal(getattr(b0, f), getattr(b1, f)), (case, f)


@pytest.mark.parametrize("case", ["wave3d_4blk", "blast3d_8blk_floor", "ot2d_ragged", "turb3d", "wave3d_tiny_blocks"])
def test_early_x1_flux_bitwise(gpu_available, case, monkeypatch):
    """The stage-1 x2 / x3 ghost exchanges on a third stream, overlapping the
    stage-2 x1 flux launch (PMHD_EARLY_X1, on for meshes up to 2^24 cells),
    give the serial order's bits in the product build, also when the run
    loop replays the cycle as a CUDA graph."""
    kw, ncyc = CASES[case]
    cfg = RunConfig(**kw)
    out = []
    for e in ("0", "1"):
        monkeypatch.setenv("PMHD_EARLY_X1", e)
        g = GpuSolver(cfg)
        g.load_pgen()
        dt = g.new_dt()
        dts = []
        for _ in range(ncyc):
            dt, _st = g.vl2_step(dt)
            dts.append(dt)
        out.append((dts, [g.get_block(gid) for gid in range(cfg.nblocks)]))
    assert out[0][0] == out[1][0]
    for b0, b1 in zip(out[0][1], out[1][1]):
        for f in ("u", "b1f", "b2f", "b3f"):
            assert np.array_equal(getattr(b0, f), getattr(b1, f)), (case, f)


@pytest.mark.parametrize("march", ["1", "2"])
@pytest.mark.parametrize("case", ["wave3d_4blk", "blast3d_8blk_floor", "ot2d_4blk"])
def test_overlap_prefetch_bitwise(gpu_available, case, march, monkeypatch):
    """Stage-2 interior flux tiles enqueued on a second stream while the
    stage-1 ghost exchange runs (PMHD_OVERLAP=1; on by default only with
    remote neighbours) are bit-identical to the oracle; march "2" forces the
    column-march x2 / x3 kernels (their region split) on these small meshes."""
    monkeypatch.setenv("PMHD_OVERLAP", "1")
    monkeypatch.setenv("PMHD_FLUX_MARCH", march)
    monkeypatch.setenv("PMHD_FLUX_MARCH_STAGES", "3")
    kw, ncyc = CASES[case]
    cfg = RunConfig(**kw)
    o, g, _, (fo, fg), dts = run_pair(cfg, ncyc, parity=True)
    assert fo == fg
    for a, b in dts:
        assert a == b
    for gid in range(cfg.nblocks):
        bo, bg = o.get_block(gid), g.get_block(gid)
        for f in ("u", "b1f", "b2f", "b3f"):
            assert np.array_equal(getattr(bo, f), getattr(bg, f)), (case, gid, f)


@pytest.mark.parametrize("slab", [16, 32])
@pytest.mark.parametrize("case", ["blast", "wave"])
def test_kslab_pipeline_bitwise(gpu_available, slab, case, monkeypatch):
    """The two-stream k-slab pipeline (flux kernels of slab q+1 overlapping
    the update kernel of slab q) is bit-identical to the oracle."""
    monkeypatch.setenv("PMHD_SLAB_PLANES", str(slab))
    if case == "blast":
        kw = dict(nx1=32, nx2=32, nx3=64, mb1=32, mb2=16, mb3=32, x1min=-0.5, x1max=0.5,
                  x2min=-0.5, x2max=0.5, x3min=-1.0, x3max=1.0, pgen="blast", eos_mode="floor",
                  blast_r=0.2)
    else:
        kw = dict(nx1=16, nx2=16, nx3=64, mb1=16, mb2=16, mb3=64, x3max=4.0, wave_n1=1, wave_n3=1,
                  wave_amp=1e-3)
    cfg = RunConfig(**kw)
    o, g, _, (fo, fg), dts = run_pair(cfg, 3, parity=True)
    assert fo == fg
    for a, b in dts:
        assert a == b
    for gid in range(cfg.nblocks):
        bo, bg = o.get_block(gid), g.get_block(gid)
        for f in ("u", "b1f", "b2f", "b3f"):
            assert np.array_equal(getattr(bo, f), getattr(bg, f)), (gid, f)


MULTIRANK = {
    "wave": dict(nx1=32, nx2=16, nx3=16, mb1=8, mb2=8, mb3=8, x2max=0.5, x3max=0.5, wave_n1=1,
                 wave_n2=1, wave_amp=1e-3),
    "blast": CASES["blast3d_8blk_floor"][0],
    "ot2d": CASES["ot2d_4blk"][0],
}


@pytest.mark.parametrize("nranks,stream_ordered,case,p2p", [(2, False, "wave", False), (4, False, "wave", False),
                                                            (2, True, "wave", False), (4, True, "wave", False),
                                                            (2, True, "blast", False), (4, True, "ot2d", False),
                                                            (2, False, "wave", True), (4, False, "blast", True),
                                                            (4, False, "ot2d", True), (8, False, "blast", True),
                                                            (8, True, "blast", False)])
@pytest.mark.parametrize("march", ["1", "2"])
def test_multirank_halo_path_bitwise(gpu_available, nranks, stream_ordered, case, p2p, march, monkeypatch):
    """The multi-rank data path (stage_compute + local sweeps + halo pack /
    unpack kernels + transport) with nranks rank-engines on ONE GPU, stepped in
    lockstep by the host (no kernel waits on another), is bit-identical to the
    oracle: the GPU side of SURVEY.md §8e.  stream_ordered: the async ABI mode
    with the hand-over ordered by events between the engines' streams (what
    DistributedVL2 does with NCCL), i.e. no host synchronization in a stage.
    p2p: remote faces read straight from the other engines' memory by the
    exchange kernels (pmhd_gpu_peer_attach), no pack / unpack.  march "2":
    the column-march x2 / x3 kernels forced on these small meshes, so their
    interior / boundary split (the halo overlap) is covered too, and the
    two-kernel update (edge EMFs + cell update; in 3D, without the rim
    stores, since the neighbours are remote)."""
    from paper_1905_04341_b200.parallel import plan_for, LoopbackWorld
    monkeypatch.setenv("PMHD_FLUX_MARCH", march)
    monkeypatch.setenv("PMHD_FLUX_MARCH_STAGES", "3")
    monkeypatch.setenv("PMHD_UPDATE", "emf" if march == "2" else "ldg")
    cfg = RunConfig(**MULTIRANK[case])
    plan = plan_for(cfg, nranks)
    engines = [GpuSolver(cfg, parity=True, gids=plan.local_gids(r)) for r in range(nranks)]
    for e in engines:
        e.load_pgen(exchange=False)
    world = LoopbackWorld(engines, plan, stream_ordered=stream_ordered, p2p=p2p)
    world.exchange(half=0)
    if stream_ordered:
        for s in world.streams:
            s.synchronize()
    o = OracleSolver(cfg, workers=8)
    o.load_pgen()
    dt = o.new_dt()
    assert min(e.new_dt() for e in engines) == dt
    for _ in range(3):
        dto, _ = o.vl2_step(dt)
        dtg = world.vl2_step(dt)
        assert dto == dtg
        dt = dto
    for r, e in enumerate(engines):
        for gid in plan.local_gids(r):
            assert np.array_equal(e.get_block(gid).u, o.get_block(gid).u), (r, gid)


@pytest.mark.parametrize("parity", [True, False])
def test_driven_turbulence(gpu_available, parity):
    """Turbulence driving: kicks between VL2 cycles; the
    parity build is bit-identical to the oracle (dv, the ordered sums, the
    impulse and the cycles after it), the FMA build within 1e-11."""
    from paper_1905_04341_b200.drive import TurbulenceDriver
    cfg = RunConfig(nx1=24, nx2=24, nx3=24, mb1=12, mb2=24, mb3=12, pgen="turbulence", turb_drive=1,
                    turb_dedt=2.0, turb_every=2)
    o, g = OracleSolver(cfg, workers=8), GpuSolver(cfg, parity=parity)
    o.load_pgen()
    g.load_pgen()
    drv = TurbulenceDriver(cfg)
    dt, acc, event = o.new_dt(), 0.0, 0
    for n in range(6):
        dno, _ = o.vl2_step(dt)
        g.vl2_step(dt)
        acc += dt
        dt = dno
        if (n + 1) % 2 == 0:
            so = drv.kick(o, event, drv.energy(acc))
            sg = drv.kick(g, event, drv.energy(acc))
            if parity:
                assert so == sg
            else:
                assert abs(so - sg) <= TOL * so
            acc, event = 0.0, event + 1
            dt = o.new_dt()
            if parity:
                assert g.new_dt() == dt
    if parity:
        for gid in range(cfg.nblocks):
            bo, bg = o.get_block(gid), g.get_block(gid)
            for f in ("u", "b1f", "b2f", "b3f"):
                assert np.array_equal(getattr(bo, f), getattr(bg, f)), (gid, f)
    else:
        assert scaled_diff(cfg, blocks(o, cfg), blocks(g, cfg)) <= TOL


@pytest.mark.parametrize("graph", ["1", "0"])
@pytest.mark.parametrize("case,ncyc", [("blast3d_8blk_floor", 5), ("ot2d_4blk", 7), ("wave3d_roe", 3)])
def test_run_loop_graph_replay_bitwise(gpu_available, graph, case, ncyc, monkeypatch):
    """pmhd_gpu_run with the cycle captured as a CUDA graph and the dt / t /
    floor bookkeeping on the device (PMHD_GRAPH=1, the default) and with the
    host loop (0): both bit-identical to the oracle's run loop, odd cycle
    counts included (the state ends in the other table), then more cycles
    through vl2_step continue from the right table."""
    monkeypatch.setenv("PMHD_GRAPH", graph)
    cfg = RunConfig(**CASES[case][0])
    o, g = OracleSolver(cfg, workers=8), GpuSolver(cfg, parity=True)
    o.load_pgen()
    g.load_pgen()
    to, no, dto, fo = o.run(ncycles=ncyc)
    tg, ng_, dtg, fg = g.run(ncycles=ncyc)
    assert (to, no, dto, fo) == (tg, ng_, dtg, fg)
    for _ in range(2):
        dto, _ = o.vl2_step(dto)
        dtg, _ = g.vl2_step(dtg)
        assert dto == dtg
    for gid in range(cfg.nblocks):
        bo, bg = o.get_block(gid), g.get_block(gid)
        for f in ("u", "b1f", "b2f", "b3f"):
            assert np.array_equal(getattr(bo, f), getattr(bg, f)), (case, gid, f)


def test_run_loop_graph_error(gpu_available):
    """An unphysical state met inside a graph-replayed run is reported like
    the host loop reports it (stage tag and global cell)."""
    cfg = RunConfig(nx1=8, nx2=8, nx3=8, mb1=8, mb2=8, mb3=8, pgen="uniform", rho=1, p=1e-3,
                    b1=0.0, b2=0.0, b3=0.0)
    b = cfg.pgen_block(0)
    b.u[4, 2 + 3, 2 + 1, 2 + 6] = -1.0
    errs = []
    for s in (OracleSolver(cfg), GpuSolver(cfg, parity=True)):
        s.set_block(0, b)
        s.exchange()
        with pytest.raises(UnphysicalStateError) as ei:
            s.run(ncycles=4, dt=1e-3)
        errs.append((ei.value.stage_tag, ei.value.kk, ei.value.jj, ei.value.ii))
    assert errs[0] == errs[1] == ("stage1", 3, 1, 6)


def test_gpu_restart_bitwise_continuous(gpu_available, tmp_path):
    """PMHD1 snapshot / restart on the GPU path: 3 cycles,
    snapshot, a fresh mesh restarted from the file, 3 more cycles == 6
    uninterrupted cycles, bit for bit (parity build)."""
    cfg = RunConfig(**CASES["blast3d_8blk_floor"][0])
    ref = GpuSolver(cfg, parity=True)
    ref.load_pgen()
    dt = ref.new_dt()
    dts = []
    for _ in range(6):
        dt, _ = ref.vl2_step(dt)
        dts.append(dt)
    a = GpuSolver(cfg, parity=True)
    a.load_pgen()
    dt = a.new_dt()
    for _ in range(3):
        dt, _ = a.vl2_step(dt)
    p = tmp_path / "r.pmhd"
    cfg.snapshot_write(p, [a.get_block(g) for g in range(cfg.nblocks)], 0.0)
    del a
    blocks, _ = cfg.snapshot_read(p)
    b = GpuSolver(cfg, parity=True)
    for g, blk in enumerate(blocks):
        b.set_block(g, blk)
    b.exchange()
    for q in range(3):
        dt, _ = b.vl2_step(dt)
        assert dt == dts[3 + q]
    for g in range(cfg.nblocks):
        assert np.array_equal(ref.get_block(g).u, b.get_block(g).u), g


def _ipc_worker(rank, world, port, kw, ncyc, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1905_04341_b200.parallel import plan_for, DistributedVL2, TorchDistTransport
        cfg = RunConfig(**kw)
        plan = plan_for(cfg, world)
        eng = GpuSolver(cfg, parity=True, gids=plan.local_gids(rank))
        eng.load_pgen(exchange=False)
        drv = DistributedVL2(eng, plan, rank, TorchDistTransport(dist, host_staging=True))
        assert drv.p2p  # peer-memory halo over CUDA IPC
        drv.exchange(half=0)
        dt = drv.new_dt()
        for _ in range(ncyc):
            dt, _ = drv.vl2_step(dt)
        q.put((rank, dt, {gid: eng.get_block(gid).u for gid in eng.gids}))
    finally:
        dist.destroy_process_group()


def test_ipc_peer_halo_two_processes(gpu_available):
    """Two rank processes on one GPU, halo read over CUDA IPC peer memory
    (host barriers between sweep directions, no kernel waits on another):
    bit-identical to the oracle in one process."""
    import socket
    import torch.multiprocessing as mp
    kw = MULTIRANK["blast"]
    cfg = RunConfig(**kw)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, kw, 3, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    o = OracleSolver(cfg, workers=8)
    o.load_pgen()
    dt = o.new_dt()
    for _ in range(3):
        dt, _ = o.vl2_step(dt)
    for rank, dtr, blocks in res:
        assert dtr == dt
        for gid, u in blocks.items():
            assert np.array_equal(u, o.get_block(gid).u), (rank, gid)
