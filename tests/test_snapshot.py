"""PMHD1 snapshot / restart: the file
layout, a bitwise write -> read round trip, and restart continuity (3 + 3
cycles through a snapshot == 6 uninterrupted cycles, bitwise)."""
import struct

import numpy as np
import pytest

from paper_1905_04341_b200 import RunConfig, ParseError
from oracle.binding import OracleSolver

CFG = dict(nx1=32, nx2=16, nx3=16, mb1=16, mb2=8, mb3=16, x2max=0.5, x3max=0.5, wave_n1=1,
           wave_n2=1, wave_amp=1e-3)


def test_snapshot_layout_and_roundtrip(tmp_path):
    cfg = RunConfig(**CFG)
    blocks = [cfg.pgen_block(g) for g in range(cfg.nblocks)]
    p = tmp_path / "s.pmhd"
    cfg.snapshot_write(p, blocks, 0.125)
    raw = p.read_bytes()
    hdr_end = raw.index(b"END\n") + 4
    assert raw[:hdr_end].decode().splitlines() == ["PMHD1", "dims 32 16 16",
                                                   f"gamma {5.0 / 3.0!r}".replace("1.6666666666666667", "1.6666666666666667"),
                                                   "time 0.125", "END"]
    n = 32 * 16 * 16
    nfaces = 33 * 16 * 16 + 32 * 17 * 16 + 32 * 16 * 17
    assert len(raw) - hdr_end == 8 * (8 * n + nfaces)
    # first payload value = rho of global cell (0,0,0) = block 0, local (2,2,2)
    assert struct.unpack("<d", raw[hdr_end:hdr_end + 8])[0] == blocks[0].u[0, 2, 2, 2]
    back, t = cfg.snapshot_read(p)
    assert t == 0.125
    ks, js, is_ = cfg.active_slices()
    for b0, b1 in zip(blocks, back):
        assert np.array_equal(b0.u[:, ks, js, is_], b1.u[:, ks, js, is_])
        assert np.array_equal(b0.b1f[ks, js, 2:-2], b1.b1f[ks, js, 2:-2])
        assert np.array_equal(b0.b2f[ks, 2:-2, is_], b1.b2f[ks, 2:-2, is_])
        assert np.array_equal(b0.b3f[2:-2, js, is_], b1.b3f[2:-2, js, is_])


def test_snapshot_rejects_other_mesh(tmp_path):
    cfg = RunConfig(**CFG)
    p = tmp_path / "s.pmhd"
    cfg.snapshot_write(p, [cfg.pgen_block(g) for g in range(cfg.nblocks)], 0.0)
    other = RunConfig(**dict(CFG, nx1=64, mb1=32))
    with pytest.raises(ParseError):
        other.snapshot_read(p)


@pytest.mark.parametrize("kw", [CFG, dict(nx1=32, nx2=32, nx3=1, mb1=16, mb2=16, mb3=1,
                                          pgen="orszag_tang", cfl=0.4)])
def test_restart_is_bitwise_continuous(tmp_path, kw):
    cfg = RunConfig(**kw)
    ref = OracleSolver(cfg, workers=4)
    ref.load_pgen()
    ref.run(ncycles=6)
    a = OracleSolver(cfg, workers=4)
    a.load_pgen()
    t, _, _, _ = a.run(ncycles=3)
    p = tmp_path / "r.pmhd"
    cfg.snapshot_write(p, [a.get_block(g) for g in range(cfg.nblocks)], t)
    blocks, t2 = cfg.snapshot_read(p)
    assert t2 == t
    b = OracleSolver(cfg, workers=4)
    for g, blk in enumerate(blocks):
        b.set_block(g, blk)
    b.exchange()
    b.run(ncycles=3)
    for g in range(cfg.nblocks):
        assert np.array_equal(ref.get_block(g).u, b.get_block(g).u)
