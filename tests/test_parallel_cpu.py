"""Multi-rank path on CPU: world_size 2 (and 4) over gloo, the CPU oracle as
the rank engine, halo slabs through torch.distributed point-to-point.  The
sharded run must be bit-identical to the single-process run (decomposition
independence lifted to ranks)."""
import os
import socket

import numpy as np
import pytest

from paper_1905_04341_b200 import RunConfig
from paper_1905_04341_b200.parallel import partition, plan_for, HaloPlan

CFG = dict(nx1=32, nx2=16, nx3=16, mb1=8, mb2=8, mb3=8, x2max=0.5, x3max=0.5, wave_n1=1,
           wave_n2=1, wave_amp=1e-3)
CFG2D = dict(nx1=64, nx2=64, nx3=1, mb1=16, mb2=32, mb3=1, pgen="orszag_tang", cfl=0.4)
# 2 x 2 x 2 blocks on 8 ranks: every neighbour remote, the same rank on both sides
CFG8 = dict(nx1=16, nx2=16, nx3=16, mb1=8, mb2=8, mb3=8, wave_n1=1, wave_n2=1, wave_amp=1e-3)
CFGTURB = dict(nx1=16, nx2=16, nx3=16, mb1=8, mb2=8, mb3=8, pgen="turbulence", turb_drive=1,
               turb_dedt=0.5, turb_every=2)


def test_partition_bricks():
    own = partition((4, 2, 2), 2)
    assert sorted(set(own)) == [0, 1] and own.count(0) == 8
    own8 = partition((4, 2, 2), 8)
    assert sorted(set(own8)) == list(range(8))
    with pytest.raises(ValueError):
        partition((3, 1, 1), 2)


def test_plan_messages_pair_up():
    cfg = RunConfig(**CFG)
    plan = plan_for(cfg, 4)
    for d in range(3):
        sends = {}
        recvs = {}
        for r in range(4):
            s, rc = plan.messages(r, d)
            for peer, key, gid, side in s:
                sends[(r, peer, key)] = 1
            for peer, key in rc:
                recvs[(peer, r, key)] = 1
        assert set(sends) == set(recvs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg_kw, ncyc, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.binding import OracleSolver
        from paper_1905_04341_b200.parallel import DistributedVL2, TorchDistTransport
        cfg = RunConfig(**cfg_kw)
        plan = plan_for(cfg, world)
        eng = OracleSolver(cfg, workers=1, gids=plan.local_gids(rank))
        eng.load_pgen(exchange=False)
        drv = DistributedVL2(eng, plan, rank, TorchDistTransport(dist))
        drv.exchange(half=0)
        dt = drv.new_dt()
        driver = None
        if cfg.c.turb_drive:
            from paper_1905_04341_b200.drive import TurbulenceDriver
            driver = TurbulenceDriver(cfg)
        acc, event = 0.0, 0
        for n in range(ncyc):  # the loop of drive.run_driven, across ranks
            dn, _ = drv.vl2_step(dt)
            acc += dt
            dt = dn
            if driver is not None and (n + 1) % cfg.c.turb_every == 0:
                drv.kick(driver, event, driver.energy(acc))
                acc, event = 0.0, event + 1
                dt = drv.new_dt()
        out = {gid: eng.get_block(gid).u for gid in eng.gids}
        q.put((rank, dt, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg_kw", [(2, CFG), (4, CFG), (2, CFG2D), (2, CFGTURB), (8, CFG8)])
def test_gloo_sharded_equals_single_process(world, cfg_kw):
    import torch.multiprocessing as mp
    from oracle.binding import OracleSolver
    ncyc = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_kw, ncyc, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = RunConfig(**cfg_kw)
    ref = OracleSolver(cfg, workers=4)
    ref.load_pgen()
    if cfg.c.turb_drive:
        from paper_1905_04341_b200.drive import run_driven
        _, dt, _ = run_driven(ref, cfg, ncyc)
    else:
        dt = ref.new_dt()
        for _ in range(ncyc):
            dt, _ = ref.vl2_step(dt)
    seen = set()
    for rank, dtr, blocks in results:
        assert dtr == dt
        for gid, u in blocks.items():
            assert np.array_equal(u, ref.get_block(gid).u), (rank, gid)
            seen.add(gid)
    assert seen == set(range(cfg.nblocks))
