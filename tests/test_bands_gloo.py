"""Row-band decomposition and halo exchange (paper_2112_09728_b200.bands)
across 2 and 3 processes with the gloo backend on CPU: every rank ends up
with exactly the full-frame rows its extended buffers cover."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2112_09728_b200.bands import Extent, band_rows, check_band_geometry, gather_rows, halo_exchange


def test_band_rows_partition():
    for h in (1, 7, 1080, 4321):
        for world in (1, 2, 3, 8):
            if world > h:
                continue
            rows = [band_rows(h, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == h
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            sizes = [r1 - r0 for r0, r1 in rows]
            assert max(sizes) - min(sizes) <= 1


def test_extent_and_geometry():
    e = Extent.around(100, 200, 10, 1080)
    assert (e.lo, e.hi, e.rows) == (90, 210, 120)
    e = Extent.around(0, 50, 10, 60)
    assert (e.lo, e.hi) == (0, 60)
    t = torch.arange(60 * 2).reshape(60, 2)
    assert torch.equal(e.own(t), t[0:50])
    check_band_geometry(1080, 8, 10)
    with pytest.raises(ValueError):
        check_band_geometry(40, 8, 10)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H, W, halo, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        full_a = torch.rand(H, W, 4, generator=g)                       # a float4 plane (Pi / Gamma)
        full_b = (torch.rand(H, W, generator=g) * 255).to(torch.uint8)   # a flag plane
        r0, r1 = band_rows(H, world, rank)
        ext = Extent.around(r0, r1, halo, H)
        a = torch.full((ext.rows, W, 4), -1.0)
        b = torch.zeros(ext.rows, W, dtype=torch.uint8)
        ext.own(a).copy_(full_a[r0:r1])        # each rank only knows its own band
        ext.own(b).copy_(full_b[r0:r1])
        halo_exchange([a, b], ext, rank, world, tag=3)
        ok = torch.equal(a, full_a[ext.lo:ext.hi]) and torch.equal(b, full_b[ext.lo:ext.hi])
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,halo", [(2, 64, 10), (3, 50, 10), (2, 31, 2)])
def test_halo_exchange_gloo(world, H, halo):
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, 24, halo, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert list(out) == [1] * world


def _gather_worker(rank, world, port, H, W, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(11)
        full_a = torch.rand(H, W, 4, generator=g)
        full_b = (torch.rand(H, W, generator=g) * 255).to(torch.uint8)
        r0, r1 = band_rows(H, world, rank)
        a, b = gather_rows([full_a[r0:r1].clone(), full_b[r0:r1].clone()], rank, world, H)
        out[rank] = 1 if (torch.equal(a, full_a) and torch.equal(b, full_b)) else 0
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H", [(2, 31), (3, 50)])
def test_gather_rows_gloo(world, H):
    """The full-history fallback's all-gather of unequal row bands."""
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, H, 20, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert list(out) == [1] * world
