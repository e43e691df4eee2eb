"""Multi-rank host logic on CPU (gloo, world size 2): view sharding + gradient
all-reduce reproduces the single-process sum over views (the reference's
per-view accumulate semantics, rasterizer.cpp:329-331); z-slab sharding of the
voxelizer partitions the bricks and the all-reduced partial gradients equal
the full gradient. The per-rank compute here is the CPU oracle (test
infrastructure); on GPUs the same host logic drives the engine (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2405_20693_b200 import dist as pdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from oracle import oracle as O
    cl = O.random_cloud(O.Rng(11), 60, 0.7, 0.03, 0.15)
    thetas = O.full_circle_angles(5)
    ups = [np.random.default_rng(100 + v).uniform(-1, 1, (48, 48)) for v in range(5)]
    return cl, thetas, ups


def _raster_grads(cl, thetas, ups, views):
    from oracle import oracle as O
    g = O.Grads.zeros(cl.m)
    cfg = O.test_scanner(48)
    for v in views:
        r = O.render(cl, cfg, thetas[v])
        O.render_backward(cl, cfg, thetas[v], r, ups[v], g)
    return g.flat()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cl, thetas, ups = _scene()
        mine = pdist.shard_views(len(thetas), rank, world)
        g = torch.from_numpy(_raster_grads(cl, thetas, ups, mine))
        pdist.allreduce_([g])
        # voxelizer z-slabs: partial gradient from this rank's brick layers
        from oracle import oracle as O
        grid = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (24, 24, 24))
        up = np.random.default_rng(3).uniform(-1, 1, grid.shape_zyx)
        z0, z1 = pdist.shard_z_bricks(3, rank, world)
        mask = np.zeros_like(up)
        mask[8 * z0:8 * z1] = 1.0
        gv = O.Grads.zeros(cl.m)
        O.voxelize_backward(cl, grid, up * mask, gv)
        gvt = torch.from_numpy(gv.flat())
        pdist.allreduce_([gvt])
        if rank == 0:
            out.put((g.numpy(), gvt.numpy()))
    finally:
        dist.destroy_process_group()


def test_view_sharding_and_slab_allreduce_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    g_dist, gv_dist = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cl, thetas, ups = _scene()
    g_full = _raster_grads(cl, thetas, ups, range(len(thetas)))
    np.testing.assert_allclose(g_dist, g_full, rtol=1e-10, atol=1e-12)
    from oracle import oracle as O
    grid = O.grid_for_extent((-1, -1, -1), (1, 1, 1), (24, 24, 24))
    up = np.random.default_rng(3).uniform(-1, 1, grid.shape_zyx)
    gv = O.Grads.zeros(cl.m)
    O.voxelize_backward(cl, grid, up, gv)
    np.testing.assert_allclose(gv_dist, gv.flat(), rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("n,world", [(75, 1), (75, 2), (75, 8), (5, 8), (100, 3)])
def test_shard_views_partition(n, world):
    seen = []
    for r in range(world):
        v = pdist.shard_views(n, r, world)
        seen += v
        assert len(v) in (n // world, n // world + 1)
    assert sorted(seen) == list(range(n))


@pytest.mark.parametrize("layers,world", [(32, 1), (32, 8), (5, 8), (33, 4)])
def test_shard_z_bricks_partition(layers, world):
    cuts = [pdist.shard_z_bricks(layers, r, world) for r in range(world)]
    assert cuts[0][0] == 0 and cuts[-1][1] == layers
    for a, b in zip(cuts, cuts[1:]):
        assert a[1] == b[0]
    w = np.abs(np.sin(np.arange(layers))) + 0.1
    cuts = [pdist.shard_z_bricks(layers, r, world, list(w)) for r in range(world)]
    assert cuts[0][0] == 0 and cuts[-1][1] == layers
    for a, b in zip(cuts, cuts[1:]):
        assert a[1] == b[0]
