"""NCCL-aware entry points (comm.cu) on one GPU: a
world-size-1 communicator made through the C-ABI. The sum over one rank is the
identity, so the fused backward+all-reduce variants must equal the plain
backward and keep its accumulate (+=) contract. (Multi-rank sharding logic is
covered on CPU with gloo in test_dist_cpu.py; this box has one GPU.)"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests import _golden as G  # noqa: E402


def _setup():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    s_min, *arrs = G.cloud_arrays()
    return P, s_min, arrs


def test_comm_required_and_info():
    P, s_min, arrs = _setup()
    eng = P.Engine(0)
    c = P.GaussianCloud(s_min, *arrs)
    g = P.CloudGrads(c.size())
    with pytest.raises(P.ConfigError):
        eng.allreduce_grads(g)
    eng.comm_init(0, 1)
    assert eng.comm_info() == (1, 0)
    g.buffer.copy_(torch.arange(g.buffer.numel(), dtype=torch.float32))
    eng.allreduce_grads(g, c)
    torch.cuda.synchronize()
    assert torch.equal(g.buffer.cpu(), torch.arange(g.buffer.numel(), dtype=torch.float32))


def test_render_backward_allreduce_matches_plain():
    P, s_min, arrs = _setup()
    man, imgs, dL, z = G.raster("rectified")
    w, h = man["raster"]["res"]
    eng = P.Engine(0)
    eng.comm_init(0, 1)
    sc = P.ScannerConfig(detector_res_px=(w, h))
    up = torch.from_numpy(dL).cuda()
    c1, c2 = P.GaussianCloud(s_min, *arrs), P.GaussianCloud(s_min, *arrs)
    g1, g2 = P.CloudGrads(c1.size()), P.CloudGrads(c2.size())
    g1.buffer.fill_(0.5)
    g2.buffer.fill_(0.5)  # accumulate semantics: the reduced contribution is added
    f1 = eng.render(c1, sc, man["raster"]["thetas"])
    eng.render_backward(c1, f1, up, g1, accumulate_stats=True)
    f2 = eng.render(c2, sc, man["raster"]["thetas"])
    eng.render_backward_allreduce(c2, f2, up, g2, accumulate_stats=True)
    torch.cuda.synchronize()
    assert torch.equal(g1.buffer, g2.buffer)  # deterministic mode: bitwise
    assert torch.equal(c1.grad_count, c2.grad_count)
    assert torch.equal(c1.grad2d_norm_accum, c2.grad2d_norm_accum)
    assert torch.equal(c1.grad3d_accum, c2.grad3d_accum)
    f1.free()
    f2.free()


def test_voxelize_backward_allreduce_matches_plain():
    P, s_min, arrs = _setup()
    grid, vol, dL, z = G.voxel()
    eng = P.Engine(0)
    eng.comm_init(0, 1)
    c = P.GaussianCloud(s_min, *arrs)
    g1, g2 = P.CloudGrads(c.size()), P.CloudGrads(c.size())
    up = torch.from_numpy(dL).cuda()
    eng.voxelize_backward(c, grid, up, g1)
    eng.voxelize_backward_allreduce(c, grid, up, g2)
    torch.cuda.synchronize()
    assert torch.equal(g1.buffer, g2.buffer)
