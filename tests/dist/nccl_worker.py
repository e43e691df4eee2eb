"""torchrun worker for tests/test_gpu_multi.py: N ranks (one GPU each) shard the
golden views strided, run render_backward_allreduce (context-owned NCCL
communicator through the C-ABI) and the z-slab voxelize_backward_allreduce;
rank 0 compares the reduced gradients with a one-rank render / voxelize of the
whole set and prints PASS."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2405_20693_b200 as P  # noqa: E402
from paper_2405_20693_b200 import dist as pdist  # noqa: E402
from tests import _golden as G  # noqa: E402


def rel(a, b):
    a, b = a.double().cpu(), b.double().cpu()
    return float((a - b).norm() / max(float(b.norm()), 1e-30))


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    eng = P.Engine(local)
    eng.comm_init(rank, world)
    assert eng.comm_info() == (world, rank)
    s_min, *arrs = G.cloud_arrays()
    man, imgs, dL, z = G.raster("rectified")
    w, h = man["raster"]["res"]
    thetas = man["raster"]["thetas"]
    sc = P.ScannerConfig(detector_res_px=(w, h))
    views = pdist.shard_views(len(thetas), rank, world)
    cloud = P.GaussianCloud(s_min, *arrs)
    g = P.CloudGrads(cloud.size())
    f = eng.render(cloud, sc, [thetas[v] for v in views])
    eng.render_backward_allreduce(cloud, f, torch.from_numpy(dL[views]).cuda(), g, accumulate_stats=True)
    f.free()
    # voxelizer: z-slab of brick layers per rank
    grid, vol, vdl, _ = G.voxel()
    layers = (grid.dims[2] + 7) // 8
    zb = pdist.shard_z_bricks(layers, rank, world)
    gv = P.CloudGrads(cloud.size())
    eng.voxelize_backward_allreduce(cloud, grid, torch.from_numpy(vdl).cuda(), gv, z_bricks=zb)
    torch.cuda.synchronize()
    if rank == 0:
        ref_cloud = P.GaussianCloud(s_min, *arrs)
        rg = P.CloudGrads(ref_cloud.size())
        rf = eng.render(ref_cloud, sc, thetas)
        eng.render_backward(ref_cloud, rf, torch.from_numpy(dL).cuda(), rg, accumulate_stats=True)
        rf.free()
        rv = P.CloudGrads(ref_cloud.size())
        eng.voxelize_backward(ref_cloud, grid, torch.from_numpy(vdl).cuda(), rv)
        torch.cuda.synchronize()
        errs = {"raster_grads": rel(g.buffer, rg.buffer), "voxel_grads": rel(gv.buffer, rv.buffer),
                "grad2d_norm": rel(cloud.grad2d_norm_accum, ref_cloud.grad2d_norm_accum)}
        cnt_ok = torch.equal(cloud.grad_count, ref_cloud.grad_count)
        print("errors", errs, "grad_count exact", cnt_ok, flush=True)
        ok = cnt_ok and all(v < 1e-5 for v in errs.values())
        print("PASS" if ok else "FAIL", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
