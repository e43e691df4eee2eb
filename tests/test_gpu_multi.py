"""Multi-GPU path on real NCCL: skipped on boxes with fewer
than two GPUs (the development pool's boxes have one; the driver's 8-GPU node
runs them). (a) the torchrun worker tests/dist/nccl_worker.py — view-sharded
render_backward_allreduce and z-slab voxelize_backward_allreduce against one
rank doing the whole set; (b) bench.py under torchrun at N = 2 prints one
JSON line with n_gpus = 2."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _need(n):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")


def _torchrun(n, args, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), *args]
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)


@pytest.mark.parametrize("n", [2])
def test_nccl_sharded_backward_matches_one_rank(n):
    _need(n)
    r = _torchrun(n, [os.path.join(ROOT, "tests", "dist", "nccl_worker.py")], 29611)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "PASS" in r.stdout, r.stdout


def test_bench_torchrun_two_ranks():
    _need(2)
    r = _torchrun(2, ["bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e",
                      "--no-train", "--no-simt-arm"], 29612)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
