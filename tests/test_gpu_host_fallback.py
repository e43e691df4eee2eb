"""The host-buffer entry points without stream memory operations
(SCT_HOST_UNITS=0: one composite then one copy; the backward's upstream
gradient in event-chained view chunks) give the same results as the device
path: the host-entry parity tests re-run in a subprocess with the switch set
(it is read once per process)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_host_entry_points_without_stream_memops():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    env = dict(os.environ, SCT_HOST_UNITS="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-k", "host_entry",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
