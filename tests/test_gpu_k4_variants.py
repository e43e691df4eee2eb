"""The alternative K4 statistics kernels (selected once per process by SCT_K4):
the tcgen05 + TMEM form ("tc") and the FP32 SIMT form ("simt"), each run through
__graft_entry__.smoke() in a fresh process (tile lists bit-exact, image and
gradients against the oracle), and the tc form through the golden fixtures."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(code, impl):
    env = dict(os.environ, SCT_K4=impl)
    return subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=600)


@pytest.mark.gpu
@pytest.mark.parametrize("impl", ["tc", "simt"])
def test_k4_variant_smoke(impl):
    r = _run("import __graft_entry__ as g; g.smoke()", impl)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "smoke ok" in r.stdout


@pytest.mark.gpu
def test_k4_tc_golden_and_fullsize():
    """The tc form against the golden fixtures and the cfg3 full-size atomic check."""
    env_tests = ["tests/test_gpu_golden.py", "tests/test_gpu_narrow.py"]
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", *env_tests], cwd=ROOT,
                       env=dict(os.environ, SCT_K4="tc"), capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
