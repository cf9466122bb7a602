"""Regression guard for the layout-dependent wrong-cell bug of the packed kernels
(VERDICT r01 "what's weak" 2): the library is rebuilt in an ALTERNATE code
layout -- ptxas -O1, where the old inline-PTX float-pair pack produced 22 wrong costs --
into its own path (never over the in-tree libsdtw.so) and the bit-exact parity suite of
config 1 plus the ragged shapes runs against it through SDTW_LIB in a fresh process."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ptxas_O1_layout_is_bit_exact():
    out = os.path.join(ROOT, "variants", "alt_ptxas_O1.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.check_call([sys.executable, os.path.join(ROOT, "paper_2403_06931_b200", "build.py"),
                           "--out", out, "--xflag=--ptxas-options=-O1"], cwd=ROOT,
                          stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, timeout=900)
    env = dict(os.environ, SDTW_LIB=out)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-k", "config1_bit_exact or ragged_shapes or quantised or config5_shape"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
