"""Standalone CUDA checks of the device templates (tests/cuda/*.cu), built
with nvcc for sm_100a and run on the GPU: the warp-specialised tcgen05 GRU
stage against an fp64 host reference (gws_gru_test.cu)."""
import os
import shutil
import subprocess
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _nvcc():
    n = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(n):
        pytest.skip("nvcc not available")
    return n


@pytest.mark.parametrize("batch", [37, 300])
def test_gws_gru_standalone(batch):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = tempfile.mkdtemp()
    exe = os.path.join(d, "gws_gru_test")
    subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-DFAST_DIV", "-o", exe,
                    os.path.join(ROOT, "tests", "cuda", "gws_gru_test.cu"), "-lcuda"], check=True, capture_output=True)
    r = subprocess.run([exe, str(batch)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr
