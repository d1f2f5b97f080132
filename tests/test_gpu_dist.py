"""Multi-GPU parity of the NCCL SUMMA / 3D drivers (needs >= 2 GPUs; each
case launches tests/dist_worker.py under torchrun, one process per GPU)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(nproc, *args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + nproc), os.path.join(ROOT, "tests",
                                                                                       "dist_worker.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "DIST_OK" in r.stdout, r.stdout[-2000:]


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
def test_ca3d_p2_c2():
    run(2, "--case", "ca3d", "--layers", "2")


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("concat", [0, 1])
def test_summa_p4(concat):
    run(4, "--case", "summa", "--concat", str(concat))


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
def test_ca3d_p4_c4():
    run(4, "--case", "ca3d", "--layers", "4")


@pytest.mark.skipif(NGPU < 8, reason="needs 8 GPUs")
def test_ca3d_p8_c2():
    run(8, "--case", "ca3d", "--layers", "2")


@pytest.mark.skipif(NGPU < 1, reason="needs a GPU")
def test_mcl_dist_p1():
    run(1, "--case", "mcl", "--layers", "1")


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
def test_mcl_dist_p2_3d():
    run(2, "--case", "mcl", "--layers", "2")


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
def test_mcl_dist_p4_2d_and_3d():
    run(4, "--case", "mcl", "--layers", "4")
