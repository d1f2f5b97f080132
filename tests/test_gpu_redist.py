"""Device redistribution (slapcu_distribute_triples / slapcu_redistribute over
NCCL) parity: tests/redist_worker.py under torchrun on 1, 2 and 4 GPUs."""
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
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + nproc),
           os.path.join(ROOT, "tests", "redist_worker.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "REDIST_OK" in r.stdout, r.stdout[-2000:]


@pytest.mark.skipif(NGPU < 1, reason="needs a GPU")
def test_redistribute_p1():
    run(1)


@pytest.mark.skipif(NGPU < 2, reason="needs 2 GPUs")
def test_redistribute_p2():
    run(2)


@pytest.mark.skipif(NGPU < 4, reason="needs 4 GPUs")
def test_redistribute_p4():
    run(4)
