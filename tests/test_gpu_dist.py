"""Multi-GPU parity of the distributed path (needs >= 2 GPUs; one spawned process per GPU), for both
transports: P2P (CUDA IPC peer memory over NVLink, the default) and NCCL send/recv."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
@pytest.mark.parametrize("world", [2, 4])
def test_dist_parity(world, transport):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world), os.path.join(ROOT, "tests", "dist_worker.py")]
    env = dict(os.environ, ARROW_TEST_TRANSPORT=transport, ARROW_DIST_TRACE="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and out.count("DIST_OK") == world, out[-4000:]
    if transport == "p2p":  # the P2P transport must actually be in use (no silent NCCL fallback)
        assert out.count("transport p2p") >= world, out[-2000:]
