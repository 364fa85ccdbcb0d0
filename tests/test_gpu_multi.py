"""The NCCL exchange with world >= 2 (-m gpu; skipped when fewer than 2 GPUs are visible,
e.g. on the 1-GPU test box): tests/dist_worker.py under torchrun shards the batch over the
ranks and compares the sharded engine's best record (u*, t*, b*), the winner's bits
(broadcast from the owner), the step count and every member's count with a 1-GPU engine of
the same global batch, and the record with the fp64 oracle's run. The host side of the
protocol is covered on CPU by tests/test_dist_gloo.py."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count() if torch.cuda.is_available() else 0
    except Exception:
        return 0


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_nccl_equals_one_gpu_and_oracle(world, tmp_path):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "multi.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "dist_worker.py"),
           str(out)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    for res in json.load(open(out)):
        assert res["rc"][0] == res["rc"][1], res
        assert res["best"][0] == res["best"][1] == res["oracle_best"], res
        assert res["bits_equal"] and res["bits_reproduce"], res
        assert res["steps"][0] == res["steps"][1], res
        assert res["counts_equal"] in (True, None), res
