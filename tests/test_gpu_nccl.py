"""Row (e) on NCCL: the count all-reduce hook under torchrun, eager and captured
inside the step graphs (StepGraphs and Engine.run), one rank per GPU.

world = 1 runs on any GPU box (a one-rank NCCL communicator still exercises
the capture of the collective); world = 2 needs two GPUs and is skipped
otherwise.  NCCL_DEBUG=INFO is set so the communicator's rank count is in the
log (checked below)."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2])
def test_nccl_count_allreduce_in_graphs(world):
    if not torch.cuda.is_available() or torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    env = dict(os.environ, NCCL_DEBUG="INFO", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "tools" / "check_nccl_graph.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600, cwd=str(ROOT))
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-3000:]
    assert "OK graph==eager True" in text, text[-3000:]
    assert f"nranks {world}" in text or f"nRanks {world}" in text, "no NCCL communicator line in the log"
