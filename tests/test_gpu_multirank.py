"""Real multi-process NCCL slabs: 2 ranks on 2 GPUs via torchrun
(tools/multirank_check.py), the gathered snapshot, stable_dt and the folded
totals bitwise equal to the undecomposed run.  Needs >= 2 GPUs: the round's
GPU box has one, so this is skipped there and runs on any multi-GPU node; the
same phase sequence is covered on one GPU by the slab groups
(test_gpu_slabs.py), which share the orchestration, the split kernels, the
halo overlap and the per-slab error words with this path."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.skipif(_ngpus() < 2, reason="needs >= 2 GPUs (one process per GPU)")
@pytest.mark.parametrize("case", ["tgv3d", "tgv2d", "h2o2"])
def test_two_rank_nccl_slabs_bitwise(case):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tools", "multirank_check.py"), "--case", case]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["snapshot_bitwise"] and d["stable_dt_equal"] and d["totals_bitwise"], d
