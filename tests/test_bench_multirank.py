"""The driver's multi-GPU launch of bench.py (torchrun, one rank per GPU, NCCL process group,
CUDA IPC halo mappings) exercised on the single B200: 2 ranks share cuda:0 (--same-device), so
the partitioned headline sweep and the partitioned C5 strong-scaling leg run end to end."""
import json
import os
import socket
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_bench_two_ranks_same_device():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--same-device", "--steps", "3", "--warmup", "3", "--orders", "1,3", "--e2e-steps", "2",
           "--box", "64", "--c5-n", "100", "--c5-orders", "2,3", "--no-cpu"]
    out = subprocess.run(cmd, cwd=HERE, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0
    assert [o["p"] for o in d["per_order"]] == [1, 3]
    assert "failed" not in d["c5"], d["c5"]
    assert d["c5"]["scaling"] == "strong" and d["c5"]["value"] > 0
    assert all(o["halo_rank0"] > 0 for o in d["c5"]["per_order"])
