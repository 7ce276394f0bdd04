"""bench.py's multi-rank plumbing on CPU: torchrun with 2 ranks (gloo, the
--dry-run rehearsal: same cell / direction sharding, barrier + max-over-ranks
timing, rank-0 JSON line; the oracle on a few nodes stands in for the GPU)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("workload,scaling", [("c5", "strong"), ("c5", "weak"), ("c3", "strong")])
def test_torchrun_two_ranks_dry_run(workload, scaling):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "3", "--dry-run", "--workload", workload,
           "--scaling", scaling]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_ranks"] == 2
    if workload == "c5":
        spans = d["rank_spans"]
        if scaling == "strong":
            assert d["global_cells"] == 512 and spans == [[0, 256], [256, 256]]
        else:
            assert d["global_cells"] == 1024 and spans == [[0, 512], [512, 512]]
