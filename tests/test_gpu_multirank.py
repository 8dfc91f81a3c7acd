"""Multi-rank bench path on the GPU box (one rank per process under torchrun).  With one GPU the
ranks share device 0 and the 16-byte collective goes through gloo (the product path uses NCCL,
one GPU per rank); shards, all-gather, fixed-order finalize and max-over-ranks timing all run."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nproc,cfg", [(2, 3), (3, 4)])
def test_torchrun_bench_shards_match_oracle(nproc, cfg):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
           "--gpus", str(nproc), "--steps", "3", "--warmup", "3", "--config", str(cfg),
           "--dist-backend", "gloo", "--device-index", "0", "--no-cpu-baseline"]
    if nproc > 2:
        cmd.append("--no-configs")
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("{")][-1]
    d = json.loads(line)
    assert d["n_gpus"] == nproc and d["value"] > 0
    assert d["parity"]["rel_err_vs_oracle"] <= 1e-15
