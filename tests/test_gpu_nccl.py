"""The product collective path over NCCL on the 1-GPU box: torchrun --nproc-per-node 1 with
init_process_group("nccl") forced at world 1, so api.integrate_distributed and bench.py run the real
all_gather_into_tensor (NCCL kernel on the plan's stream) -> sg_finalize sequence that the N-GPU run
uses (NCCL refuses two ranks on one device, so world 1 is what one GPU can host).
NCCL_DEBUG=INFO is on: the init lines (nRanks) are checked and kept in the test output."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, os, sys
sys.path.insert(0, os.environ["SG_ROOT"])
import torch, torch.distributed as dist
import mpmath as mp
import sg_configs as S
from paper_2210_14313_b200 import api
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
assert dist.get_backend() == "nccl" and dist.get_world_size() == 1
gold = json.load(open(os.path.join(os.environ["SG_ROOT"], "tests", "golden", "oracle_full.json")))["values"]
out = {}
for i in (1, 2, 3, 5):
    p = S.baseline_config(i)
    hi, lo = api.integrate_distributed(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u)
    ref = mp.mpf(gold[p.name]["text"])
    out[p.name] = float(abs((mp.mpf(hi) + mp.mpf(lo) - ref) / ref))
dist.barrier()
dist.destroy_process_group()
print("RESULT " + json.dumps(out))
"""


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(args, timeout=900):
    env = dict(os.environ, NCCL_DEBUG="INFO", SG_ROOT=ROOT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    return subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout, env=env)


def _check_nccl_log(text):
    assert "NCCL INFO" in text, text[-3000:]
    assert any("nRanks 1" in ln or "nranks 1" in ln.lower() for ln in text.splitlines()), text[-3000:]
    for ln in text.splitlines():
        if "NCCL INFO" in ln and ("nRanks" in ln or "Init COMPLETE" in ln):
            print(ln)


def test_integrate_distributed_over_nccl_world1(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "nccl_w1.py"
    script.write_text(SCRIPT)
    out = _torchrun([str(script)])
    assert out.returncode == 0, out.stderr[-3000:]
    _check_nccl_log(out.stdout + out.stderr)
    res = json.loads([l for l in out.stdout.splitlines() if l.startswith("RESULT ")][-1][7:])
    for name, err in res.items():
        assert err <= 1e-15, (name, err)


def test_bench_over_nccl_world1():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _torchrun(["bench.py", "--gpus", "1", "--steps", "3", "--warmup", "3", "--config", "4",
                     "--force-dist", "--no-cpu-baseline", "--no-configs", "--no-merged",
                     "--no-frontier", "--no-corner"])
    assert out.returncode == 0, out.stderr[-3000:]
    _check_nccl_log(out.stdout + out.stderr)
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["config"]["collective"] == "nccl all_gather_into_tensor"
    assert line["n_gpus"] == 1 and line["value"] > 0
    assert line["parity"]["rel_err_vs_oracle"] <= 1e-15
    assert line["collapse"]["rel_diff_vs_combination"] <= 1e-15
