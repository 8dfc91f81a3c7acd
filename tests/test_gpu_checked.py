"""The checked build (-DSG_CHECKS): bounds checks of every frontier read/write and of the leaf-row
table slices, every partial slot written exactly once per step (the atomic task counters hand out
each task exactly once), bitwise-equal reruns, parity with the oracle — on the small cases and
configs 1-4 whole and sharded (tools/checked_run.py --quick).  compute-sanitizer is closed on this
GPU pool; this is the race / out-of-bounds evidence instead (profiles/r02_checked_run.txt)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_quick():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "checked_run.py"), "--quick"],
                         cwd=ROOT, capture_output=True, text=True, timeout=1500)
    assert out.returncode == 0, (out.stdout[-3000:], out.stderr[-3000:])
    assert "CHECKED_RUN_OK" in out.stdout
