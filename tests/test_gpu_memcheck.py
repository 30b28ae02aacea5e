"""Poisoned-workspace + canary run of every kernel family (tests/memcheck_child.py) in a process of
its own with AUTOBYTE_DEBUG_MEM=1 — the stand-in for compute-sanitizer, which this GPU pool does
not allow."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a GPU")
def test_poisoned_workspaces_and_canaries():
    env = dict(os.environ, AUTOBYTE_DEBUG_MEM="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "memcheck_child.py")], capture_output=True,
                         text=True, timeout=600, cwd=ROOT, env=env)
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0 and "MEMCHECK_OK" in out.stdout
