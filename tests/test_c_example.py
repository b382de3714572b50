"""The C ABI from a C++ program (examples/moe_forward.cpp): AWQ tensors -> w4a16_repack_awq ->
w4a16_route_topk -> w4a16_moe_forward, checked inside the program against a plain CPU restatement
(exit 0 = routing identical and every output within rtol/atol 1e-2). It builds here (no GPU needed)
and runs on the GPU box."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _build():
    out = subprocess.run(["make", "-B", "-C", str(ROOT / "examples")], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    return ROOT / "examples" / "moe_forward"


def test_c_example_builds():
    assert _build().exists()


@pytest.mark.gpu
def test_c_example_runs():
    exe = _build()
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
