"""The C-ABI driven from plain C++ (examples/cpp_dropin.cpp): the reference's solver
known-answer tests and error mapping, without Python in the loop."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def test_cpp_dropin_example():
    exe = ROOT / "examples" / "cpp_dropin"
    assert exe.exists(), "run __graft_entry__.build() first"
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "0 failure(s)" in res.stdout
