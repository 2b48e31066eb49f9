"""The programmatic-launch protocol of the line passes (csrc/line_conv.cu, pass_enter: a row
pass runs ahead of its column pass and waits for it only in its first epilogue) must not change
a single bit: long chains of dependent applies and V-cycles with programmatic launches on
equal the same chains with every launch fully serialised (FDE_PDL=0).  A race between a row
pass and the kernels before it would show up here as a digest mismatch."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _digest(pdl):
    env = dict(os.environ, FDE_PDL=pdl)
    out = subprocess.run([sys.executable, str(ROOT / "tests" / "launch_protocol_worker.py")],
                         capture_output=True, text=True, env=env, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [l for l in out.stdout.splitlines() if l.startswith("DIGEST")]
    assert line, out.stdout[-2000:]
    return line[-1].split()[1]


@pytest.mark.gpu
def test_pdl_on_equals_serialised(cuda):
    a, b, c = _digest("1"), _digest("0"), _digest("1")
    assert a == b == c
