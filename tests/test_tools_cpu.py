"""Every measurement tool under tools/ parses its arguments without a GPU
(`--help` exits 0 before any CUDA work), so a broken tool shows up in the
CPU suite rather than in a GPU call."""
import glob
import os
import subprocess
import sys

import pytest

from conftest import ROOT

TOOLS = sorted(glob.glob(os.path.join(ROOT, "tools", "*.py")))


@pytest.mark.parametrize("tool", TOOLS, ids=[os.path.basename(t) for t in TOOLS])
def test_tool_help(tool):
    r = subprocess.run([sys.executable, tool, "--help"], capture_output=True, text=True,
                       timeout=120, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "usage" in r.stdout.lower()
