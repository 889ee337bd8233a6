"""Runs tests/cpp/test_dropin (built against the unmodified reference headers
by tests/cpp/Makefile): the reference's own run_simulation driving
djg::GpuDjEngine through the Engine::assemble seam, and djg::run_simulation
with the state resident on the GPU, both against the reference DjEngine."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "test_dropin"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not BIN.exists(), reason="drop-in test binary not built (needs the reference headers)")
def test_reference_loop_drives_gpu_engine():
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
