"""compute-sanitizer over the library's kernels: memcheck (out-of-bounds / misaligned
accesses), racecheck (shared-memory hazards), synccheck (barrier misuse), initcheck (reads of
uninitialised device memory)."""
import os
import shutil
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer(tool):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not found")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "7", "--print-limit", "20",
                        sys.executable, os.path.join(HERE, "sanitize_workload.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert "SANITIZE_WORKLOAD_OK" in out, out[-4000:]
    clean = "ERROR SUMMARY: 0 errors" in out or "(0 errors, 0 warnings)" in out
    assert r.returncode == 0 and clean, out[-4000:]
