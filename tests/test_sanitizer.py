"""compute-sanitizer over small end-to-end runs (memcheck,
racecheck, synccheck, initcheck): every kernel of the fused pipeline (FP32 /
FP64 weighting, aidw / idw, grid / brute engines), the raster path and a
crowded-cell grid build must report zero errors and zero hazards."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    p = subprocess.run([SAN, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    assert "sanitize run ok" in p.stdout
