"""compute-sanitizer memcheck / racecheck / synccheck over the library's kernels (tools/
sanitize_case.py: cold + warm OptV2 of every kind, general path, two-level plan, row block,
k_compact, triplets, element loops).  Only the library's kernels (fa::) are checked."""

import shutil
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

REPO = Path(__file__).resolve().parents[1]
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not Path(SAN).exists(), reason="compute-sanitizer not installed")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_kernels_are_sanitizer_clean(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--kernel-name", "regex:fa::",
           sys.executable, str(REPO / "tools" / "sanitize_case.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=3000)
    text = out.stdout + out.stderr
    if "closed on this pool" in text:  # the gpurun pool's wrapper refuses compute-sanitizer
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + text.strip().splitlines()[0][:200])
    assert out.returncode == 0 and "sanitize case done" in out.stdout, text[-4000:]
    assert "ERROR SUMMARY: 0 errors" in text or "RACECHECK SUMMARY: 0 hazards" in text, text[-4000:]
