"""The kernels under device-side checks (the pool refuses compute-sanitizer): the checked build
libfemasm_b200_checked.so (FA_DCHECK: shared/global indices against their bounds, spin-wait
limits on the look-back and compaction waits, trap with the location) runs the sanitizer case
(every kernel family: cold and warm OptV2 of the four kinds, general path and overflowing
bucket, two-level plan with a row block, k_compact, triplets, element loops) and the small
bitwise parity tests."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

REPO = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def checked_lib():
    from paper_1305_3122_b200 import build

    return build.build_checked()


def _run(cmd, lib, timeout=1800):
    env = dict(os.environ, FEMASM_B200_LIB=str(lib))
    return subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=REPO, timeout=timeout)


def test_sanitizer_case_under_device_checks(checked_lib):
    out = _run([sys.executable, str(REPO / "tools" / "sanitize_case.py")], checked_lib)
    text = out.stdout + out.stderr
    assert out.returncode == 0 and "sanitize case done" in out.stdout, text[-4000:]
    assert "FA_CHECKED failure" not in text, text[-4000:]


def test_parity_suite_under_device_checks(checked_lib):
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-m", "gpu and not slow",
           str(REPO / "tests" / "test_gpu_parity.py"), str(REPO / "tests" / "test_gpu_api.py")]
    out = _run(cmd, checked_lib)
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-4000:]
    assert "FA_CHECKED failure" not in text, text[-4000:]
