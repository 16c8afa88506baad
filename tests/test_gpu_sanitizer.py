"""compute-sanitizer over every kernel (race detection):
memcheck, racecheck (shared-memory hazards), initcheck, synccheck on tiny
inputs (tests/tools/sanitize_run.py, oracle-checked)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "initcheck", "synccheck"])
def test_compute_sanitizer(tool):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, SAN_COUNT="40", PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    extra = []
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "99", "--target-processes", "all", *extra,
                        sys.executable, os.path.join(ROOT, "tests", "tools", "sanitize_run.py")],
                       capture_output=True, text=True, timeout=900, env=env)
    tail = (r.stdout + r.stderr)[-3000:]
    if "compute-sanitizer is closed" in tail:
        # the GPU pool's operators disabled the tool (its wrapper refuses to run);
        # the committed logs under profiles/sanitizer/ are the last runs
        pytest.skip("compute-sanitizer closed on this GPU pool: " + tail.strip().splitlines()[0][:200])
    assert r.returncode == 0, tail
    assert "sanitize_run ok" in r.stdout, tail
    out = r.stdout + r.stderr
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out, tail
