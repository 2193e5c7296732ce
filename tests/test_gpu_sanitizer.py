"""compute-sanitizer over a few eager training steps on mag-mini:
memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory hazards:
the sampler's scans, the warp sorts, the tcgen05 staging) and synccheck (barrier
misuse). The kernels use decoupled look-back spin waits, PDL chains and a second
sampling stream; each tool must report zero errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer_clean(tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not found")
    cmd = [exe, "--tool", tool, "--error-exitcode", "3", "--target-processes", "all", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_step.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    out = r.stdout + r.stderr
    print(out[-3000:])
    if "ERROR SUMMARY" not in out and "closed on this pool" in out:
        pytest.skip("compute-sanitizer is disabled on this GPU pool: " + out.strip()[:200])
    assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
    assert r.returncode == 0, out[-3000:]
