"""compute-sanitizer suites (SURVEY.md §4 layer 9, §5; the paper's concern with "deadlock risks",
PAPER.md:164): memcheck (out-of-bounds / misaligned device accesses, leaks of device errors),
racecheck (shared-memory hazards: the staged programs, privatised accumulators, the TMA event ring
and the hash key cache), synccheck (illegal barriers / warp-sync masks in the divergent paths)
over every config on both engines (tests/sanitize_target.py), each run checked against the oracle."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _sanitizer():
    p = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(p):
        pytest.skip("compute-sanitizer not installed")
    return p


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(gpu, tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "97", "--print-limit", "20",
           "--target-processes", "all", sys.executable, os.path.join(HERE, "sanitize_target.py"), tool]
    if tool == "memcheck":
        cmd[1:1] = ["--leak-check", "no"]
    env = dict(os.environ, PYTORCH_NO_CUDA_MEMORY_CACHING="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, env=env)
    tail = (r.stdout[-4000:] + "\n" + r.stderr[-4000:])
    if "compute-sanitizer is closed" in tail:     # the GPU pool's wrapper refuses the tool
        pytest.skip("compute-sanitizer is disabled on this GPU pool (tests/test_gpu_bounds.py covers the bounds side)")
    assert r.returncode == 0, f"{tool}: rc={r.returncode}\n{tail}"
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr, tail
    assert r.stdout.count(" ok") >= 18, tail
