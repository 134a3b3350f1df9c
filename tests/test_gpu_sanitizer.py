"""compute-sanitizer over one small fwd+bwd (sanitizers) at N = 1024, d in
{64, 128}: memcheck (out-of-bounds / misaligned global and shared accesses) and synccheck (illegal
barrier use) over every kernel of the tcgen05 path; racecheck (shared-memory hazards between the
threads of a CTA) over the path whose shared memory is ordered by block barriers -- the
classification and aggregation kernels and the shape-generic SIMT kernels.

racecheck is not gated on the tcgen05 attention kernels: their shared-memory reuse is ordered
by mbarrier chains that run through tcgen05.commit (compute warps store P / dS, arrive; the MMA
warp waits, issues, commits; the epilogue waits on the commit barrier and reuses the buffer).
racecheck does not model the commit as a release, so it reports every such reuse as a WAW /
WAR hazard; memcheck and synccheck over the same kernels are clean."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer not found")
@pytest.mark.parametrize("tool,path", [("memcheck", "fast"), ("synccheck", "fast"), ("racecheck", "generic")])
@pytest.mark.parametrize("d", [64, 128])
def test_sanitizer_clean(tool, path, d):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "hazard"]
    cmd += [sys.executable, os.path.join(HERE, "tools", "sanitize_step.py"), str(d), path]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    log = out.stdout[-4000:] + out.stderr[-4000:]
    if out.returncode != 0 and "closed on this pool" in log:
        # the GPU pool's compute-sanitizer wrapper refuses every run (it has left GPUs needing a
        # reset); the bounds / determinism / reference-parity suites stand in for it there
        pytest.skip("compute-sanitizer is closed on this GPU pool")
    assert out.returncode == 0, log
    assert "sanitize step ok" in out.stdout
    text = out.stdout + out.stderr
    assert "ERROR SUMMARY: 0 errors" in text or "(0 errors, 0 warnings)" in text, log
