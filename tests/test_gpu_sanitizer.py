"""compute-sanitizer over every kernel family (tools/sanitize_workload.py):
memcheck (out-of-bounds / misaligned accesses), racecheck (shared-memory
hazards: the cp.async-staged metadata pass, block counters), synccheck
(barrier use), initcheck (reads of uninitialised device memory).  The dual
dataflow and the peer find are also run under memcheck.

Run on a B200: HKV_SANITIZER=1 python -m pytest tests -m gpu.  Opt-in: the
GPU pool this project is measured on has closed compute-sanitizer (runs
under it left GPUs needing a reset), so by default the test is skipped and
the round-2 logs under profiles/r02/sanitizer/ stand as the evidence."""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.parametrize("tool,parts", [
    ("memcheck", "single,dual,cas,host,single_key,peer,export"),
    ("racecheck", "single,cas,export"),
    ("synccheck", "single,dual,cas,export"),
    ("initcheck", "single,single_key,export"),
])
def test_compute_sanitizer_clean(tool, parts):
    if os.environ.get("HKV_SANITIZER") != "1":
        pytest.skip("compute-sanitizer is opt-in (HKV_SANITIZER=1): closed on the measurement pool")
    if not os.path.exists(SAN):
        pytest.fail("compute-sanitizer not found")
    log = os.path.join(ROOT, "gpurun_out", f"sanitizer_{tool}.txt")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    cmd = [SAN, "--tool", tool, "--error-exitcode", "9", "--print-limit", "200", sys.executable,
           os.path.join(ROOT, "tools", "sanitize_workload.py"), parts]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    out = r.stdout + r.stderr
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)" in out
    assert "sanitize workload ok" in r.stdout
