"""compute-sanitizer over every kernel family.

tools/sanitize_workload.py drives each kernel once at a small shape; here it
runs under `compute-sanitizer` with memcheck (out-of-bounds / misaligned
global and shared accesses, leaks of device allocations), racecheck
(shared-memory hazards: the ADC windows' shared atomics, the encoder's
volatile weight reads, the assembly's staged batches, the Cholesky panel's
barriers) and synccheck (divergent / invalid barriers), once per variant
switch the parity tests pin. Every run must report zero errors."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for p in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if p and os.path.exists(p):
            return p
    raise AssertionError("compute-sanitizer not found")


CASES = [
    ("memcheck", "encode", {}),
    ("memcheck", "train", {"AQ_ASM_VARIANT": "1"}),
    ("memcheck", "train", {"AQ_ASM_VARIANT": "3"}),
    ("memcheck", "search", {"AQ_ADC_TC": "0"}),
    ("memcheck", "search", {"AQ_ADC_TC": "1"}),
    ("memcheck", "search", {"AQ_EXACT_TC": "0"}),
    ("racecheck", "encode", {}),
    ("racecheck", "train", {"AQ_ASM_VARIANT": "1"}),
    ("racecheck", "train", {"AQ_ASM_VARIANT": "3"}),
    ("racecheck", "search", {"AQ_ADC_TC": "0"}),
    ("racecheck", "search", {"AQ_ADC_TC": "1"}),
    ("synccheck", "encode", {}),
    ("synccheck", "train", {}),
    ("synccheck", "search", {"AQ_ADC_TC": "1"}),
]


@pytest.mark.parametrize("tool,part,env", CASES,
                         ids=[f"{t}-{p}-{'-'.join(f'{k}{v}' for k, v in e.items()) or 'default'}"
                              for t, p, e in CASES])
def test_sanitizer(tool, part, env):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "9"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py"), part]
    r = subprocess.run(cmd, cwd=ROOT, env={**os.environ, **env}, capture_output=True,
                       text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-6000:]
    assert "sanitize workload done" in out, out[-6000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-6000:]
    if tool == "racecheck":
        assert "RACECHECK SUMMARY: 0 hazards" in out or "hazard" not in out.lower(), out[-6000:]
