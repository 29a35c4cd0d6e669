"""The reference's own unit tests (proj/tests/test_pq.cpp, test_index.cpp,
test_vq.cpp), compiled UNMODIFIED against the C++ drop-in headers
(include/anisoq/) by tests/cpp/Makefile, run on the B200.

Every TEST_CASE of the three files runs; none is excluded (the out-of-scope
theory suites test_geometry.cpp / test_dataset.cpp's `diagnose` cases are not
part of this set). The binaries are built in this container from
/root/reference and travel to the GPU box; a missing binary is a failure,
not a skip.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_reftests")
SUITES = {"pq": 21, "index": 10, "vq": 17}  # TEST_CASE count per file


def _exe(suite):
    exe = os.path.join(BIN, f"test_{suite}")
    assert os.path.exists(exe), f"{exe} missing: run `make -C tests/cpp` (build())"
    return exe


@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suite_registered(suite):
    """CPU: the binary loads the drop-in library and registers every case of
    the reference file (listing runs no device code)."""
    r = subprocess.run([_exe(suite), "--list"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stderr
    names = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(names) == SUITES[suite], names
    if os.path.isdir("/root/reference/proj/tests"):
        src = open(f"/root/reference/proj/tests/test_{suite}.cpp").read()
        assert src.count("TEST_CASE(") == SUITES[suite]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", sorted(SUITES))
def test_reference_suite_passes_on_b200(suite):
    r = subprocess.run([_exe(suite)], capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out
    assert f"{SUITES[suite]} cases run, 0 skipped, 0 failed" in out, out


@pytest.mark.gpu
def test_reference_index_suite_on_multi_device_session():
    """The reference's test_index.cpp with $ANISOQ_DEVICES set: adc_search runs
    over row shards of a multi-device session (three shards on this box's one
    B200) and every case still passes — results depend only on the shard
    count and equal the single-device ones."""
    env = dict(os.environ, ANISOQ_DEVICES="0,0,0")
    r = subprocess.run([_exe("index")], capture_output=True, text=True, timeout=900, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out
    assert f"{SUITES['index']} cases run, 0 skipped, 0 failed" in out, out
