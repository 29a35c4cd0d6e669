"""Compiles tests/cpp/test_dropin.cpp against the C++ drop-in headers
(include/anisoq/) + libanisoq_b200.so and runs it on the GPU."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1908_10396_b200")


def _build(out):
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"), "-o", out,
           "-L", PKG, "-lanisoq_b200", f"-Wl,-rpath,{PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_dropin_compiles(tmp_path):
    """CPU: the drop-in headers compile and link (no device calls)."""
    _build(str(tmp_path / "dropin"))


@pytest.mark.gpu
def test_dropin_runs_on_gpu(tmp_path):
    exe = str(tmp_path / "dropin")
    _build(exe)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_dropin_host_parts_match_reference(tmp_path):
    """CPU: generate_synthetic / fvecs / ivecs / Rng / to_vq from the drop-in
    headers; the generated data equals the reference's generator bit for bit."""
    exe = str(tmp_path / "dropin_host")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "test_dropin_host.cpp"), "-o", exe,
           "-L", PKG, "-lanisoq_b200", f"-Wl,-rpath,{PKG}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    from oracle import Reference
    from paper_1908_10396_b200 import anisoq as aq
    assert Reference.available(), "oracle/_ref/libanisoq_ref.so missing (make -C oracle)"
    R = Reference()
    mix = aq.read_fvecs(str(tmp_path / "mix.fvecs")).values
    sph = aq.read_fvecs(str(tmp_path / "sphere.fvecs")).values
    assert np.array_equal(mix, R.generate_synthetic(1, 200, 8, 7, centers=6, spread=0.25,
                                                    normalize=True))
    assert np.array_equal(sph, R.generate_synthetic(0, 50, 5, 3))
