"""anisoq_b200 command-line tool (reference proj/tools/anisoq_main.cpp), host
side: usage and exit codes (0 / 2 validation / 3 runtime), option and
--config parsing, and the gen verb against the reference generator (pinned
through the Python mirror). The GPU verbs are in tests/test_cli_gpu.py."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1908_10396_b200 import anisoq as aq
from paper_1908_10396_b200 import build

EXE = os.path.join(os.path.dirname(build.LIB), "anisoq_b200")


def run(*args, cwd=None):
    if not os.path.exists(EXE):
        build.build()
    return subprocess.run([EXE, *args], capture_output=True, text=True, cwd=cwd)


def test_usage_and_unknown_verbs():
    assert run().returncode == 2
    assert run("--help").returncode == 0
    r = run("frobnicate")
    assert r.returncode == 2 and "unknown subcommand" in r.stderr
    for verb in ("convert", "diagnose", "eta"):
        assert run(verb).returncode == 2


def test_option_errors(tmp_path):
    r = run("train", "--data", "x.fvecs")
    assert r.returncode == 2 and "--out is required" in r.stderr
    r = run("gen", "--out", str(tmp_path / "a.fvecs"), "--bogus", "1")
    assert r.returncode == 2 and "unknown option --bogus" in r.stderr
    r = run("gen", "--out", str(tmp_path / "a.fvecs"), "--n", "ten")
    assert r.returncode == 2 and "not an integer" in r.stderr
    r = run("gen", "--out", str(tmp_path / "a.fvecs"), "--kind", "cubes")
    assert r.returncode == 2 and "unknown kind" in r.stderr
    r = run("encode", "--data", str(tmp_path / "missing.fvecs"), "--codebook", "c", "--out", "o")
    assert r.returncode == 2  # MalformedFile is a validation error (error.hpp)


@pytest.mark.parametrize("kind,normalize", [("uniform_sphere", False),
                                            ("gaussian_mixture", True)])
def test_gen_matches_reference_generator(tmp_path, kind, normalize):
    out = tmp_path / "g.fvecs"
    args = ["gen", "--out", str(out), "--kind", kind, "--n", "300", "--d", "12", "--seed", "9",
            "--centers", "5", "--spread", "0.3"] + (["--normalize"] if normalize else [])
    r = run(*args)
    assert r.returncode == 0, r.stderr
    assert r.stdout == f"wrote 300 x 12 to {out}\n"
    want = aq.generate_synthetic(kind, 300, 12, 9, centers=5, spread=0.3, normalize=normalize)
    assert np.array_equal(aq.read_fvecs(str(out)).values, want.values)
    meta = json.loads((tmp_path / "g.fvecs.meta.json").read_text())
    assert meta["command"] == "gen" and meta["options"]["n"] == 300
    assert meta["options"]["spread"] == 0.3 and meta["outputs"] == [str(out)]
    assert len(meta["output_digest"]) == 16


def test_config_document(tmp_path):
    # section values, then top-level scalars; explicit flags win (anisoq_main.cpp:75-98)
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"seed": 4, "gen": {"n": 50, "d": 6, "kind": "gaussian_mixture",
                                                   "normalize": True}}))
    out = tmp_path / "g.fvecs"
    r = run("gen", "--out", str(out), "--config", str(cfg), "--d", "10")
    assert r.returncode == 0, r.stderr
    want = aq.generate_synthetic("gaussian_mixture", 50, 10, 4, normalize=True)
    assert np.array_equal(aq.read_fvecs(str(out)).values, want.values)
    bad = tmp_path / "bad.json"
    bad.write_text("{\"gen\": {\"n\": }")
    r = run("gen", "--out", str(out), "--config", str(bad))
    assert r.returncode == 2 and "config" in r.stderr
    cfg2 = tmp_path / "c2.json"
    cfg2.write_text(json.dumps({"gen": {"out": str(tmp_path / "h.fvecs"), "n": 7}}))
    r = run("gen", "--config", str(cfg2))  # a required option may come from the config
    assert r.returncode == 0 and (tmp_path / "h.fvecs").exists()
