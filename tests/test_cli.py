"""the reference's own command-line tool (proj/tools/main.cpp, compiled
unmodified by tools/cli/Makefile) linked against the B200 engine's ginimds:: facade, against
the same tool on the reference core (oracle/_ref/gini_mds_ref, test infrastructure): same
subcommands, flags, outputs and exit codes; byte-identical reruns except timings
(tests/cli/test_cli.cpp:138-164 in the reference); the 594 worked example in the manifest
(test_cli.cpp:111-120)."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = os.path.join(ROOT, "paper_2605_25124_b200", "lib", "gini_mds")
REF = os.path.join(ROOT, "oracle", "_ref", "gini_mds_ref")

pytestmark = pytest.mark.gpu


def run(binary, args, cwd):
    if not os.path.exists(binary):
        pytest.skip(f"{binary} not built")
    p = subprocess.run([binary] + args, cwd=cwd, capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout + p.stderr


def manifest(d):
    with open(os.path.join(d, "manifest.json")) as f:
        m = json.load(f)
    m.pop("timings")
    return m


@pytest.fixture()
def data(tmp_path):
    g = np.random.default_rng(5)
    X = g.standard_normal((80, 5)) * np.linspace(3.0, 0.5, 5)
    np.savetxt(tmp_path / "data.csv", X, delimiter=",", fmt="%.17g")
    return tmp_path


def test_embed_matches_reference_cli_and_reruns_identically(data):
    args = ["embed", "data.csv", "--metric", "gini", "--nu", "2", "--loss", "kruskal", "--max-iters", "200"]
    assert run(OURS, args + ["-o", "a"], data)[0] == 0
    assert run(OURS, args + ["-o", "b"], data)[0] == 0
    for f in ("coords.csv", "scatter.svg"):  # byte-identical reruns
        assert open(data / "a" / f, "rb").read() == open(data / "b" / f, "rb").read()
    assert manifest(data / "a") == manifest(data / "b")
    if not os.path.exists(REF):
        pytest.skip("reference CLI not built")
    assert run(REF, args + ["-o", "r"], data)[0] == 0
    ca = np.loadtxt(data / "a" / "coords.csv", delimiter=",", skiprows=1)
    cr = np.loadtxt(data / "r" / "coords.csv", delimiter=",", skiprows=1)
    assert np.max(np.abs(ca - cr)) <= 1e-6 * np.max(np.abs(cr))
    ma, mr = manifest(data / "a"), manifest(data / "r")
    assert ma["config"] == mr["config"] and ma["command"] == mr["command"] and ma["inputs"] == mr["inputs"]
    ra, rr = ma["results"], mr["results"]
    assert ra["iterations"] == rr["iterations"] and ra["converged"] == rr["converged"]
    assert abs(ra["stress"] - rr["stress"]) <= 1e-6 * rr["stress"]
    for k, v in rr["distance_stats"].items():
        assert abs(ra["distance_stats"][k] - v) <= 1e-12 * abs(v)


def test_tune_matches_reference_cli(data):
    args = ["tune", "data.csv", "--grid", "1.5:4:6", "--folds", "3", "--loss", "classical"]
    assert run(OURS, args + ["-o", "a"], data)[0] == 0
    if not os.path.exists(REF):
        pytest.skip("reference CLI not built")
    assert run(REF, args + ["-o", "r"], data)[0] == 0
    ta = json.load(open(data / "a" / "tune_report.json"))
    tr = json.load(open(data / "r" / "tune_report.json"))
    assert ta["nu_star"] == tr["nu_star"] and ta["folds"] == tr["folds"]
    for x, y in zip(ta["per_nu"], tr["per_nu"]):
        assert x["nu"] == y["nu"] and abs(x["mean_stress"] - y["mean_stress"]) <= 1e-9 * y["mean_stress"]
    ba, br = ta["best"], tr["best"]  # embedding_diagnostics: every field the CLI reports
    assert ba["method"] == br["method"] == "classical" and ba["clamped_count"] == br["clamped_count"]
    assert np.allclose(ba["eigenvalues"], br["eigenvalues"], rtol=1e-9)
    assert abs(ba["clamped_mass"] - br["clamped_mass"]) <= 1e-9


def test_594_worked_example_and_exit_codes(tmp_path):
    # D_G((10, 1200), (10, 12)) at nu = 3 is 594 (test_cli.cpp:111-120)
    (tmp_path / "two.csv").write_text("10,1200\n10,12\n")
    rc, _ = run(OURS, ["embed", "two.csv", "--metric", "gini", "--nu", "3", "--dims", "1", "-o", "o"], tmp_path)
    assert rc == 0
    assert manifest(tmp_path / "o")["results"]["distance_stats"]["max_offdiag"] == 594.0
    # exit codes (main.cpp:590-608): config error 2, data error 3
    assert run(OURS, ["embed", "two.csv", "--metric", "gini"], tmp_path)[0] == 2
    assert run(OURS, ["embed", "missing.csv"], tmp_path)[0] == 3
    assert run(OURS, ["embed", "two.csv", "--bogus"], tmp_path)[0] == 2
