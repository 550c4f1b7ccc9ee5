"""primkit-driver, the CLI front end (reference proj/tools/driver.cpp; cases
follow proj/tests/test_driver.cpp): exit codes, report formats, determinism
under the fake clock, perf-db tuning and the fusion comparison.

Usage errors need no GPU (`not gpu`); everything that runs a solver is
`gpu`."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "paper_1910_00078_b200", "bin", "primkit-driver")


@pytest.fixture(scope="module")
def driver():
    if not os.path.exists(DRIVER):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_1910_00078_b200", "csrc")])
    return DRIVER


def run(driver, args, cwd, fake_clock=True):
    env = dict(os.environ)
    if fake_clock:
        env["PRIMKIT_FAKE_CLOCK"] = "1"
    env["PRIMKIT_CACHE_DIR"] = str(cwd / "cache")
    r = subprocess.run([driver] + args.split(), cwd=cwd, env=env, capture_output=True, text=True,
                       timeout=600)
    return r.returncode, r.stdout, r.stderr


def test_missing_required_flag_exits_2(driver, tmp_path):
    rc, _, err = run(driver, "conv -n 1 -H 16 -W 16 -k 8", tmp_path)
    assert rc == 2 and "-c" in err


def test_bad_direction_exits_2(driver, tmp_path):
    rc, _, err = run(driver, "conv -n 1 -c 4 -H 8 -W 8 -k 4 -F 3", tmp_path)
    assert rc == 2 and "-F" in err


def test_usage_errors(driver, tmp_path):
    assert run(driver, "", tmp_path)[0] == 2
    assert run(driver, "bogus -c 1", tmp_path)[0] == 2
    assert run(driver, "conv -c 4 -H 8 -W 8 -k 4 --frobnicate", tmp_path)[0] == 2
    assert run(driver, "fusion -c 4 -H 8 -W 8 --combo XYZ", tmp_path)[0] == 2
    assert run(driver, "fusion -c 4 -H 8 -W 8 -k 4 --act swish", tmp_path)[0] == 2
    assert run(driver, "fusion -c 4 -H 8 -W 8 --combo CBA", tmp_path)[0] == 2  # no -k
    rc, out, _ = run(driver, "--help", tmp_path)
    assert rc == 0 and "conv" in out


def _lines(p):
    return p.read_text().splitlines()


@pytest.mark.gpu
def test_conv_report_sorted(driver, tmp_path):
    rc, out, _ = run(driver, "conv -n 1 -c 8 -H 16 -W 16 -k 8 -y 3 -x 3 -p 1 -q 1 -u 1 -v 1 "
                             "-o conv.csv", tmp_path)
    assert rc == 0 and out == "conv.csv\n"
    lines = _lines(tmp_path / "conv.csv")
    assert len(lines) >= 5
    assert lines[0] == "# primkit-report v1"
    assert lines[1] == "label,solver,median_ms,workspace_bytes,speedup_vs_im2colgemm"
    prev = 0.0
    for ln in lines[2:]:
        assert ln.startswith("3-3-8-16-16-8-1-1,")
        t = float(ln.split(",")[2])
        assert t >= prev
        prev = t
    assert any(",Im2colGemm," in ln for ln in lines[2:])


@pytest.mark.gpu
def test_reports_deterministic_under_fake_clock(driver, tmp_path):
    args = "conv -n 1 -c 8 -H 16 -W 16 -k 8 -y 3 -x 3 -p 1 -q 1"
    assert run(driver, args + " -o d1.csv", tmp_path)[0] == 0
    assert run(driver, args + " -o d2.csv", tmp_path)[0] == 0
    assert (tmp_path / "d1.csv").read_bytes() == (tmp_path / "d2.csv").read_bytes()


@pytest.mark.gpu
def test_json_report(driver, tmp_path):
    rc, _, _ = run(driver, "conv -n 1 -c 4 -H 8 -W 8 -k 4 -y 3 -x 3 -p 1 -q 1 --json -o c.json",
                   tmp_path)
    assert rc == 0
    body = (tmp_path / "c.json").read_text()
    assert '"schema": "primkit-report v1"' in body and '"solver": "Direct"' in body
    import json
    doc = json.loads(body)
    assert all(set(r) == {"label", "solver", "median_ms", "workspace_bytes",
                          "speedup_vs_im2colgemm"} for r in doc["rows"])


@pytest.mark.gpu
def test_bf16_backward_weights_report(driver, tmp_path):
    rc, _, err = run(driver, "conv -n 2 -c 64 -H 14 -W 14 -k 64 -y 3 -x 3 -p 1 -q 1 -F 4 --bf16 "
                             "-o bw.csv", tmp_path, fake_clock=False)
    assert rc == 0, err
    solvers = [ln.split(",")[1] for ln in _lines(tmp_path / "bw.csv")[2:]]
    assert set(solvers) == {"Im2colGemm", "Direct"}


@pytest.mark.gpu
def test_tune_writes_and_reuses_db(driver, tmp_path):
    args = "tune -n 1 -c 4 -H 6 -W 6 -k 4 -y 3 -x 3 -p 1 -q 1 --db tune.db"
    assert run(driver, args, tmp_path)[0] == 0
    first = (tmp_path / "tune.db").read_text()
    assert "ImplicitGemm:" in first and "1-4-6-6-4-3-3-1-1-1-1-1-1-1-F-C-f32=" in first
    assert run(driver, args, tmp_path)[0] == 0
    assert (tmp_path / "tune.db").read_text() == first


@pytest.mark.gpu
def test_tune_without_tunable_solver(driver, tmp_path):
    rc, _, err = run(driver, "tune -n 1 -c 4 -H 8 -W 8 -k 4 -y 3 -x 3 -l 2 -j 2 --db none.db",
                     tmp_path)
    assert rc == 1 and "no tunable solver" in err
    assert not (tmp_path / "none.db").exists()


@pytest.mark.gpu
def test_fusion_round_trips(driver, tmp_path):
    rc, _, _ = run(driver, "fusion -n 1 -c 4 -H 8 -W 8 -k 4 -y 1 -x 1 --combo CBA -o cba.csv",
                   tmp_path)
    assert rc == 0
    lines = _lines(tmp_path / "cba.csv")
    assert len(lines) == 4
    assert "CBA/fused," in lines[2] and ",1," in lines[2]
    assert "CBA/unfused," in lines[3] and ",3," in lines[3]


@pytest.mark.gpu
def test_rejected_fusion_cites_constraint(driver, tmp_path):
    rc, _, err = run(driver, "fusion -n 1 -c 17 -H 24 -W 24 -k 4 -y 3 -x 3 --combo CBA "
                             "--algo Winograd", tmp_path)
    assert rc == 1 and "c >= 18" in err


@pytest.mark.gpu
def test_na_and_cbna_fusions(driver, tmp_path):
    rc, _, _ = run(driver, "fusion -n 1 -c 4 -H 8 -W 8 --combo NA --act sigmoid -o na.csv", tmp_path)
    assert rc == 0 and "NA/fused," in _lines(tmp_path / "na.csv")[2]
    rc, _, _ = run(driver, "fusion -n 1 -c 3 -H 9 -W 9 -k 4 -y 3 -x 3 -p 1 -q 1 --combo CBNA "
                           "--act tanh -o cbna.csv", tmp_path)
    assert rc == 0
    lines = _lines(tmp_path / "cbna.csv")
    assert ",1," in lines[2] and ",4," in lines[3]
