"""The `fde_b200` command line (csrc/cli.cpp): drop-in for the reference's
`fde solve` / `fde table` (proj/src/cli.cpp:84-211) with its CSV + manifest
report (proj/src/report.cpp:28-80).

CPU: flag validation and exit codes (usage errors exit 2 before touching the
device).  GPU: `solve` and `table` runs whose CSV cells equal the reference's
own time_march (oracle/_ref) at the CSV's printed precision.
"""
import csv
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracles import spec

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "paper_1706_06844_b200" / "fde_b200"


@pytest.fixture(scope="module")
def cli():
    if not BIN.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "paper_1706_06844_b200" / "csrc")], check=True)
    return BIN


def run(cli, *args, cwd=None):
    return subprocess.run([str(cli), *map(str, args)], capture_output=True, text=True, cwd=cwd,
                          timeout=600)


@pytest.mark.parametrize("args,msg", [
    (["solve", "--n", "16"], "solve needs --example or --coeff-preset"),
    (["solve", "--example", "4", "--n", "16"], "--example must be in [1, 3]"),
    (["solve", "--example", "1", "--n", "0"], "--n must be in [1, 4096]"),
    (["solve", "--example", "1", "--n", "5000"], "--n must be in [1, 4096]"),
    (["solve", "--example", "1", "--n", "16", "--precond", "ilu"], "unknown preconditioner"),
    (["solve", "--example", "1", "--n", "16", "--coarse", "direct"], "unknown coarse solve"),
    (["solve", "--example", "1", "--n", "16", "--tol", "-1"], "--tol must be positive"),
    (["solve", "--example", "1", "--n", "16", "--vcycles-per-apply", "17"], "must be in [1, 16]"),
    (["solve", "--example", "1", "--n", "x"], "not an integer"),
    (["solve", "--example", "1", "--n", "16", "--bogus"], "unknown option"),
    (["table"], "--table is required"),
    (["table", "--table", "1", "--sizes", "24"], "--sizes: 16, 32, 64 or 128"),
    (["frobnicate"], "unknown subcommand"),
])
def test_usage_errors_exit_2(cli, args, msg):
    r = run(cli, *args)
    assert r.returncode == 2, (r.returncode, r.stderr)
    assert msg in r.stderr


def test_help(cli):
    r = run(cli, "--help")
    assert r.returncode == 0 and "solve" in r.stdout and "table" in r.stdout
    assert run(cli).returncode == 2


def read_report(out_dir: Path, command: str):
    csvs = sorted(out_dir.glob(f"{command}-*.csv"))
    assert len(csvs) == 1, csvs
    rows = [r for r in csv.reader(open(csvs[0])) if r and not r[0].startswith("#")]
    man = json.loads(csvs[0].with_suffix(".manifest").read_text())
    return rows, man


@pytest.mark.gpu
@pytest.mark.parametrize("example,n,precond", [(1, 32, "mgm"), (2, 32, "mgm"), (3, 16, "p2"),
                                               (1, 16, "p2-exact"), (2, 16, "mgm-galerkin")])
def test_solve_matches_reference(cuda, ref, cli, tmp_path, example, n, precond):
    r = run(cli, "solve", "--example", example, "--n", n, "--precond", precond, "--out-dir", tmp_path)
    assert r.returncode == 0, r.stderr
    rows, man = read_report(tmp_path, "solve")
    assert rows[0] == ["example", "n", "precond", "avg_iters", "error_inf", "wall_time"]
    label, n_s, pc, avg, err, _ = rows[1]
    assert (label, n_s, pc) == (str(example), str(n), precond)
    # the reference CLI's defaults: tol 1e-7, restart 20, omega 0.9, m = n (cli.cpp:42-58)
    s = spec(100 + example, n1=n, n2=n, steps=n, tol=1e-7, omega=0.9,
             precond={"none": 0, "p2": 1, "mgm": 2, "p2-exact": 3, "mgm-galerkin": 4}[precond])
    ro = ref.time_march(s)
    assert avg == f"{np.mean(ro['its']):.3f}"
    e_ref = ref.error_inf(s, ro["u"], 1.0)
    # equal at the CSV's printed precision (report.cpp:66-70: %.5e)
    assert abs(float(err) - e_ref) <= 5e-6 * e_ref, (err, e_ref)
    assert man["command"] == "solve" and man["parameters"]["n"] == str(n)
    assert man["parameters"]["precond"] == precond and man["parameters"]["m"] == str(n)


@pytest.mark.gpu
def test_solve_baseline_config(cuda, cli, tmp_path):
    """--config K (extension): BASELINE configuration 1 through the CLI."""
    r = run(cli, "solve", "--config", "1", "--precond", "mgm", "--tol", "1e-8", "--omega", "0.7",
            "--m", "4", "--out-dir", tmp_path)
    assert r.returncode == 0, r.stderr
    rows, man = read_report(tmp_path, "solve")
    assert rows[1][0] == "config-1" and rows[1][1] == "63" and rows[1][4] == "nan"
    assert float(rows[1][3]) > 0


@pytest.mark.gpu
def test_table_matches_reference(cuda, ref, cli, tmp_path):
    r = run(cli, "table", "--table", "2", "--sizes", "16", "--out-dir", tmp_path)
    assert r.returncode == 0, r.stderr
    rows, man = read_report(tmp_path, "table")
    assert rows[0] == ["n", "none", "p2", "mgm", "error_inf"]
    assert rows[1][0] == "16"
    for col, pc in ((2, 1), (3, 2)):  # preconditioned columns: identical averages
        s = spec(102, n1=16, n2=16, steps=16, tol=1e-7, omega=0.9, precond=pc)
        assert rows[1][col] == f"{np.mean(ref.time_march(s)['its']):.3f}"
    assert man["parameters"]["table"] == "2" and man["parameters"]["sizes"] == "16"
