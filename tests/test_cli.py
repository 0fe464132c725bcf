"""spardl_cli surface (tests/CMakeLists.txt:22-41 of the reference, SPEC
"MODULE cli"): rejection messages on CPU, the GPU subcommands on a B200."""
import csv
import io
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args):
    env = dict(os.environ, PYTHONPATH=ROOT)
    return subprocess.run([sys.executable, "-m", "paper_2304_00737_b200.cli", *args],
                          capture_output=True, text=True, env=env, cwd=ROOT, timeout=600)


def test_cli_rejects_nondivisible_k():
    r = _cli("allreduce", "--P", "6", "--k", "601", "--N", "6000")
    assert r.returncode != 0 and "k must be divisible by P" in r.stdout + r.stderr


def test_cli_rejects_bad_rsag():
    r = _cli("allreduce", "--P", "8", "--k", "800", "--N", "8000", "--d", "3", "--sag", "rsag")
    assert r.returncode != 0 and "rsag requires power-of-two d" in r.stdout + r.stderr


def test_csv_writers_match_reference_formats():
    from paper_2304_00737_b200 import cli, api
    buf = io.StringIO()
    cli.write_run_report_header(buf)
    cli.write_run_report_row(buf, api.ClusterConfig(6, 6000, 600), {
        "max_rounds": 6, "max_scalars": 2000, "pred_rounds": 6, "pred_low": 2000,
        "pred_high": 2000, "consistent": 1, "conservation_error": 0.0})
    assert buf.getvalue() == ("P,N,k,d,sag,residual,timing,seed,max_rounds,max_scalars,"
                              "predicted_rounds,predicted_scalars_low,predicted_scalars_high,"
                              "consistent,conservation_error\n"
                              "6,6000,600,1,none,gres,optimized,0,6,2000,6,2000,2000,1,0\n")
    buf = io.StringIO()
    cli.write_ledger_csv(buf, [2, 2], [300, 300])
    assert buf.getvalue() == "worker_id,rounds,scalars_received\n0,2,300\n1,2,300\n"
    buf = io.StringIO()
    cli.write_controller_trace_header(buf)
    cli.write_controller_trace_row(buf, 0, {"h": 100.0, "step": 2.0, "flag": True,
                                            "target": 200}, 199)
    assert buf.getvalue() == "iteration,h,step,flag,N_t,L\n0,100,2,1,199,200\n"


@pytest.mark.gpu
def test_cli_allreduce_gpu(built):
    r = _cli("allreduce", "--P", "6", "--k", "600", "--N", "6000", "--d", "1", "--seed", "7")
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert rows[0]["max_rounds"] == rows[0]["predicted_rounds"] == "6"
    assert rows[0]["max_scalars"] == "2000" and rows[0]["consistent"] == "1"
    assert float(rows[0]["conservation_error"]) <= 1e-6


@pytest.mark.gpu
def test_cli_verify_complexity_gpu(built):
    r = _cli("verify-complexity", "--P-set", "2,3,4,5,6,8", "--d-set", "1,2", "--k-mult", "100")
    assert r.returncode == 0, r.stdout + r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert rows and all(x["pass"] == "pass" for x in rows)
    assert {x["sag"] for x in rows} >= {"none", "rsag", "bsag", "topka"}


@pytest.mark.gpu
def test_cli_bsag_trace_gpu(built):
    import numpy as np
    r = _cli("bsag-trace", "--P", "6", "--k", "600", "--d", "3", "--iterations", "40")
    assert r.returncode == 0, r.stdout + r.stderr
    rows = list(csv.DictReader(io.StringIO(r.stdout)))
    assert len(rows) == 40 and float(rows[0]["h"]) == 100.0        # h0 = k/P
    assert all(100.0 <= float(x["h"]) <= 300.0 for x in rows)      # [k/P, dk/P]
    L = int(rows[0]["L"])
    dev = [abs(int(x["N_t"]) - L) / L for x in rows[20:]]
    assert float(np.median(dev)) <= 0.2
