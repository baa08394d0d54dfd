"""fse-report-v1 reporting (harness.cpp:191-251) from the GPU
drop-in of the reference's harness API (csrc/cpp/fse_harness.cpp): a program
written against harness.hpp links with libfse_b200.so; its CSV keeps the
reference's columns in order with the GPU columns appended, its JSON keeps the
reference's record keys plus a "gpu" object, the oracle errors sit at the
method's level and the second run hits the FSEG cache (precompute 0)."""
import csv
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "harness_main.cpp")
INC = os.path.join(ROOT, "paper_1607_04808_b200", "csrc", "cpp", "include")
LIBDIR = os.path.join(ROOT, "paper_1607_04808_b200")
REF_COLS = ("kernel,N,L,xi,rc,M,P,Mtilde,tol,oracle,rel_rms_error,abs_rms_error,"
            "predicted_real_rms,predicted_fourier_rms,t_precompute,t_spread,t_fft,"
            "t_scale,t_quadrature,t_realspace,t_total,t_total_with_precompute").split(",")


def build(tmp_path):
    exe = str(tmp_path / "harness_main")
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O2", SRC, "-I", INC, "-I",
                    os.path.join(ROOT, "include"), "-L", LIBDIR, "-lfse_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_harness_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_harness_reports(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = open(tmp_path / "report.csv").read().splitlines()
    assert lines[0] == "# fse-report-v1"
    hdr = lines[1].split(",")
    assert hdr[: len(REF_COLS)] == REF_COLS
    assert hdr[len(REF_COLS):] == ["device", "n_gpus", "t_e2e", "targets_per_s"]
    rows = list(csv.DictReader(lines[1:]))
    assert len(rows) == 5
    assert float(rows[0]["t_precompute"]) > 0 and float(rows[1]["t_precompute"]) == 0
    for row in rows:
        assert row["oracle"] == "1" and 0 < float(row["rel_rms_error"]) < 1e-3
        assert "B200" in row["device"] and float(row["targets_per_s"]) > 0
    assert float(rows[2]["tol"]) == 1e-6 and float(rows[2]["rel_rms_error"]) < 1e-5
    j = json.load(open(tmp_path / "report.json"))
    assert j["schema"] == "fse-report-v1" and len(j["records"]) == 5
    rec = j["records"][0]
    for k in ("kernel", "N", "L", "xi", "rc", "M", "P", "Mtilde", "tol", "oracle",
              "rel_rms_error", "abs_rms_error", "predicted_real_rms", "predicted_fourier_rms"):
        assert k in rec
    assert set(rec["times"]) == {"precompute", "spread", "fft", "scale", "quadrature",
                                 "realspace", "total", "total_with_precompute"}
    assert rec["gpu"]["n_gpus"] == 1 and rec["gpu"]["t_e2e"] >= rec["times"]["total"]
