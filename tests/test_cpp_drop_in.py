"""The C++ drop-in: a program written against the reference's fse:: API,
compiled against our headers and linked with libfse_b200.so, reproduces the
reference's recorded acceptance numbers on the GPU (criterion 2) and its
error behaviour.  Building is CPU-only; running needs the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "drop_in_main.cpp")
INC = os.path.join(ROOT, "paper_1607_04808_b200", "csrc", "cpp", "include")
LIBDIR = os.path.join(ROOT, "paper_1607_04808_b200")


def build(tmp_path):
    exe = str(tmp_path / "drop_in")
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O2", SRC, "-I", INC, "-I",
                    os.path.join(ROOT, "include"), "-L", LIBDIR, "-lfse_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_drop_in_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_drop_in_runs_reference_acceptance(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout


@pytest.mark.gpu
def test_drop_in_runs_on_the_multi_gpu_context(tmp_path):
    """The same program with FSE_CUDA_DEVICES set: fse::total_sum runs the
    partitioned evaluation (fse_cuda_multi_*, NCCL inside the library) over the
    listed GPUs -- here the one GPU of the pool -- and still reproduces the
    reference's recorded accuracies."""
    exe = build(tmp_path)
    env = dict(os.environ, FSE_CUDA_DEVICES="0")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout
