"""Shared fixtures.  `-m gpu` tests need a B200 (run through gpurun); the rest
run on CPU.  Oracle libraries (oracle/build, oracle/_ref) are test
infrastructure; they are (re)built here when missing and the sources exist."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_SRC = "/root/reference/proj/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def _ensure_oracle():
    restated = os.path.join(ROOT, "oracle", "build", "libfse_oracle.so")
    if not os.path.exists(restated):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "restated"], check=True)
    ref = os.path.join(ROOT, "oracle", "_ref", "libfse_ref.so")
    if not os.path.exists(ref) and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)


_ensure_oracle()


@pytest.fixture(scope="session")
def oracle():
    from oracle import restated
    return restated


@pytest.fixture(scope="session")
def ref():
    from oracle import refimpl
    if not refimpl.available():
        pytest.skip("oracle/_ref (the reference compiled from /root/reference) not available")
    return refimpl


@pytest.fixture(scope="session")
def fse():
    import paper_1607_04808_b200 as m
    return m


@pytest.fixture(scope="session")
def ctx(fse):
    return fse.Context(0)


@pytest.fixture
def rng():
    return np.random.default_rng(20261019)


def rel_max(a, b):
    a, b = np.asarray(a), np.asarray(b)
    scale = np.abs(b).max()
    return float(np.abs(a - b).max() / (scale if scale > 0 else 1.0))
