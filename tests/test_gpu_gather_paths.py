"""The quadrature's two staging paths give bit-identical velocities: the
TMA box per x-plane (k_gather_tma: even M~, every tensor-core tile shape) and the per-thread
cp.async staging (k_gather_mma), selected with FSE_GATHER_TMA in a fresh
process (the switch is read once per process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1607_04808_b200 as fse
ctx = fse.Context(0)
rng = np.random.default_rng(11)
L, xi, rc, M, P = {args!r}
cfg = fse.make_config(L, xi, rc, M, P)
pos = rng.uniform(0, L, (4000, 3))
tgt = rng.uniform(0, L, (3000, 3))
g = ctx.precompute_mollified_green(1, cfg.Ltilde, cfg.Mtilde, cfg.sf)
u = ctx.fourier_sum(fse.SourceSystem(pos, rng.standard_normal((4000, 3)), L), cfg, 0, tgt, g)
np.save({out!r}, u)
print(cfg.Mtilde)
"""


def _run(tmp_path, args, tma):
    out = str(tmp_path / f"u_{tma}.npy")
    env = dict(os.environ, FSE_GATHER_TMA=str(tma))
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, args=args, out=out)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out), int(r.stdout.split()[-1])


@pytest.mark.parametrize("args", [(1.0, 15.28, 0.25, 40, 24), (1.0, 20.0, 0.2, 62, 22),
                                  (1.0, 10.0, 0.25, 32, 16), (1.0, 8.0, 0.3, 31, 12),
                                  (1.0, 6.0, 0.3, 24, 8)])
def test_tma_and_cp_async_staging_agree(tmp_path, args):
    a, mt = _run(tmp_path, args, 1)
    b, _ = _run(tmp_path, args, 0)
    assert mt % 2 == 0  # the TMA path's precondition holds, so it ran
    assert np.array_equal(a, b)
