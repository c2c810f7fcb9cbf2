"""GEMM engine variants selected by environment knobs (read once per process, so each runs in a subprocess):
K-block 32 (64-byte swizzle, DASH_KB=32), the accumulator layouts (DASH_NACC = 1 / 2 / 4) and 256-wide pair
tiles for split launches (DASH_NT=2562) must all give fp32-class products and Newton-DB results within the
parity bounds of test_gpu_parity.py.  fp16-mode solves run with 256-wide tiles by default and with 128-wide
tiles under DASH_NT=128; both stay within the fp16 bound."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import numpy as np, torch
from paper_2602_02016_b200 import linalg, roots
from paper_2602_02016_b200.linalg import PrecisionMode
from oracle import core
torch.manual_seed(0)
for m, n, k, tb in ((256, 256, 256, False), (300, 700, 130, True), (1024, 1024, 1024, False)):
    a = torch.randn(2, m, k, device="cuda"); b = torch.randn(2, n if tb else k, k if tb else n, device="cuda")
    c = linalg.bmm(a, b, PrecisionMode.EMULATED32, trans_b=tb)
    bd = b.double().transpose(1, 2) if tb else b.double()
    ref = a.double() @ bd
    err = float((c.double() - ref).norm() / ref.norm())
    assert err < 1e-5, (m, n, k, tb, err)
for b in (200, 384):  # 384: two row tiles, a ragged last column tile in both tilings
    a = np.stack([core.random_spd(b, c, seed=i, scale=0.5) for i, c in enumerate([10.0, 1e3])])
    y, z, rep = roots.batched_newton_db(a, roots.NdbConfig(tolerance=0.0, max_iters=10))
    yo, zo, ro = core.batched_newton_db(a, 0.0, 10)
    for i in range(2):
        err = np.linalg.norm(y[i] - yo[i]) / np.linalg.norm(yo[i])
        print("ndb", b, i, err)
        assert err < 5e-5, (b, i, err)
print("ok")
"""

F16_CN_CHEB_SCRIPT = r"""
import numpy as np
from paper_2602_02016_b200 import chebyshev, roots
from paper_2602_02016_b200.linalg import PrecisionMode
from oracle import core
c = chebyshev.fit_inverse_root(4)
for b in (384, 1024):  # CN: two split outputs (M, correction) per job; Clenshaw: TMA-staged side input B_{k+2}
    a = np.stack([core.random_spd(b, cnd, seed=20 + i, scale=0.5) for i, cnd in enumerate([10.0, 1e2])])
    x, rep = roots.batched_coupled_newton(a, roots.CnConfig(p=4, tolerance=0.0, max_iters=12), PrecisionMode.F16)
    xo, ro = core.batched_coupled_newton(a, 4, 0.0, 12)
    sc = 2.0 * np.linalg.eigvalsh(a)[:, -1]
    y = chebyshev.batched_clenshaw_matrix(a, c, sc, PrecisionMode.F16)
    yo = core.batched_clenshaw(a, c.coeffs, sc, 4)
    for i in range(2):
        ex = np.linalg.norm(x[i] - xo[i]) / np.linalg.norm(xo[i])
        ey = np.linalg.norm(y[i] - yo[i]) / np.linalg.norm(yo[i])
        print("cn/cheb-f16", b, i, ex, ey)
        assert ex < 1e-2 and ey < 2e-2, (b, i, ex, ey)
print("ok")
"""

F16_SCRIPT = r"""
import numpy as np
from paper_2602_02016_b200 import roots
from paper_2602_02016_b200.linalg import PrecisionMode
from oracle import core
for b in (384, 1024):
    a = np.stack([core.random_spd(b, c, seed=i, scale=0.5) for i, c in enumerate([10.0, 1e2])])
    y, z, rep = roots.batched_newton_db(a, roots.NdbConfig(tolerance=0.0, max_iters=10), PrecisionMode.F16)
    yo, zo, ro = core.batched_newton_db(a, 0.0, 10)
    for i in range(2):
        ey = np.linalg.norm(y[i] - yo[i]) / np.linalg.norm(yo[i])
        ez = np.linalg.norm(z[i] - zo[i]) / np.linalg.norm(zo[i])
        print("ndb-f16", b, i, ey, ez)
        assert ey < F16_BOUND and ez < F16_BOUND, (b, i, ey, ez)
print("ok")
"""


def _run(script, env):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", script], cwd=root, env={**os.environ, **env, "PYTHONPATH": root},
                       capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("env", [{"DASH_KB": "32"}, {"DASH_NACC": "1"}, {"DASH_NACC": "4"}, {"DASH_NT": "2562"}])
def test_engine_variant(env):
    _run(SCRIPT, env)


@pytest.mark.parametrize("env", [{}, {"DASH_NT": "128"}])
def test_f16_cn_chebyshev_tilings(env):
    """Coupled Newton (p = 4) and Clenshaw in fp16 mode under both tilings vs float64."""
    _run(F16_CN_CHEB_SCRIPT, env)


@pytest.mark.parametrize("env", [{}, {"DASH_NT": "128"}])
def test_f16_solver_tilings(env):
    """fp16 products (one tensor pass, 11-bit operands): Newton-DB at B = 384 / 1024 within 1e-2 of float64."""
    _run(F16_SCRIPT.replace("F16_BOUND", "1e-2"), env)
