"""GPU tests of the drop-in boundary: default configurations, failure semantics, the reference names.

Each test states the reference behaviour it pins (file:line under /root/reference/pkg/src/blockshampoo).
"""
import numpy as np
import pytest
import torch

from oracle import core
from tests.golden.cases import STEP_CASES, solver_kwargs, uses_momentum

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU containers skip the whole module
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2602_02016_b200 import _lib, eigensolver, linalg, roots, shampoo, spectral  # noqa: E402
from paper_2602_02016_b200.errors import ConvergenceError, DegenerateSpectrumError, NumericalError  # noqa: E402
from paper_2602_02016_b200.linalg import PrecisionMode  # noqa: E402


def relf(x, y):
    x, y = np.asarray(x, dtype=np.float64), np.asarray(y, dtype=np.float64)
    d = np.linalg.norm(y)
    return np.linalg.norm(x - y) / (d if d > 0 else 1.0)


# ----------------------------------------------------------------------------- default configurations
def test_default_config_c1_first_step_runs_and_matches_oracle():
    """ShampooConfig() (NDB, tolerance 1e-10, FULL64) on config 1's literal first step (cond ~1e6 blocks)
    converges like the reference's float64 step: blocks at the fp32-class floor are converged there, blocks
    the iteration cannot converge are re-solved in float64 (shampoo.refresh_inverse_roots)."""
    rng = np.random.default_rng(0)
    w = rng.standard_normal((1024, 1024))
    g = rng.standard_normal((1024, 1024))
    cfg = shampoo.ShampooConfig()
    st = shampoo.init_state([w], cfg)
    out, st = shampoo.step(st, [w], [g], cfg, seed=0)
    ost = core.init_state([w], core.OracleConfig())
    oout, ost, _ = core.step(ost, [w], [g], core.OracleConfig(), seed=0)
    err = relf(out[0] - w, oout[0] - w)
    print(f"default-config C1 update relF {err:.2e}")
    # the literal first-step blocks have cond up to 4e7: their smallest eigenvalues lie below the resolution of
    # fp32-class statistics (ema relF ~5e-7), so the float64 roots are reproduced only up to that floor
    assert np.all(np.isfinite(out[0])) and err < 5e-2
    assert np.linalg.norm(out[0] - w) == pytest.approx(np.linalg.norm(oout[0] - w), rel=1e-4)


@pytest.mark.parametrize("case,shapes,b,nsteps", STEP_CASES)
@pytest.mark.parametrize("method,tol", [("ndb", (5e-3, 3e-4)), ("ndbfro", (5e-3, 3e-4)), ("cn", (5e-3, 1e-4)),
                                        ("evd", (1e-3, 1e-4))])
def test_default_tolerance_steps_vs_reference_golden(golden, case, shapes, b, nsteps, method, tol):
    """The reference's default-tolerance solver configs (tol 1e-10, FULL64) run to completion and land on the
    reference's float64 golden trajectory; EVD is the float64 device eigensolver + the same dampening.
    Tolerances (update relF): rank-deficient early statistics (mini, ragged: cond ~1e10 with eps = 1e-10 below
    fp32 resolution) 5e-3 (EVD 1e-3); full-rank warm statistics 3e-4 (CN, EVD 1e-4)."""
    tol = tol[case == "warm"]
    g = golden["steps"]
    params = [g[f"{case}_param{i}"] for i in range(len(shapes))]
    cfg = shampoo.ShampooConfig(block_size=b, solver=shampoo.SolverConfig(**solver_kwargs(method, spectral)),
                                graft=shampoo.GraftConfig(beta1=0.9 if uses_momentum(method) else 0.0))
    st = shampoo.init_state(params, cfg)
    cur = [p.copy() for p in params]
    for t in range(nsteps):
        cur, st = shampoo.step(st, cur, [g[f"{case}_grad{t}_{i}"] for i in range(len(shapes))], cfg, seed=3)
    worst = max(relf(p1 - p0, g[f"{case}_{method}_out{i}"] - p0) for i, (p0, p1) in enumerate(zip(params, cur)))
    print(f"{case}/{method}: update relF {worst:.2e}")
    assert worst < tol


# ----------------------------------------------------------------------------- failure semantics
def test_unbatched_ndb_raises_on_divergence():
    """roots.py:149-150: the unbatched iteration raises ConvergenceError when the divergence watch trips.
    A cond-1e4 block in EMULATED32 (no float64 floor rule) climbs back up after its minimum residual."""
    a = core.random_spd(256, 1e4, seed=3, scale=0.5)
    with pytest.raises(ConvergenceError, match="diverging"):
        roots.newton_db(a, roots.NdbConfig(tolerance=1e-12, max_iters=60), PrecisionMode.EMULATED32)


def test_unbatched_ndb_raises_on_non_finite():
    """roots.py:143-144: non-finite values raise NumericalError (spectrum far outside the convergence region)."""
    with pytest.raises(NumericalError):
        roots.newton_db(1e30 * np.eye(32), roots.NdbConfig(tolerance=1e-6, max_iters=20))


def test_batched_ndb_freezes_instead_of_raising():
    """roots.py:219-222: the batched solvers report a failing block and never abort its siblings."""
    a = np.stack([core.random_spd(256, 10.0, seed=1, scale=0.5), core.random_spd(256, 1e4, seed=3, scale=0.5)])
    _, z, rep = roots.batched_newton_db(a, roots.NdbConfig(tolerance=1e-12, max_iters=60), PrecisionMode.EMULATED32)
    assert not rep[1].converged and rep[1].iterations < 60
    assert rep[0].iterations > 1
    assert relf(z[0], core.batched_newton_db(a[:1], 0.0, 12)[1][0]) < 1e-4


def test_floor_rule_converges_full64_default_tolerance():
    """FULL64 with tol 1e-10 (below the fp32-class floor): well-conditioned blocks converge at the floor."""
    a = np.stack([core.random_spd(256, c, seed=i, scale=0.5) for i, c in enumerate([10.0, 1e2, 1e3])])
    y, z, rep = roots.batched_newton_db(a, roots.NdbConfig())
    assert all(r.converged for r in rep)
    assert all(r.residual <= linalg.STALL_CAP for r in rep)
    _, zo, ro = core.batched_newton_db(a, 1e-10, 100)
    for i in range(3):
        assert relf(z[i], zo[i]) < 3e-3


def test_refresh_does_not_commit_failed_group():
    """shampoo.py:330-343: a tolerance-mode failure raises before the group's roots are assigned."""
    rng = np.random.default_rng(5)
    shapes = [(48, 32)]
    params = [rng.standard_normal(s) for s in shapes]
    cfg_ok = shampoo.ShampooConfig(block_size=16, solver=shampoo.SolverConfig(method="cn", tolerance=0.0, max_iters=8))
    st = shampoo.init_state(params, cfg_ok)
    for _ in range(3):
        params, st = shampoo.step(st, params, [rng.standard_normal(s) for s in shapes], cfg_ok)
    before = [g.roots.clone() for g in st.groups]
    # EMULATED32 keeps the reference's rules: a float64 tolerance is unreachable -> ConvergenceError
    bad = shampoo.ShampooConfig(block_size=16, solver=shampoo.SolverConfig(
        method="cn", tolerance=1e-12, max_iters=6, precision=PrecisionMode.EMULATED32))
    with pytest.raises(ConvergenceError, match="inverse-root solver failed on"):
        shampoo.step(st, params, [rng.standard_normal(s) for s in shapes], bad)
    for b0, g in zip(before, st.groups):
        assert torch.equal(b0, g.roots)


def test_scale_check_kernel_codes():
    """The device scale checks: non-positive scale -> code 1 (ConvergenceError, shampoo.py:324-325), collapsed
    pool -> code 2 (DegenerateSpectrumError, spectral.py:106-107); the first failing group is recorded and gates
    every later group's commit."""
    L = _lib.lib()
    err = torch.zeros(2, dtype=torch.int32, device="cuda")
    ok = torch.zeros(3, dtype=torch.int32, device="cuda")
    good = torch.tensor([1.0, 2.0], device="cuda")
    zero = torch.tensor([1.0, 0.0], device="cuda")
    stat = torch.zeros(2, dtype=torch.int32, device="cuda")
    s = _lib.stream_ptr()
    L.dash_scale_check(good.data_ptr(), stat.data_ptr(), 2, 0, ok[0:1].data_ptr(), err.data_ptr(), s)
    L.dash_scale_check(zero.data_ptr(), stat.data_ptr(), 2, 1, ok[1:2].data_ptr(), err.data_ptr(), s)
    L.dash_scale_check(good.data_ptr(), stat.data_ptr(), 2, 2, ok[2:3].data_ptr(), err.data_ptr(), s)
    assert ok.tolist() == [1, 0, 0] and err.tolist() == [1, 1]
    err.zero_()
    stat[1] = 2
    L.dash_scale_check(good.data_ptr(), stat.data_ptr(), 2, 0, ok[0:1].data_ptr(), err.data_ptr(), s)
    assert err.tolist() == [2, 0] and int(ok[0]) == 0


def test_evd_degenerate_spectrum_raises():
    """eigensolver.py:168-169: SHIFTED_RELU removing every eigenvalue raises DegenerateSpectrumError."""
    h = eigensolver.DampeningHeuristic(eigensolver.HeuristicKind.SHIFTED_RELU)
    with pytest.raises(DegenerateSpectrumError):
        eigensolver.batched_evd_inverse_root(np.zeros((2, 8, 8)), 4, h)


def test_refresh_after_load_state_recomputes_statistics(tmp_path):
    """A refresh right after load_state (no accumulate) uses the loaded EMA's max|a| / Frobenius norm."""
    rng = np.random.default_rng(2)
    shapes = [(64, 32)]
    params = [rng.standard_normal(s) for s in shapes]
    cfg = shampoo.ShampooConfig(block_size=32, solver=shampoo.SolverConfig(
        method="ndb", scaling=spectral.Frobenius(), tolerance=0.0, max_iters=10))
    st = shampoo.init_state(params, cfg)
    for _ in range(3):
        params, st = shampoo.step(st, params, [rng.standard_normal(s) for s in shapes], cfg)
    shampoo.refresh_inverse_roots(st, cfg, seed=9)
    want = [g.roots.clone() for g in st.groups]
    path = tmp_path / "ck.txt"
    shampoo.save_state(st, cfg, path)
    st2, _ = shampoo.load_state(path)
    shampoo.refresh_inverse_roots(st2, cfg, seed=9)
    for a, b in zip(want, st2.groups):
        assert relf(b.roots.cpu().numpy(), a.cpu().numpy()) < 1e-5


# ----------------------------------------------------------------------------- reference names
def test_power_iteration_vs_golden(golden):
    """spectral.multi_power_iteration (spectral.py:87-112) with the golden seeds: lambda and the vector."""
    g = golden["solvers"]
    for i, seed in enumerate(g["pi_seeds"].tolist()):
        est = spectral.multi_power_iteration(g["a"][i], 16, 30, seed)
        assert est.lam == pytest.approx(g["pi_lams"][i], rel=2e-6)
        assert abs(float(np.dot(est.vector, g["pi_vecs"][i]))) == pytest.approx(1.0, abs=1e-5)
        assert spectral.rayleigh_quotient(g["a"][i], est.vector) == pytest.approx(g["pi_lams"][i], rel=2e-6)


def test_batched_power_iteration_vectors_and_zero_block():
    """batched_multi_power_iteration returns vectors; a zero block gives lambda 0 and its first start vector
    (spectral.py:99-101)."""
    a = np.stack([core.random_spd(96, 10.0, seed=0, scale=0.5), np.zeros((96, 96))])
    est = spectral.batched_multi_power_iteration(a, 16, 30, 11)
    lam0, v0 = core.multi_power_iteration(a[0], 16, 30, core.block_seed(11, 0), return_vector=True)
    assert est[0].lam == pytest.approx(lam0, rel=2e-6)
    assert abs(float(np.dot(est[0].vector, v0))) == pytest.approx(1.0, abs=1e-5)
    lam1, v1 = core.multi_power_iteration(a[1], 16, 30, core.block_seed(11, 1), return_vector=True)
    assert est[1].lam == 0.0 and lam1 == 0.0
    np.testing.assert_allclose(est[1].vector, v1, rtol=1e-6, atol=1e-7)


def test_linalg_names():
    """linalg.py:75-141: matmul / quantize / frobenius_norm / check_symmetric / identity_like / symmetrize."""
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((40, 30)), rng.standard_normal((30, 20))
    c = linalg.matmul(a, b)
    assert isinstance(c, np.ndarray) and relf(c, a @ b) < 1e-6
    with linalg.count_matmuls() as cnt:
        linalg.matmul(a, b)
        linalg.bmm(a[None], b[None])
    assert cnt.count == 2
    with pytest.raises(ValueError):
        linalg.matmul(a, a)
    assert linalg.quantize(np.array([0.1]), PrecisionMode.EMULATED32)[0] == np.float64(np.float32(0.1))
    assert linalg.quantize(np.array([0.1]), PrecisionMode.FULL64)[0] == 0.1
    assert linalg.frobenius_norm(a) == pytest.approx(np.linalg.norm(a))
    s = a[:30] @ a[:30].T
    linalg.check_symmetric(s)
    with pytest.raises(ValueError):
        linalg.check_symmetric(a[:30, :30])
    np.testing.assert_array_equal(linalg.identity_like(np.zeros((3, 4, 4))), np.broadcast_to(np.eye(4), (3, 4, 4)))
    np.testing.assert_allclose(linalg.symmetrize(a[:30, :30]), (a[:30, :30] + a[:30, :30].T) / 2)


def test_eigensolver_names():
    """eigensolver.eigh / evd_inverse_root (eigensolver.py:120-172) against float64 numpy."""
    a = core.random_spd(64, 1e3, seed=4, scale=2.0)
    dec = eigensolver.eigh(a)
    np.testing.assert_allclose(dec.eigenvalues, np.linalg.eigvalsh(a), rtol=1e-10, atol=1e-12)
    h = eigensolver.DampeningHeuristic(eigensolver.HeuristicKind.SHIFTED_RELU)
    r = eigensolver.evd_inverse_root(a, 4, h)
    assert relf(r, core.evd_inverse_root(a[None], 4)[0]) < 1e-10


@pytest.mark.parametrize("method", ["ndb", "cn", "cbshv"])
def test_pipelined_host_step_bitwise_equals_device_step(method):
    """Pinned host params / grads take the chunk-pipelined step (PCIe copies overlapped with the work); its
    results are bit-identical to the one-shot device-resident step (per-block work does not depend on the
    chunking)."""
    rng = np.random.default_rng(3)
    shapes = [(96, 64), (64,), (40, 72), (130, 33), (64, 64), (33,)]
    params = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    grads = [[rng.standard_normal(s).astype(np.float32) for s in shapes] for _ in range(3)]
    cfg = shampoo.ShampooConfig(block_size=32, solver=shampoo.SolverConfig(method=method, tolerance=0.0,
                                                                           max_iters=8))
    dev = [torch.as_tensor(p, device="cuda") for p in params]
    st_d = shampoo.init_state(dev, cfg)
    host = [torch.as_tensor(p).pin_memory() for p in params]
    st_h = shampoo.init_state(host, cfg)
    for gs in grads:
        dev, st_d = shampoo.step(st_d, dev, [torch.as_tensor(g, device="cuda") for g in gs], cfg, seed=2)
        host, st_h = shampoo.step(st_h, host, [torch.as_tensor(g).pin_memory() for g in gs], cfg, seed=2)
    assert st_h.runtime.chunks is not None and len(st_h.runtime.chunks) > 1  # the pipelined path ran
    for a, b in zip(dev, host):
        assert torch.equal(a.cpu(), b)
    for ga, gb in zip(st_d.groups, st_h.groups):
        assert torch.equal(ga.roots, gb.roots) and torch.equal(ga.ema, gb.ema)


def test_partition_device_bitexact_and_split_operand_bound():
    """blocking.partition (blocking.py:84-98) on a CUDA tensor == on NumPy, bit for bit; the step's in-place
    block operand (grad_split_kernel: hi + lo fp16 planes with a per-block power-of-two exponent) reproduces
    every gradient block to within 2^-21 of the block's max |g| per element (the a2 contract)."""
    from paper_2602_02016_b200.blocking import partition

    rng = np.random.default_rng(9)
    g = rng.standard_normal((300, 200)) * np.geomspace(1e-6, 1.0, 200)[None, :]
    pn = partition(g, 64)
    pt = partition(torch.as_tensor(g, device="cuda"), 64)
    assert np.array_equal(pt.full_blocks.cpu().numpy(), pn.full_blocks)
    for (s1, b1), (s2, b2) in zip(pt.blocks(), pn.blocks()):
        assert s1 == s2 and np.array_equal(b1.cpu().numpy(), b2)
    cfg = shampoo.ShampooConfig(block_size=64, solver=shampoo.SolverConfig(tolerance=0.0, max_iters=2))
    st = shampoo.init_state([g.astype(np.float32)], cfg)
    shampoo.accumulate(st, [g.astype(np.float32)], cfg)
    torch.cuda.synchronize()
    ops = st.runtime.gsm.to_float().double().cpu().numpy()
    g32 = g.astype(np.float32).astype(np.float64)
    for i, ((r0, r1), (c0, c1)) in enumerate(st.layers[0].layout.block_spans):
        blk = g32[r0:r1, c0:c1]
        err = np.abs(ops[i, : r1 - r0, : c1 - c0] - blk).max()
        assert err <= 2.0 ** -21 * np.abs(blk).max(), (i, err)
