"""Pin the CPU oracle against golden vectors produced by the reference (and the live reference)."""
import numpy as np
import pytest

import oracle
from oracle import core
from tests.golden.cases import MINI, RAGGED, STEP_CASES, STEP_METHODS, solver_kwargs, uses_momentum


class _Fro:
    @staticmethod
    def Frobenius():
        return "fro"


def oracle_config(method, b, **extra):
    kw = dict(solver_kwargs(method, _Fro))
    if "scaling" in kw:
        kw["scaling"] = "fro"
    if "method" in kw and kw["method"] == "cn" and uses_momentum(method):
        kw["beta1"] = 0.9
    return core.OracleConfig(block_size=b, **kw, **extra)


def test_structure_matches_golden(golden):
    for name, case in golden["structure"].items():
        st = core.build_structure([tuple(s) for s in case["shapes"]], case["block_size"])
        assert [[g["dim"], g["p"], len(g["members"])] for g in st["groups"]] == case["groups"], name
        assert [[list(r) for r in l["left"]] for l in st["layers"]] == case["left"], name
        assert [None if l["right"] is None else [list(r) for r in l["right"]] for l in st["layers"]] == case["right"]
        assert [None if l["spans"] is None else [list(map(list, s)) for s in l["spans"]] for l in st["layers"]] \
            == case["spans"], name
        if case["members"] is not None:
            assert [[list(m) for m in g["members"]] for g in st["groups"]] == case["members"]


def test_known_answers_partition():
    # (32000, 2048) at B=1024: 62 full blocks + 2 remainders of (256, 1024)
    full, rest = core.partition_layout((32000, 2048), 1024)
    assert len(full) == 62 and len(rest) == 2
    assert all((r1 - r0, c1 - c0) == (256, 1024) for (r0, r1), (c0, c1) in rest)
    # SURVEY §8(a1) remainder order for (37, 53) / 16
    _, rest = core.partition_layout((37, 53), 16)
    assert rest == (((0, 16), (48, 53)), ((16, 32), (48, 53)), ((32, 37), (0, 16)), ((32, 37), (16, 32)),
                    ((32, 37), (32, 48)), ((32, 37), (48, 53)))


def test_llama_group_sizes(golden):
    g953 = golden["structure"]["llama953m"]["groups"]
    assert g953 == [[256, 4, 4], [512, 4, 96], [1024, 2, 66], [1024, 4, 1820]]
    g124 = golden["structure"]["llama124m"]["groups"]
    assert g124 == [[128, 4, 1], [768, 2, 25], [768, 4, 218], [1024, 4, 121]]


def test_block_seed_and_start_vectors(golden):
    s = golden["seeds"]
    for (a, b), want in zip(s["pairs"].tolist(), s["seeds"].tolist()):
        assert core.block_seed(a, b) == want
    for key, v in s.items():
        if key.startswith("v"):
            np.testing.assert_array_equal(core.start_vectors(24, 5, int(key[1:])), v)


def test_ndb_matches_golden(golden):
    g = golden["solvers"]
    a = g["a"]
    for tag, (tol, mi) in (("tol", (1e-10, 100)), ("fix", (0.0, 10))):
        y, z, r1 = core.batched_newton_db(a, tol, mi)
        _, z4, r2 = core.batched_newton_db(y, tol, mi)
        np.testing.assert_array_equal(y, g[f"ndb_{tag}_y"])
        np.testing.assert_array_equal(z, g[f"ndb_{tag}_z"])
        np.testing.assert_array_equal(z4, g[f"ndb_{tag}_z4"])
        assert [r.iterations for r in r1 + r2] == g[f"ndb_{tag}_iters"].tolist()
        assert [r.converged for r in r1 + r2] == g[f"ndb_{tag}_conv"].tolist()


def test_ndb_known_answers():
    # NDB(I) = I in one iteration; NDB([[0.25]]) -> 0.5 / 2; NDB^4([[1/16]]) -> 2
    y, z, r = core.batched_newton_db(np.eye(3)[None])
    assert r[0].iterations == 1 and r[0].converged
    y, z, r = core.batched_newton_db(np.array([[[0.25]]]))
    assert abs(y[0, 0, 0] - 0.5) < 1e-12 and abs(z[0, 0, 0] - 2.0) < 1e-12 and r[0].iterations == 7
    y, _, _ = core.batched_newton_db(np.array([[[0.0625]]]))
    _, z, _ = core.batched_newton_db(y)
    assert abs(z[0, 0, 0] - 2.0) < 1e-10


def test_cn_matches_golden(golden):
    g = golden["solvers"]
    a = g["a"]
    for p in (2, 4):
        for tag, (tol, mi, e32) in (("tol", (1e-10, 100, False)), ("fix", (0.0, 12, False)), ("e32", (0.0, 12, True))):
            x, rep = core.batched_coupled_newton(a if not e32 else a[:2], p, tol, mi, emulate32=e32)
            np.testing.assert_allclose(x, g[f"cn{p}_{tag}_x"], rtol=0, atol=1e-12 * np.abs(x).max())
            assert [r.iterations for r in rep] == g[f"cn{p}_{tag}_iters"].tolist()


def test_chebyshev_matches_golden(golden):
    g = golden["solvers"]
    for p in (2, 4):
        c, _ = core.cheb_coefficients(p)
        np.testing.assert_allclose(c, g[f"cheb{p}_coeffs"], rtol=1e-13, atol=1e-15)
        out = core.batched_clenshaw(g["a"], c, g[f"cheb{p}_scales"], p)
        np.testing.assert_allclose(out, g[f"cheb{p}_out"], rtol=1e-10, atol=1e-10 * np.abs(out).max())


def test_power_iteration_matches_golden(golden):
    g = golden["solvers"]
    for i, s in enumerate(g["pi_seeds"].tolist()):
        lam = core.multi_power_iteration(g["a"][i], 16, 30, s)
        assert abs(lam - g["pi_lams"][i]) <= 1e-12 * abs(lam)
    np.testing.assert_allclose(core.random_spd(3, 10.0, 5, 0.5), g["rspd_3_10_5"], rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("case,shapes,b,nsteps", STEP_CASES)
@pytest.mark.parametrize("method", STEP_METHODS)
def test_full_step_matches_golden(golden, case, shapes, b, nsteps, method):
    g = golden["steps"]
    params = [g[f"{case}_param{i}"] for i in range(len(shapes))]
    cfg = oracle_config(method, b)
    st = core.init_state(params, cfg)
    cur = [p.copy() for p in params]
    for t in range(nsteps):
        cur, st, _ = core.step(st, cur, [g[f"{case}_grad{t}_{i}"] for i in range(len(shapes))], cfg, seed=3)
    for i, p in enumerate(cur):
        want = g[f"{case}_{method}_out{i}"]
        np.testing.assert_allclose(p, want, rtol=1e-9, atol=1e-12)
    for gi, grp in enumerate(st["groups"]):
        np.testing.assert_allclose(grp["roots"], g[f"{case}_{method}_root{gi}"], rtol=1e-8,
                                   atol=1e-9 * np.abs(grp["roots"]).max())


def test_oracle_vs_live_reference_step(reference):
    """Direct cross-check against the reference on a fresh seeded case (build container only)."""
    from blockshampoo import shampoo
    rng = np.random.default_rng(5)
    shapes = [(48, 32), (32,), (20, 48)]
    params = [rng.standard_normal(s) for s in shapes]
    grads = [rng.standard_normal(s) for s in shapes]
    rcfg = shampoo.ShampooConfig(block_size=16)
    rs = shampoo.init_state(params, rcfg)
    ref_out, _ = shampoo.step(rs, params, grads, rcfg, seed=9)
    ocfg = core.OracleConfig(block_size=16)
    os_ = core.init_state(params, ocfg)
    out, _, _ = core.step(os_, params, grads, ocfg, seed=9)
    for a, b in zip(out, ref_out):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-13)
