"""Generate golden vectors by running the REFERENCE implementation (read-only import).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes small ``.npz`` / ``.json`` fixtures next to this file.  They pin the CPU oracle (``oracle/``)
and the GPU parity tests on machines where /root/reference does not exist (the GPU box).
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("DASH_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, str(Path(__file__).resolve().parent))

from blockshampoo import eigensolver, chebyshev, roots, shampoo, spectral, tasks  # noqa: E402
from blockshampoo.linalg import PrecisionMode  # noqa: E402

OUT = Path(__file__).resolve().parent

from cases import C1, MINI, RAGGED, STEP_CASES, STEP_METHODS, llama_124m, llama_953m, solver_kwargs, uses_momentum  # noqa: E402


def structure_fixture():
    cases = {"mini16": (MINI, 16), "ragged16": (RAGGED, 16), "ragged8": (RAGGED, 8), "c1": (C1, 256),
             "llama124m": (llama_124m(), 1024), "llama953m": (llama_953m(), 1024)}
    out = {}
    for name, (shapes, b) in cases.items():
        st = shampoo._build_structure([tuple(s) for s in shapes], b, False)
        out[name] = {
            "shapes": [list(s) for s in shapes],
            "block_size": b,
            "groups": [[g.dim, g.exponent, len(g.members)] for g in st.groups],
            "members": [[list(m) for m in g.members] for g in st.groups] if len(shapes) < 20 else None,
            "left": [[[r.group, r.slot] for r in l.left_refs] for l in st.layers],
            "right": [None if l.right_refs is None else [[r.group, r.slot] for r in l.right_refs]
                      for l in st.layers],
            "spans": [None if l.layout is None else [list(map(list, s)) for s in l.layout.block_spans]
                      for l in st.layers],
        }
    (OUT / "structure.json").write_text(json.dumps(out))


def seeds_fixture():
    pairs = [(0, 0), (0, 1), (1, 0), (12345, 7), (2**63 + 5, 3), (2**40, 2**33), (0x5EED, 0x5EED)]
    seeds = [spectral.block_seed(a, b) for a, b in pairs]
    vecs = {f"v{s}": spectral._start_vectors(24, 5, s) for s in [0, 1, seeds[3]]}
    np.savez(OUT / "seeds.npz", pairs=np.array(pairs, dtype=np.uint64), seeds=np.array(seeds, dtype=np.uint64),
             **vecs)


def solver_fixture():
    rng = np.random.default_rng(7)
    n = 48
    a = np.stack([tasks.random_spd(n, c, seed=i, scale=0.5) for i, c in enumerate([10.0, 1e3, 1e2, 3.0])])
    res = {"a": a}
    # NDB tolerance mode and fixed mode (p=2 chain and p=4 double chain)
    for tag, cfg in (("tol", roots.NdbConfig()), ("fix", roots.NdbConfig(tolerance=0.0, max_iters=10))):
        y, z, rep = roots.batched_newton_db(a, cfg)
        y2, z2, rep2 = roots.batched_newton_db(y, cfg)
        res[f"ndb_{tag}_y"], res[f"ndb_{tag}_z"], res[f"ndb_{tag}_z4"] = y, z, z2
        res[f"ndb_{tag}_iters"] = np.array([r.iterations for r in rep] + [r.iterations for r in rep2])
        res[f"ndb_{tag}_conv"] = np.array([r.converged for r in rep] + [r.converged for r in rep2])
        res[f"ndb_{tag}_resid"] = np.array([r.residual for r in rep] + [r.residual for r in rep2])
    for p in (2, 4):
        for tag, cfg, mode in (("tol", roots.CnConfig(p=p), PrecisionMode.FULL64),
                               ("fix", roots.CnConfig(p=p, tolerance=0.0, max_iters=12), PrecisionMode.FULL64),
                               ("e32", roots.CnConfig(p=p, tolerance=0.0, max_iters=12), PrecisionMode.EMULATED32)):
            x, rep = roots.batched_coupled_newton(a if mode is PrecisionMode.FULL64 else a[:2], cfg, mode)
            res[f"cn{p}_{tag}_x"] = x
            res[f"cn{p}_{tag}_iters"] = np.array([r.iterations for r in rep])
            res[f"cn{p}_{tag}_conv"] = np.array([r.converged for r in rep])
    for p in (2, 4):
        c = chebyshev.fit_inverse_root(p)
        res[f"cheb{p}_coeffs"] = c.coeffs
        sc = np.array([1.0, 0.8, 1.3, 0.6])
        res[f"cheb{p}_scales"] = sc
        res[f"cheb{p}_out"] = chebyshev.batched_clenshaw_matrix(a, c, sc)
    ests = [spectral.multi_power_iteration(a[i], 16, 30, 100 + i) for i in range(a.shape[0])]
    res["pi_lams"] = np.array([e.lam for e in ests])
    res["pi_vecs"] = np.stack([e.vector for e in ests])
    res["pi_seeds"] = np.array([100 + i for i in range(a.shape[0])])
    res["fro_scales"] = np.sqrt((a * a).sum(axis=(1, 2)))
    # cyclic Jacobi (eigensolver.py:77-124): SPD, indefinite, odd-sized and 1x1 blocks
    rng = np.random.default_rng(31)
    sym = rng.standard_normal((24, 24))
    jac = {"spd": tasks.random_spd(16, 1e3, seed=2, scale=0.5), "indef": 0.5 * (sym + sym.T),
           "odd": tasks.random_spd(7, 30.0, seed=3), "one": np.array([[2.5]]), "blk": a[1]}
    for name, m in jac.items():
        dec, sweeps = eigensolver.eigh_with_sweeps(m)
        res[f"jac_{name}_a"] = m
        res[f"jac_{name}_lam"] = dec.eigenvalues
        res[f"jac_{name}_vec"] = dec.eigenvectors
        res[f"jac_{name}_sweeps"] = np.array(sweeps)
    res["rspd_3_10_5"] = tasks.random_spd(3, 10.0, seed=5, scale=0.5)
    np.savez_compressed(OUT / "solvers.npz", **res)


def step_fixture():
    """Three optimizer steps on the mini / ragged layer sets for every solver."""
    res = {}
    for case, shapes, b, nsteps in STEP_CASES:
        rng = np.random.default_rng(11)
        params = [rng.standard_normal(s) for s in shapes]
        grads_seq = [[rng.standard_normal(s) for s in shapes] for _ in range(nsteps)]
        for i, p in enumerate(params):
            res[f"{case}_param{i}"] = p
        for t, gs in enumerate(grads_seq):
            for i, g in enumerate(gs):
                res[f"{case}_grad{t}_{i}"] = g
        for method in STEP_METHODS:
            solver = shampoo.SolverConfig(**solver_kwargs(method, spectral))
            cfg = shampoo.ShampooConfig(block_size=b, solver=solver,
                                        graft=shampoo.GraftConfig(beta1=0.9 if uses_momentum(method) else 0.0))
            state = shampoo.init_state(params, cfg)
            cur = [p.copy() for p in params]
            for t, gs in enumerate(grads_seq):
                cur, state = shampoo.step(state, cur, gs, cfg, seed=3)
            for i, p in enumerate(cur):
                res[f"{case}_{method}_out{i}"] = p
            for gi, g in enumerate(state.groups):
                res[f"{case}_{method}_root{gi}"] = g.roots
                res[f"{case}_{method}_ema{gi}"] = g.ema
    np.savez_compressed(OUT / "steps.npz", **res)


def checkpoint_fixture():
    """Reference text checkpoint after 3 steps (mini set, NDB fixed, momentum on) + the 4th step's outputs."""
    rng = np.random.default_rng(21)
    params = [rng.standard_normal(s) for s in MINI]
    grads_seq = [[rng.standard_normal(s) for s in MINI] for _ in range(4)]
    cfg = shampoo.ShampooConfig(block_size=16, solver=shampoo.SolverConfig(method="ndb", tolerance=0.0, max_iters=10),
                                graft=shampoo.GraftConfig(beta1=0.9))
    state = shampoo.init_state(params, cfg)
    cur = [p.copy() for p in params]
    for gs in grads_seq[:3]:
        cur, state = shampoo.step(state, cur, gs, cfg, seed=3)
    shampoo.save_state(state, cfg, OUT / "ckpt_mini.txt")
    res = {f"param3_{i}": p for i, p in enumerate(cur)}
    res.update({f"grad3_{i}": g for i, g in enumerate(grads_seq[3])})
    out, state = shampoo.step(state, cur, grads_seq[3], cfg, seed=3)
    res.update({f"out4_{i}": p for i, p in enumerate(out)})
    for gi, g in enumerate(state.groups):
        res[f"ema4_{gi}"] = g.ema
        res[f"root4_{gi}"] = g.roots
    np.savez_compressed(OUT / "checkpoint.npz", **res)


def training_fixture():
    """run_training rows of the reference on its three toy tasks (tasks.py:141-161)."""
    runs = {
        "quadratic_ndbfix": (tasks.QuadraticTask(seed=0), dict(method="ndb", tolerance=0.0, max_iters=10), 16, 1, 0.1),
        "logreg_ndbfix_f2": (tasks.LogisticRegressionTask(seed=1), dict(method="ndb", tolerance=0.0, max_iters=10), 8, 2, 0.5),
        "mlp_cnfix": (tasks.TinyMlpTask(seed=2), dict(method="cn", tolerance=0.0, max_iters=10), 8, 1, 0.05),
    }
    out = {}
    for name, (task, kw, bsz, freq, lr) in runs.items():
        cfg = shampoo.ShampooConfig(block_size=bsz, update_freq=freq, lr=shampoo.LrSchedule(base=lr),
                                    solver=shampoo.SolverConfig(**kw))
        rows, params = tasks.run_training(task, cfg, 12, seed=4)
        out[name] = {"block_size": bsz, "update_freq": freq, "lr": lr, "solver": kw,
                     "rows": [list(r) for r in rows]}
    (OUT / "training.json").write_text(json.dumps(out))


if __name__ == "__main__":
    training_fixture()
    checkpoint_fixture()
    structure_fixture()
    seeds_fixture()
    solver_fixture()
    step_fixture()
    print("golden fixtures written to", OUT)
