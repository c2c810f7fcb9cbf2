"""Float64 NumPy restatement of the reference DASH step — ORACLE, test infrastructure only.

Each function cites the reference lines it restates (paths under /root/reference/pkg/src/blockshampoo).
Written independently of the reference sources: same arithmetic and control flow, different code.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


# ============================================================================ configuration
@dataclass(frozen=True)
class OracleConfig:
    """Flattened ShampooConfig + SolverConfig + GraftConfig + LrSchedule (shampoo.py:53-130)."""

    beta_lr: float = 0.95
    epsilon: float = 1e-10
    update_freq: int = 1
    block_size: int = 256
    method: str = "ndb"             # evd | cn | ndb | cbshv
    scaling: str = "pi"             # pi | fro
    pool: int = 16
    pi_iters: int = 30
    tolerance: float = 1e-10
    max_iters: int = 100
    emulate32: bool = False         # PrecisionMode.EMULATED32 for CN / Chebyshev
    cheb_degree: int = 60
    cheb_points: int = 1000
    cheb_interval: tuple[float, float] | None = None
    beta1: float = 0.0
    beta2: float = 0.999
    graft_eps: float = 1e-8
    lr_kind: str = "constant"
    lr_base: float = 1e-3
    lr_total: int = 0
    lr_final: float = 0.0
    heuristic: str = "relu"          # EVD dampening: legacy | relu | abs (eigensolver.py:31-44)
    heuristic_eps: float = 1e-10

    def lr(self, t: int) -> float:
        """LrSchedule.value (shampoo.py:103-109)."""
        if self.lr_kind == "constant":
            return self.lr_base
        frac = min(t / self.lr_total, 1.0)
        if self.lr_kind == "linear":
            return self.lr_base + (self.lr_final - self.lr_base) * frac
        return self.lr_final + (self.lr_base - self.lr_final) * 0.5 * (1.0 + math.cos(math.pi * frac))


@dataclass
class IterationReport:
    iterations: int
    residual: float
    converged: bool


# ============================================================================ block structure
def partition_layout(shape, b):
    """Full B x B spans row-major, then ragged cells row-major (blocking.py:62-81)."""
    m, n = shape
    if b < 1:
        raise ValueError("block size must be >= 1")
    nm, nn = m // b, n // b
    full, rest = [], []
    for i in range(-(-m // b)):
        for j in range(-(-n // b)):
            span = ((i * b, min(i * b + b, m)), (j * b, min(j * b + b, n)))
            (full if (i < nm and j < nn) else rest).append(span)
    return tuple(full), tuple(rest)


def chunk_bounds(length, b):
    """1-D chunks [s, min(s+B, len)) (shampoo.py:171-173)."""
    return tuple((s, min(s + b, length)) for s in range(0, length, b))


def build_structure(shapes, b, momentum=False):
    """Groups keyed (dim, exponent), members sorted (layer, L<R, idx) (shampoo.py:176-230)."""
    members: dict[tuple[int, int], list[tuple[int, int, int]]] = {}
    layers = []
    for lid, shape in enumerate(shapes):
        if len(shape) == 2:
            full, rest = partition_layout(shape, b)
            spans = full + rest
            for idx, ((r0, r1), (c0, c1)) in enumerate(spans):
                members.setdefault((r1 - r0, 4), []).append((lid, 0, idx))
                members.setdefault((c1 - c0, 4), []).append((lid, 1, idx))
            layers.append({"shape": tuple(shape), "spans": spans, "n_full": len(full), "chunks": None})
        elif len(shape) == 1:
            ch = chunk_bounds(shape[0], b)
            for idx, (s, e) in enumerate(ch):
                members.setdefault((e - s, 2), []).append((lid, 0, idx))
            layers.append({"shape": tuple(shape), "spans": None, "n_full": 0, "chunks": ch})
        else:
            raise ValueError(f"layer {lid}: only 1-D and 2-D layers are supported, got shape {shape}")
    groups, where = [], {}
    for gi, key in enumerate(sorted(members)):
        mem = sorted(members[key])  # (layer, side 0=L 1=R, idx) sorts exactly like (layer, L<R, idx)
        for slot, mm in enumerate(mem):
            where[mm] = (gi, slot)
        dim, p = key
        groups.append({
            "dim": dim, "p": p,
            "members": tuple((l, "LR"[s], i) for (l, s, i) in mem),
            "ema": np.zeros((len(mem), dim, dim)),
            "roots": np.tile(np.eye(dim), (len(mem), 1, 1)),
        })
    for lid, lay in enumerate(layers):
        nb = len(lay["spans"]) if lay["spans"] is not None else len(lay["chunks"])
        lay["left"] = tuple(where[(lid, 0, i)] for i in range(nb))
        lay["right"] = tuple(where[(lid, 1, i)] for i in range(nb)) if lay["spans"] is not None else None
    return {
        "step": 0,
        "layers": layers,
        "groups": groups,
        "adam": [np.zeros(s) for s in shapes],
        "momentum": [np.zeros(s) for s in shapes] if momentum else None,
    }


def init_state(params, cfg: OracleConfig):
    """init_state (shampoo.py:233-235)."""
    return build_structure([tuple(p.shape) for p in params], cfg.block_size, cfg.beta1 > 0.0)


# ============================================================================ statistics
def _sym(x):
    return (x + x.T) / 2.0


def accumulate(state, grads, cfg: OracleConfig):
    """EMA of G G^T / G^T G per block, g g^T per chunk, Adam / momentum (shampoo.py:238-278)."""
    beta, b2 = cfg.beta_lr, cfg.beta2
    groups = state["groups"]
    if len(grads) != len(state["layers"]):
        raise ValueError("gradient count mismatch")
    for lay, g in zip(state["layers"], grads):
        if tuple(g.shape) != lay["shape"]:
            raise ValueError("gradient shape mismatch")
        if lay["spans"] is not None:
            for idx, ((r0, r1), (c0, c1)) in enumerate(lay["spans"]):
                blk = g[r0:r1, c0:c1]
                for (gi, slot), prod in ((lay["left"][idx], blk @ blk.T), (lay["right"][idx], blk.T @ blk)):
                    e = groups[gi]["ema"]
                    e[slot] = _sym(beta * e[slot] + (1.0 - beta) * prod)
        else:
            for idx, (s, t) in enumerate(lay["chunks"]):
                v = g[s:t][:, None]
                gi, slot = lay["left"][idx]
                e = groups[gi]["ema"]
                e[slot] = _sym(beta * e[slot] + (1.0 - beta) * (v @ v.T))
    for i, g in enumerate(grads):
        state["adam"][i] = b2 * state["adam"][i] + (1.0 - b2) * g * g
        if state["momentum"] is not None:
            state["momentum"][i] = cfg.beta1 * state["momentum"][i] + (1.0 - cfg.beta1) * g
    return state


# ============================================================================ seeds and scaling
def block_seed(seed, index):
    """Child seed = SeedSequence([seed, index]).generate_state(1, uint64)[0] (spectral.py:53-55)."""
    return int(np.random.SeedSequence([int(seed), int(index)]).generate_state(1, np.uint64)[0])


def start_vectors(n, pool, seed):
    """uniform(-1, 1) rows per vector from default_rng(seed), columns normalized (spectral.py:67-74)."""
    v = np.random.default_rng(seed).uniform(-1.0, 1.0, size=(pool, n)).T
    nrm = np.linalg.norm(v, axis=0)
    nrm[nrm == 0.0] = 1.0
    return v / nrm


def _power_pool(a, v, iters):
    """iters x (W = A V, normalize columns, dead columns -> 0) + quotients (spectral.py:77-84)."""
    for _ in range(iters):
        w = a @ v
        nrm = np.linalg.norm(w, axis=0)
        ok = nrm > 0.0
        v = np.where(ok[None, :], w / np.where(ok, nrm, 1.0)[None, :], 0.0)
    return v, np.einsum("ij,ij->j", v, a @ v)


RETRY_SALT = 0x5EED  # spectral.py:50


def multi_power_iteration(a, pool, iters, seed, return_vector=False):
    """Best Rayleigh quotient over the pool, one reseeded retry (spectral.py:87-112). Returns lambda
    (and the selected unit vector with return_vector=True)."""
    n = a.shape[0]
    v0 = start_vectors(n, pool, seed)
    v, q = _power_pool(a, v0, iters)
    alive = np.linalg.norm(v, axis=0) > 0.0
    if not alive.any() or q[alive].max() == 0.0:
        if np.linalg.norm(a) == 0.0:
            return (0.0, v0[:, 0]) if return_vector else 0.0
        v, q = _power_pool(a, start_vectors(n, pool, block_seed(seed, RETRY_SALT)), iters)
        alive = np.linalg.norm(v, axis=0) > 0.0
        if not alive.any() or q[alive].max() == 0.0:
            raise ArithmeticError("power iteration pool collapsed twice")
    best = int(np.argmax(np.where(alive, q, -np.inf)))
    x = v[:, best] / np.linalg.norm(v[:, best])
    lam = float(x @ (a @ x)) / float(x @ x)
    return (lam, x) if return_vector else lam


def group_scales(a, scaling, pool, iters, seed):
    """Frobenius norm or 2 * lambda_PI with per-block seeds (shampoo.py:294-298, spectral.py:115-117)."""
    if scaling == "fro":
        return np.sqrt((a * a).sum(axis=(1, 2)))
    return np.array([2.0 * multi_power_iteration(a[i], pool, iters, block_seed(seed, i))
                     for i in range(a.shape[0])])


# ============================================================================ matmul-only roots
class _Watch:
    """Divergence watch: last 4 residuals strictly rising and r4 > 10 r1 (roots.py:71-86)."""

    def __init__(self):
        self.h = []

    def push(self, r):
        self.h = (self.h + [r])[-4:]
        h = self.h
        return len(h) == 4 and h[0] < h[1] < h[2] < h[3] and h[3] > 10.0 * h[0]


def _eye_dist(m):
    n = m.shape[-1]
    return np.abs(m - np.eye(n)).max(axis=(1, 2))


def _freeze_update(k, res, active, reports, watches, last, tol):
    """Per-active-block freeze rules in reference order (roots.py:291-301 / 243-253)."""
    for i in np.flatnonzero(active):
        r = float(res[i])
        last[i] = r
        if not np.isfinite(r):
            reports[i], active[i] = IterationReport(k, r, False), False
        elif r <= tol:
            reports[i], active[i] = IterationReport(k, r, True), False
        elif watches[i].push(r):
            reports[i], active[i] = IterationReport(k, r, False), False


def batched_newton_db(a, tol=1e-10, max_iters=100):
    """Denman-Beavers with closed-form first step and per-block freezing (roots.py:262-305).

    Returns (Y ~ a^(1/2), Z ~ a^(-1/2), reports)."""
    nb, n = a.shape[0], a.shape[1]
    eye = np.eye(n)
    e = 1.5 * eye - 0.5 * a
    y = a @ e
    z = e.copy()
    res = _eye_dist(e)
    active = np.ones(nb, dtype=bool)
    reports = [None] * nb
    watches = [_Watch() for _ in range(nb)]
    last = res.copy()
    for i in range(nb):
        if res[i] <= tol:
            reports[i], active[i] = IterationReport(1, float(res[i]), True), False
        else:
            watches[i].push(float(res[i]))
    k = 1
    while active.any() and k < max_iters:
        k += 1
        e = 0.5 * (3.0 * eye - z @ y)
        e[~active] = eye
        y = y @ e
        z = e @ z
        _freeze_update(k, _eye_dist(e), active, reports, watches, last, tol)
    for i in range(nb):
        if reports[i] is None:
            reports[i] = IterationReport(max_iters, float(last[i]), False)
    return y, z, reports


def _q32(x, on):
    return x.astype(np.float32).astype(np.float64) if on else x


def _mm32(a, b, on):
    """EMULATED32 product: rank-1 updates accumulated in float32 (linalg.py:82-90)."""
    if not on:
        return a @ b
    a32, b32 = a.astype(np.float32), b.astype(np.float32)
    out = np.zeros(a.shape[:-1] + (b.shape[-1],), dtype=np.float32)
    for k in range(a.shape[-1]):
        out += a32[..., :, k, None] * b32[..., None, k, :]
    return out.astype(np.float64)


def batched_coupled_newton(a, p=2, tol=1e-10, max_iters=100, c=None, emulate32=False):
    """Coupled Newton for a^(-1/p) with per-block freezing (roots.py:216-259). Returns (X, reports)."""
    if p not in (2, 4):
        raise ValueError("p must be 2 or 4")
    nb, n = a.shape[0], a.shape[1]
    cc = c if c is not None else (1.0 + p) ** (-1.0 / p)
    eye = np.eye(n)
    x = _q32(np.tile(eye / cc, (nb, 1, 1)), emulate32)
    m = _q32(a / cc**p, emulate32)
    active = np.ones(nb, dtype=bool)
    reports = [None] * nb
    watches = [_Watch() for _ in range(nb)]
    last = np.full(nb, np.inf)
    for k in range(1, max_iters + 1):
        corr = _q32((1.0 + 1.0 / p) * eye - m / p, emulate32)
        corr[~active] = eye
        x = _mm32(x, corr, emulate32)
        cp = _mm32(corr, corr, emulate32)
        if p == 4:
            cp = _mm32(cp, cp, emulate32)
        m = _mm32(cp, m, emulate32)
        _freeze_update(k, _eye_dist(m), active, reports, watches, last, tol)
        if not active.any():
            break
    for i in range(nb):
        if reports[i] is None:
            reports[i] = IterationReport(max_iters, float(last[i]), False)
    return x, reports


# ============================================================================ Chebyshev
def cheb_coefficients(p, degree=60, points=1000, interval=None, eps=1e-10):
    """DCT projection of x^(-1/p) at Chebyshev nodes of [a, b] (chebyshev.py:46-84)."""
    lo, hi = interval if interval is not None else (eps, 1.0 + eps)
    theta = (2 * np.arange(points) + 1) * np.pi / (2 * points)
    x = 0.5 * (hi - lo) * np.cos(theta) + 0.5 * (hi + lo)
    c = (2.0 / points) * (np.cos(np.arange(degree + 1)[:, None] * theta[None, :]) @ np.power(x, -1.0 / p))
    c[0] *= 0.5
    return c, (lo, hi)


def batched_clenshaw(a, coeffs, scales, p, emulate32=False):
    """Optimized matrix Clenshaw, d-1 products, times scale^(-1/p) (chebyshev.py:137-184)."""
    d = len(coeffs) - 1
    n = a.shape[1]
    eye = np.eye(n)
    s = 2.0 * (a / scales[:, None, None]) - eye
    b1 = 2.0 * coeffs[d] * s + coeffs[d - 1] * eye
    b2 = coeffs[d] * np.tile(eye, (a.shape[0], 1, 1))
    for k in range(d - 2, 0, -1):
        b1, b2 = 2.0 * _mm32(s, b1, emulate32) - b2 + coeffs[k] * eye, b1
    out = _mm32(s, b1, emulate32) - b2 + coeffs[0] * eye
    return out * np.power(scales, -1.0 / p)[:, None, None]


# ============================================================================ refresh + step
_cheb_memo: dict = {}


def refresh(state, cfg: OracleConfig, seed=0):
    """Recompute inverse roots every update_freq steps (shampoo.py:312-349). Returns reports per group."""
    all_reports = []
    if state["step"] % cfg.update_freq != 0:
        return all_reports
    for gi, grp in enumerate(state["groups"]):
        p, n = grp["p"], grp["dim"]
        if cfg.method == "evd":
            grp["roots"] = evd_inverse_root(grp["ema"], p, cfg.heuristic, cfg.heuristic_eps)
            all_reports.append(())
            continue
        a = grp["ema"] + cfg.epsilon * np.eye(n)
        sc = group_scales(a, cfg.scaling, cfg.pool, cfg.pi_iters, block_seed(seed, gi))
        if (sc <= 0).any():
            raise ArithmeticError(f"non-positive scale in group of dim {n}")
        ahat = a / sc[:, None, None]
        if cfg.method == "cn":
            roots, rep = batched_coupled_newton(ahat, p, cfg.tolerance, cfg.max_iters, emulate32=cfg.emulate32)
            all_reports.append((rep,))
        elif cfg.method == "ndb":
            if p == 2:
                _, roots, rep = batched_newton_db(ahat, cfg.tolerance, cfg.max_iters)
                all_reports.append((rep,))
            else:
                y1, _, r1 = batched_newton_db(ahat, cfg.tolerance, cfg.max_iters)
                _, roots, r2 = batched_newton_db(y1, cfg.tolerance, cfg.max_iters)
                all_reports.append((r1, r2))
        else:
            key = (p, cfg.cheb_degree, cfg.cheb_points, cfg.cheb_interval)
            if key not in _cheb_memo:
                _cheb_memo[key] = cheb_coefficients(p, cfg.cheb_degree, cfg.cheb_points, cfg.cheb_interval)
            coeffs, _ = _cheb_memo[key]
            grp["roots"] = batched_clenshaw(a, coeffs, sc, p, cfg.emulate32)
            all_reports.append(())
            continue
        grp["roots"] = roots * np.power(sc, -1.0 / p)[:, None, None]
    return all_reports


def evd_inverse_root(ema, p, heuristic="relu", eps=1e-10):
    """Batched EVD inverse root of ema + eps I with the LEGACY / SHIFTED_RELU / ABS spectrum heuristics
    (eigensolver.py:133-179); numpy's eigh stands in for the reference's cyclic Jacobi (both converge to the
    float64 eigendecomposition)."""
    n = ema.shape[-1]
    lam, q = np.linalg.eigh(ema + eps * np.eye(n))
    if heuristic == "legacy":
        proc = lam - np.minimum(lam.min(axis=-1, keepdims=True), 0.0) + eps
    elif heuristic == "relu":
        proc = np.maximum(lam - eps - eps, 0.0)
    else:
        proc = np.abs(lam - eps) + eps
    if (~(proc > 0).any(axis=-1)).any():
        raise ArithmeticError("all eigenvalues removed by dampening heuristic")
    inv = np.where(proc > 0, np.power(np.where(proc > 0, proc, 1.0), -1.0 / p), 0.0)
    return (q * inv[..., None, :]) @ np.swapaxes(q, -1, -2)


def graft_scale(u, p):
    """||p||_F / ||u||_F, 0 when u vanishes (shampoo.py:352-359)."""
    nu = float(np.linalg.norm(u))
    return 0.0 if nu == 0.0 else float(np.linalg.norm(p)) / nu


def step(state, params, grads, cfg: OracleConfig, seed=0):
    """One optimizer step, returns (new params, state, reports) (shampoo.py:362-404)."""
    t = state["step"]
    accumulate(state, grads, cfg)
    reports = refresh(state, cfg, seed=block_seed(seed, t))
    eta = cfg.lr(t)
    n_acc = t + 1
    groups = state["groups"]
    out = []
    for li, (lay, theta, g) in enumerate(zip(state["layers"], params, grads)):
        theta = np.array(theta, dtype=np.float64, copy=True)
        num = g if cfg.beta1 == 0.0 else state["momentum"][li] / (1.0 - cfg.beta1 ** n_acc)
        direction = num / (cfg.graft_eps + np.sqrt(state["adam"][li] / (1.0 - cfg.beta2 ** n_acc)))
        if lay["spans"] is not None:
            for idx, ((r0, r1), (c0, c1)) in enumerate(lay["spans"]):
                gl, sl = lay["left"][idx]
                gr, sr = lay["right"][idx]
                u = (groups[gl]["roots"][sl] @ g[r0:r1, c0:c1]) @ groups[gr]["roots"][sr]
                theta[r0:r1, c0:c1] -= eta * graft_scale(u, direction[r0:r1, c0:c1]) * u
        else:
            for idx, (s0, e0) in enumerate(lay["chunks"]):
                gl, sl = lay["left"][idx]
                u = groups[gl]["roots"][sl] @ g[s0:e0][:, None]
                theta[s0:e0] -= eta * graft_scale(u, direction[s0:e0][:, None]) * u[:, 0]
        out.append(theta)
    state["step"] = t + 1
    return out, state, reports


# ============================================================================ synthetic inputs
def random_spd(n, cond, seed, scale=1.0):
    """SPD with geometric spectrum [scale/cond, scale] and a Haar-like basis (tasks.py:11-26)."""
    rng = np.random.default_rng(seed)
    q, r = np.linalg.qr(rng.standard_normal((n, n)))
    q = q * np.sign(np.diag(r))[None, :]
    lam = np.geomspace(1.0 / cond, 1.0, n) * scale
    return (q * lam[None, :]) @ q.T
