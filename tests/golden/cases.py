"""Layer-shape lists shared by the golden generator and the tests (no reference import here)."""

# Mini golden case and a ragged set exercising remainder blocks and 1-D chunks.
MINI = [(40, 24), (24,), (24, 40)]
RAGGED = [(37, 53), (5,), (16, 33), (33,)]
C1 = [(1024, 1024)]
# Warm case: every block's statistics become full rank within the 8 steps (tolerance-mode parity).
WARM = [(48, 32), (32, 48)]
STEP_CASES = (("mini", MINI, 16, 3), ("ragged", RAGGED, 8, 3), ("warm", WARM, 16, 8))


def llama_124m():
    """Llama-style 124M: E=768, 12 layers, SwiGLU F=2048, V=50304 tied."""
    e, layers, f, v = 768, 12, 2048, 50304
    shapes = [(v, e)]
    for _ in range(layers):
        shapes += [(e, e)] * 4 + [(f, e), (f, e), (e, f), (e,), (e,)]
    shapes += [(e,)]
    return shapes


def llama_953m():
    """Llama-style ~1B (953,223,168 params): E=2048, 16 layers, F=5632, V=32000 untied."""
    e, layers, f, v = 2048, 16, 5632, 32000
    shapes = [(v, e)]
    for _ in range(layers):
        shapes += [(e, e)] * 4 + [(f, e), (f, e), (e, f), (e,), (e,)]
    shapes += [(e,), (v, e)]
    return shapes


# Solver configurations of the golden optimizer-step fixtures (reference SolverConfig kwargs).
STEP_METHODS = ("ndb", "cn", "cbshv", "ndbfix", "ndbfro", "ndbtol5", "cntol5", "cnfix4", "ndbfrofix", "evd")


def solver_kwargs(method, spectral):
    """SolverConfig kwargs per fixture name; `spectral` provides Frobenius (reference or B200 module)."""
    return {
        "ndb": dict(method="ndb"),
        "cn": dict(method="cn"),
        "cbshv": dict(method="cbshv"),
        "ndbfix": dict(method="ndb", tolerance=0.0, max_iters=10),
        "ndbfro": dict(method="ndb", scaling=spectral.Frobenius()),
        "ndbtol5": dict(method="ndb", tolerance=1e-5),
        "cntol5": dict(method="cn", tolerance=1e-5),
        "cnfix4": dict(method="cn", tolerance=0.0, max_iters=8),
        "ndbfrofix": dict(method="ndb", scaling=spectral.Frobenius(), tolerance=0.0, max_iters=10),
        "evd": dict(method="evd"),
    }[method]


def uses_momentum(method):
    return method in ("cn", "cntol5")
