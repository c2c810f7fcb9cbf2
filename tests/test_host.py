"""CPU tests: host-side logic of the B200 package (no GPU needed).

Block structure bit-exactness, seeds, config validation, and that the C-ABI library loads and exports
every symbol declared in include/dash_b200.h (no compute calls).
"""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2602_02016_b200 import _lib
from paper_2602_02016_b200.blocking import chunk_bounds, partition, partition_layout, reassemble
from paper_2602_02016_b200.shampoo import (GraftConfig, LrSchedule, ShampooConfig, SolverConfig, build_layout)
from paper_2602_02016_b200.spectral import PowerIterationScaling, block_seed

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "dash_b200.h").read_text()
    declared = set(re.findall(r"\b(dash_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    lib = _lib.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), f"libdash_b200.so does not export {name}"
    assert declared == set(_lib.exported_symbols()), "ctypes signature table out of sync with the header"
    assert lib.dash_version().startswith(b"dash-b200")


def test_structure_bit_exact_vs_golden(golden):
    for name, case in golden["structure"].items():
        layers, specs = build_layout([tuple(s) for s in case["shapes"]], case["block_size"])
        assert [[g.dim, g.exponent, len(g.members)] for g in specs] == case["groups"], name
        assert [[[r.group, r.slot] for r in l.left_refs] for l in layers] == case["left"], name
        assert [None if l.right_refs is None else [[r.group, r.slot] for r in l.right_refs] for l in layers] \
            == case["right"], name
        assert [None if l.layout is None else [list(map(list, s)) for s in l.layout.block_spans] for l in layers] \
            == case["spans"], name
        if case["members"] is not None:
            assert [[list(m) for m in g.members] for g in specs] == case["members"]


@pytest.mark.parametrize("shape,b", [((37, 53), 16), ((32000, 2048), 1024), ((5, 5), 7), ((1024, 1024), 256),
                                     ((50304, 768), 1024), ((1, 9), 4)])
def test_partition_roundtrip_and_coverage(shape, b):
    rng = np.random.default_rng(0)
    g = rng.standard_normal(shape)
    part = partition(g, b)
    back = reassemble(part, list(part.blocks()))
    np.testing.assert_array_equal(back, g)
    lay = partition_layout(shape, b)
    cover = np.zeros(shape, dtype=int)
    for (r0, r1), (c0, c1) in lay.block_spans:
        cover[r0:r1, c0:c1] += 1
    assert (cover == 1).all()


def test_reassemble_rejects_bad_input():
    lay = partition_layout((8, 8), 4)
    blocks = [(s, np.zeros((4, 4))) for s in lay.block_spans]
    with pytest.raises(ValueError):
        reassemble(lay, blocks[:-1])
    with pytest.raises(ValueError):
        reassemble(lay, blocks + blocks[:1])


def test_chunk_bounds():
    assert chunk_bounds(10, 4) == ((0, 4), (4, 8), (8, 10))
    assert chunk_bounds(8, 8) == ((0, 8),)


@pytest.mark.parametrize("a,b", [(0, 0), (1, 2), (12345, 7), (2**63 + 5, 3), (2**40, 2**33), (2**64 - 1, 2**64 - 1)])
def test_block_seed_matches_numpy(a, b):
    want = int(np.random.SeedSequence([a, b]).generate_state(1, np.uint64)[0])
    assert block_seed(a, b) == want


def test_block_seed_golden(golden):
    s = golden["seeds"]
    for (a, b), want in zip(s["pairs"].tolist(), s["seeds"].tolist()):
        assert block_seed(a, b) == want


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        ShampooConfig(beta_lr=0.0)
    with pytest.raises(ValueError):
        ShampooConfig(epsilon=0.0)
    with pytest.raises(ValueError):
        ShampooConfig(update_freq=0)
    with pytest.raises(ValueError):
        ShampooConfig(block_size=0)
    with pytest.raises(ValueError):
        SolverConfig(method="qr")
    with pytest.raises(ValueError):
        GraftConfig(beta2=1.0)
    with pytest.raises(ValueError):
        GraftConfig(graft_eps=0.0)
    with pytest.raises(ValueError):
        LrSchedule(kind="linear")
    with pytest.raises(ValueError):
        PowerIterationScaling(pool=0)
    assert LrSchedule(kind="cosine", total_steps=10, base=1.0, final=0.0).value(10) == pytest.approx(0.0)
    assert LrSchedule(kind="linear", total_steps=4, base=1.0, final=0.0).value(2) == pytest.approx(0.5)
    assert SolverConfig(tolerance=0.0).require_convergence is False


def test_layer_rank_validation():
    with pytest.raises(ValueError):
        build_layout([(2, 2, 2)], 4)
