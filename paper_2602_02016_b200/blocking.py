"""Gradient blocking: the integer block table (bit-exact with the reference) and device partitioning.

Mirrors ``blocking.py``'s layout API (``PartitionLayout`` ``:29-44``, ``partition_layout`` ``:62-81``,
``partition`` ``:84-98``, ``reassemble`` ``:101-120``, ``preconditioner_shapes`` ``:123-132``): a layer of
shape (m, n) is cut into full B x B blocks in row-major order, then ragged remainder blocks in
row-major cell order.  On the B200 the blocks are never copied on the host: the step kernels read
them straight out of the flat gradient through this table (``dash_block`` in include/dash_b200.h).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Iterator

import numpy as np
import torch

Span = tuple[tuple[int, int], tuple[int, int]]


@dataclass(frozen=True)
class PartitionLayout:
    """Shape-level description of a blocked layer (no data)."""

    layer_shape: tuple[int, int]
    block_size: int
    full_spans: tuple[Span, ...]
    remainder_spans: tuple[Span, ...]

    @property
    def block_spans(self) -> tuple[Span, ...]:
        return self.full_spans + self.remainder_spans

    @property
    def num_blocks(self) -> int:
        return len(self.full_spans) + len(self.remainder_spans)


def partition_layout(shape: tuple[int, int], block_size: int) -> PartitionLayout:
    """Full spans over the divisible region, then edge cells with i >= m//B or j >= n//B."""
    m, n = (int(shape[0]), int(shape[1]))
    b = int(block_size)
    if b < 1:
        raise ValueError("block size must be >= 1")
    n_m, n_n = m // b, n // b
    rows = [(i * b, min(i * b + b, m)) for i in range(-(-m // b))]
    cols = [(j * b, min(j * b + b, n)) for j in range(-(-n // b))]
    full = tuple((rows[i], cols[j]) for i in range(n_m) for j in range(n_n))
    rest = tuple((rows[i], cols[j]) for i in range(len(rows)) for j in range(len(cols)) if i >= n_m or j >= n_n)
    return PartitionLayout(layer_shape=(m, n), block_size=b, full_spans=full, remainder_spans=rest)


@dataclass
class BlockPartition:
    """A blocked gradient: layout plus block views (device tensors, no copies)."""

    layout: PartitionLayout
    full_blocks: torch.Tensor | np.ndarray
    remainder_blocks: tuple[tuple[Span, object], ...]

    def blocks(self) -> Iterator[tuple[Span, object]]:
        for i, span in enumerate(self.layout.full_spans):
            yield span, self.full_blocks[i]
        yield from self.remainder_blocks


def partition(g, block_size: int) -> BlockPartition:
    """Split a gradient matrix into full B x B blocks (stacked) plus ragged edge blocks."""
    layout = partition_layout(tuple(g.shape), block_size)
    b = block_size
    if isinstance(g, torch.Tensor):
        nm, nn = g.shape[0] // b, g.shape[1] // b
        full = g[: nm * b, : nn * b].reshape(nm, b, nn, b).permute(0, 2, 1, 3).reshape(nm * nn, b, b)
    else:
        nm, nn = g.shape[0] // b, g.shape[1] // b
        full = np.ascontiguousarray(g[: nm * b, : nn * b].reshape(nm, b, nn, b).transpose(0, 2, 1, 3)).reshape(
            nm * nn, b, b)
    rest = tuple((span, g[span[0][0]:span[0][1], span[1][0]:span[1][1]]) for span in layout.remainder_spans)
    return BlockPartition(layout=layout, full_blocks=full, remainder_blocks=rest)


def reassemble(p: BlockPartition | PartitionLayout, blocks: Iterable[tuple[Span, object]]):
    """Rebuild the layer matrix from (span, block) pairs in any order (blocking.py:101-120)."""
    layout = p.layout if isinstance(p, BlockPartition) else p
    expected = set(layout.block_spans)
    seen: set[Span] = set()
    out = None
    for span, data in blocks:
        if span not in expected:
            raise ValueError(f"unknown block span {span}")
        if span in seen:
            raise ValueError(f"duplicate block span {span}")
        (r0, r1), (c0, c1) = span
        if tuple(data.shape) != (r1 - r0, c1 - c0):
            raise ValueError(f"block at {span} has shape {tuple(data.shape)}, expected {(r1 - r0, c1 - c0)}")
        if out is None:
            out = (torch.empty(layout.layer_shape, dtype=data.dtype, device=data.device)
                   if isinstance(data, torch.Tensor) else np.empty(layout.layer_shape))
        out[r0:r1, c0:c1] = data
        seen.add(span)
    missing = expected - seen
    if missing:
        raise ValueError(f"missing blocks for spans {sorted(missing)}")
    return out


def preconditioner_shapes(p: BlockPartition | PartitionLayout):
    """Left/right preconditioner shapes per block, in canonical block order."""
    layout = p.layout if isinstance(p, BlockPartition) else p
    left = [(r1 - r0, r1 - r0) for (r0, r1), _ in layout.block_spans]
    right = [(c1 - c0, c1 - c0) for _, (c0, c1) in layout.block_spans]
    return left, right


def chunk_bounds(length: int, block_size: int) -> tuple[tuple[int, int], ...]:
    """1-D layer chunks [s, min(s + B, len)) (shampoo.py:171-173)."""
    return tuple((s, min(s + block_size, length)) for s in range(0, length, block_size))
