"""Llama-style decoder for config 5's full training step (model forward / backward around the DASH step).

Harness code outside the optimizer hot path: BASELINE config 5 times "fused stat update +
scaling + Newton-DB + grafted apply" inside a real training step of the Llama-style ~1B model of §8(d)
(E = 2048, 16 layers, SwiGLU F = 5632, V = 32000, untied embedding / head, RMSNorm).  The
parameters are registered in exactly the order of ``tests/golden/cases.llama_953m`` -- embedding, then per layer
wq wk wv wo w1 w3 w2 attn_norm ffn_norm, then the final norm and the head -- so the optimizer state, block
table and preconditioner groups are those of the optimizer-only benchmark.  Master weights are fp32; the
forward runs under bf16 autocast with PyTorch's fused attention (a library kernel, like cuBLAS).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F


@dataclass(frozen=True)
class LlamaShape:
    dim: int = 2048
    layers: int = 16
    ffn: int = 5632
    vocab: int = 32000
    heads: int = 16
    norm_eps: float = 1e-5
    rope_base: float = 10000.0

    def param_shapes(self) -> list[tuple[int, ...]]:
        e, f, v = self.dim, self.ffn, self.vocab
        shapes = [(v, e)]
        for _ in range(self.layers):
            shapes += [(e, e)] * 4 + [(f, e), (f, e), (e, f), (e,), (e,)]
        return shapes + [(e,), (v, e)]


def init_params(shape: LlamaShape, device, seed: int = 0) -> list[torch.Tensor]:
    """fp32 master weights: N(0, 0.02^2) matrices (output projections scaled by 1/sqrt(2 layers)), unit norms."""
    g = torch.Generator(device=device).manual_seed(seed)
    out = []
    for i, s in enumerate(shape.param_shapes()):
        if len(s) == 1:
            out.append(torch.ones(s, device=device))
            continue
        std = 0.02
        per_layer = (i - 1) % 9 if 0 < i < 1 + 9 * shape.layers else -1
        if per_layer in (3, 6):  # wo, w2: residual-branch outputs
            std /= math.sqrt(2 * shape.layers)
        out.append(torch.randn(s, device=device, generator=g) * std)
    for p in out:
        p.requires_grad_(True)
    return out


def _rms(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    x32 = x.float()
    return (x32 * torch.rsqrt(x32.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype) * w.to(x.dtype)


def _rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    x1, x2 = x[..., 0::2], x[..., 1::2]
    return torch.stack((x1 * cos - x2 * sin, x1 * sin + x2 * cos), dim=-1).flatten(-2)


def loss_fn(params: list[torch.Tensor], tokens: torch.Tensor, shape: LlamaShape) -> torch.Tensor:
    """Next-token cross entropy of a (batch, seq) token block; params in param_shapes() order."""
    b, t = tokens.shape
    hd = shape.dim // shape.heads
    pos = torch.arange(t, device=tokens.device, dtype=torch.float32)
    inv = shape.rope_base ** (-torch.arange(0, hd, 2, device=tokens.device, dtype=torch.float32) / hd)
    ang = pos[:, None] * inv[None, :]
    cos, sin = ang.cos().to(torch.bfloat16), ang.sin().to(torch.bfloat16)
    with torch.autocast("cuda", dtype=torch.bfloat16):
        h = F.embedding(tokens[:, :-1], params[0]).to(torch.bfloat16)
        tq = t - 1
        cq, sq = cos[:tq], sin[:tq]
        for layer in range(shape.layers):
            wq, wk, wv, wo, w1, w3, w2, n_attn, n_ffn = params[1 + 9 * layer: 10 + 9 * layer]
            x = _rms(h, n_attn, shape.norm_eps)
            q = (x @ wq.t()).view(b, tq, shape.heads, hd)
            k = (x @ wk.t()).view(b, tq, shape.heads, hd)
            v = (x @ wv.t()).view(b, tq, shape.heads, hd)
            q, k = _rope(q, cq[:, None], sq[:, None]), _rope(k, cq[:, None], sq[:, None])
            att = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                                 is_causal=True)
            h = h + att.transpose(1, 2).reshape(b, tq, shape.dim) @ wo.t()
            x = _rms(h, n_ffn, shape.norm_eps)
            h = h + (F.silu(x @ w1.t()) * (x @ w3.t())) @ w2.t()
        h = _rms(h, params[-2], shape.norm_eps)
        logits = h @ params[-1].t()
    return F.cross_entropy(logits.float().reshape(-1, shape.vocab), tokens[:, 1:].reshape(-1))


class TrainStep:
    """One full training step: forward, backward, then the DASH optimizer step on the parameter gradients
    (shampoo.step with CUDA tensors, updated in place)."""

    def __init__(self, shape: LlamaShape, cfg, device, seed: int = 0):
        from .shampoo import init_state

        self.shape, self.cfg = shape, cfg
        self.params = init_params(shape, device, seed)
        self.state = init_state([p.detach() for p in self.params], cfg)

    def __call__(self, tokens: torch.Tensor, seed: int = 0, events: dict | None = None) -> torch.Tensor:
        from .shampoo import step

        for p in self.params:
            p.grad = None
        loss = loss_fn(self.params, tokens, self.shape)
        loss.backward()
        if events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            events.setdefault("backward_done", []).append(ev)
        with torch.no_grad():
            step(self.state, [p.detach() for p in self.params], [p.grad for p in self.params], self.cfg, seed=seed,
                 inplace=True, events=events)
        return loss.detach()
