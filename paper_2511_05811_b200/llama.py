"""Llama-style decoder whose linear layers run the MOSS FP8 hot path
(BASELINE configs 3-5: ~125M model loss curves, Llama-2-7B-shape steps).

The reference's training harness is a 2-layer MLP (train.py:126-204); the
north_star replaces it with a Llama decoder whose every projection (QKV, O,
gate/up, down) is a ``MossLinear``.  Everything else is plain bf16 PyTorch
glue (RMSNorm, RoPE, causal SDPA, SwiGLU, the LM head and the cross
entropy), with FP32 master parameters updated by ``MossAdamW``.

``LlamaConfig(moss=False)`` builds the identical model with bf16 torch
linears — the full-precision baseline the quantized run is compared against
(test_train.py:53-60 band semantics).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.nn.functional as F
from torch import nn

from .nn import MossLinear
from .producers import AddRMSNormFn, CrossEntropyFn, RMSNormFn, RopeQKVFn, SwiGLUFn

__all__ = ["LlamaConfig", "LlamaModel", "MarkovTokens", "LLAMA_125M", "LLAMA2_7B"]


@dataclass(frozen=True)
class LlamaConfig:
    vocab: int = 32000
    d_model: int = 768
    n_layers: int = 12
    n_heads: int = 12
    d_ffn: int = 2048
    max_seq: int = 4096
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    init_std: float = 0.02
    moss: bool = True
    interval: int = 500
    compute_dtype: torch.dtype = torch.bfloat16
    fp8_backward: bool = True       # False: reference semantics, full-precision backward (train.py:187-192)
    fused_ops: bool = True          # sm_100a producer kernels (RMSNorm/SwiGLU/RoPE + amax); False: torch glue

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def linear_params_per_layer(self) -> int:
        return 4 * self.d_model * self.d_model + 3 * self.d_model * self.d_ffn

    def gemm_flops_per_token(self) -> int:
        """6 x parameters of the FP8 linears (fwd + dgrad + wgrad), SURVEY.md 8(d)."""
        return 6 * self.n_layers * self.linear_params_per_layer()


LLAMA_125M = LlamaConfig(vocab=32000, d_model=768, n_layers=12, n_heads=12, d_ffn=2048)
LLAMA2_7B = LlamaConfig(vocab=32000, d_model=4096, n_layers=32, n_heads=32, d_ffn=11008)


class _BF16Linear(nn.Module):
    """Baseline linear: FP32 master weight, bf16 compute (cuBLAS)."""

    def __init__(self, d_in: int, d_out: int, device, std: float):
        super().__init__()
        self.weight = nn.Parameter(torch.empty(d_out, d_in, device=device).normal_(0.0, std))

    def forward(self, x):
        return F.linear(x, self.weight.to(x.dtype))


_LINEAR_FACTORY = None   # test hook: callable(cfg, d_in, d_out, device) -> nn.Module


def _linear(cfg: LlamaConfig, d_in: int, d_out: int, device):
    if _LINEAR_FACTORY is not None:
        return _LINEAR_FACTORY(cfg, d_in, d_out, device)
    if cfg.moss:
        return MossLinear(d_in, d_out, device=device, interval=cfg.interval, init_std=cfg.init_std,
                          fp8_backward=cfg.fp8_backward)
    return _BF16Linear(d_in, d_out, device, cfg.init_std)


class RMSNorm(nn.Module):
    def __init__(self, d: int, eps: float, device):
        super().__init__()
        self.eps = eps
        self.weight = nn.Parameter(torch.ones(d, device=device))

    def forward(self, x):
        xf = x if x.dtype == torch.float64 else x.float()
        y = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps)
        return (y * self.weight).to(x.dtype)


def _rope_tables(cfg: LlamaConfig, device):
    hd = cfg.head_dim
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, hd, 2, device=device, dtype=torch.float32) / hd))
    t = torch.arange(cfg.max_seq, device=device, dtype=torch.float32)
    f = torch.outer(t, inv)
    return f.cos(), f.sin()


def _apply_rope(x, cos, sin):
    # x [B, H, S, hd]; rotate pairs (even, odd)
    up = (lambda t: t) if x.dtype == torch.float64 else (lambda t: t.float())
    x1, x2 = up(x[..., 0::2]), up(x[..., 1::2])
    c, s = cos[: x.shape[2]][None, None], sin[: x.shape[2]][None, None]
    out = torch.stack((x1 * c - x2 * s, x1 * s + x2 * c), dim=-1).flatten(-2)
    return out.to(x.dtype)


class Block(nn.Module):
    def __init__(self, cfg: LlamaConfig, device):
        super().__init__()
        d, f = cfg.d_model, cfg.d_ffn
        self.cfg = cfg
        self.attn_norm = RMSNorm(d, cfg.norm_eps, device)
        self.qkv = _linear(cfg, d, 3 * d, device)
        self.o = _linear(cfg, d, d, device)
        self.mlp_norm = RMSNorm(d, cfg.norm_eps, device)
        self.gate_up = _linear(cfg, d, 2 * f, device)
        self.down = _linear(cfg, f, d, device)
        self.fused = cfg.fused_ops and all(isinstance(m, MossLinear) for m in (self.qkv, self.o, self.gate_up, self.down))

    def forward(self, x, cos, sin, delta=None, prev=None):
        """Returns the block output.  Fused path (``cfg.fused_ops`` with MOSS
        linears): takes and returns the residual stream lazily as (x, delta)
        with x + delta folded into the next RMSNorm kernel; ``prev`` is the
        MossLinear that produced delta (its dY comes out of that kernel)."""
        if self.fused:
            return self._forward_fused(x, cos, sin, delta, prev)
        if delta is not None:
            x = x + delta
        B, S, d = x.shape
        H, hd = self.cfg.n_heads, self.cfg.head_dim
        q, k, v = self.qkv(self.attn_norm(x)).split(d, dim=-1)
        q = _apply_rope(q.view(B, S, H, hd).transpose(1, 2), cos, sin)
        k = _apply_rope(k.view(B, S, H, hd).transpose(1, 2), cos, sin)
        v = v.view(B, S, H, hd).transpose(1, 2)
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + self.o(a.transpose(1, 2).reshape(B, S, d))
        g, u = self.gate_up(self.mlp_norm(x)).split(self.cfg.d_ffn, dim=-1)
        return x + self.down(F.silu(g) * u), None

    def _forward_fused(self, x, cos, sin, delta, prev):
        B, S, d = x.shape
        H = self.cfg.n_heads
        eps = self.cfg.norm_eps
        if delta is None:
            y, am = RMSNormFn.apply(x, self.attn_norm.weight, eps, prev)
        else:
            x, y, am = AddRMSNormFn.apply(x, delta, self.attn_norm.weight, eps, prev)
        q, k, v = RopeQKVFn.apply(self.qkv(y, am), cos, sin, H, self.qkv)
        a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        o = self.o(a.transpose(1, 2).reshape(B, S, d))
        x, y, am = AddRMSNormFn.apply(x, o, self.mlp_norm.weight, eps, self.o)
        h, am = SwiGLUFn.apply(self.gate_up(y, am), self.gate_up)
        return x, self.down(h, am)


class LlamaModel(nn.Module):
    def __init__(self, cfg: LlamaConfig, device="cuda"):
        super().__init__()
        self.cfg = cfg
        self.embed = nn.Parameter(torch.empty(cfg.vocab, cfg.d_model, device=device).normal_(0.0, cfg.init_std))
        self.blocks = nn.ModuleList([Block(cfg, device) for _ in range(cfg.n_layers)])
        self.norm = RMSNorm(cfg.d_model, cfg.norm_eps, device)
        self.head = nn.Parameter(torch.empty(cfg.vocab, cfg.d_model, device=device).normal_(0.0, cfg.init_std))
        cos, sin = _rope_tables(cfg, device)
        self.register_buffer("cos", cos, persistent=False)
        self.register_buffer("sin", sin, persistent=False)

    def forward(self, tokens: torch.Tensor, targets: torch.Tensor | None = None):
        x = F.embedding(tokens, self.embed).to(self.cfg.compute_dtype)
        delta, prev = None, None
        for blk in self.blocks:
            x, delta = blk(x, self.cos, self.sin, delta, prev)
            prev = blk.down
        if delta is not None:
            _, x, _ = AddRMSNormFn.apply(x, delta, self.norm.weight, self.cfg.norm_eps, prev)
        else:
            x = self.norm(x)
        logits = F.linear(x, self.head.to(self.cfg.compute_dtype))
        if targets is None:
            return logits
        if self.blocks[0].fused and logits.dtype == torch.bfloat16 and logits.shape[-1] % 8 == 0:
            return CrossEntropyFn.apply(logits, targets)       # fused f32 log-softmax on the bf16 logits
        lg = logits if logits.dtype == torch.float64 else logits.float()
        return F.cross_entropy(lg.reshape(-1, lg.shape[-1]), targets.reshape(-1))

    @staticmethod
    def no_decay(name: str, p: nn.Parameter) -> bool:
        """Norm weights and the embedding are not decayed (usual Llama practice)."""
        return p.dim() == 1 or name == "embed"


class MarkovTokens:
    """Seeded synthetic token stream with learnable structure: a fixed random
    sparse Markov chain (each token has ``fanout`` successors with Dirichlet
    probabilities), so the loss falls from ln(V) towards the chain's entropy."""

    def __init__(self, vocab: int, seed: int = 0, fanout: int = 4, active: int | None = None):
        rng = np.random.default_rng(seed)
        self.vocab = active or vocab       # states actually visited (<= model vocab)
        vocab = self.vocab
        self.succ = rng.integers(0, vocab, size=(vocab, fanout))
        self.prob = rng.dirichlet(np.ones(fanout) * 0.5, size=vocab)
        self.cum = np.cumsum(self.prob, axis=1)
        self.rng = np.random.default_rng(seed + 1)

    def batch(self, batch: int, seq: int) -> tuple[np.ndarray, np.ndarray]:
        out = np.empty((batch, seq + 1), dtype=np.int64)
        out[:, 0] = self.rng.integers(0, self.vocab, size=batch)
        u = self.rng.random((batch, seq))
        for t in range(seq):
            cur = out[:, t]
            j = (u[:, t, None] > self.cum[cur]).sum(axis=1)
            out[:, t + 1] = self.succ[cur, np.minimum(j, self.succ.shape[1] - 1)]
        return out[:, :-1], out[:, 1:]

    def entropy(self) -> float:
        p = self.prob
        return float(-(p * np.log(p + 1e-30)).sum(axis=1).mean())
