"""Synthetic KV on the device with the reference generator's distribution
(tensors.py:79-105): N(0,1) per element times a per-(layer, head, channel)
LogNormal(0, 0.5) scale, with max(1, round(0.01*C)) outlier channels per
(layer, head) scaled by 10; head importance U(0,1).  Drawn with a CUDA
generator (not numpy's stream), then rounded to bf16 — the serving dtype."""

from __future__ import annotations

import torch


def synthetic_kv(layers: int, heads: int, tokens: int, channels: int, seed: int = 0, device=None,
                 dtype: torch.dtype = torch.bfloat16, outlier_fraction: float = 0.01, outlier_scale: float = 10.0):
    """Returns (kv (L,H,T,C) `dtype` on `device`, importance float64 numpy (L,H))."""
    device = torch.device(device) if device is not None else torch.device("cuda")
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    scales = torch.exp(0.5 * torch.randn(layers, heads, channels, generator=g, device=device))
    n_hot = max(1, round(outlier_fraction * channels))
    hot = torch.rand(layers, heads, channels, generator=g, device=device).argsort(dim=-1)[..., :n_hot]
    scales.scatter_(-1, hot, scales.gather(-1, hot) * outlier_scale)
    out = torch.empty(layers, heads, tokens, channels, dtype=dtype, device=device)
    for li in range(layers):  # one layer at a time keeps the fp32 temporary small
        z = torch.randn(heads, tokens, channels, generator=g, device=device)
        out[li] = (z * scales[li, :, None, :]).to(dtype)
    imp = torch.rand(layers, heads, generator=g, device=device, dtype=torch.float64).cpu().numpy()
    return out, imp
