"""Helpers shared by the -m gpu parity tests: move the same seeded inputs to both sides."""
import numpy as np
import torch


def to_host(t: torch.Tensor) -> np.ndarray:
    """Logits tensor -> numpy for the oracle (bf16 as raw uint16 bits, fp32 as float32)."""
    t = t.detach().cpu().contiguous()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def np_(t):
    return None if t is None else t.detach().cpu().numpy()


def max_abs(a, b, mask=None):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_inf = (a == b)
    d = np.where(both_inf, 0.0, np.abs(a - b))
    d = np.where(np.isnan(a) & np.isnan(b), 0.0, d)
    if mask is not None:
        d = d[mask]
    return float(np.max(d)) if d.size else 0.0
