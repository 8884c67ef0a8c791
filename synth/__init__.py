"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no log-softmax, no weights, no
normalisation, no resampling): it only draws logits, drafted tokens, log-weight
priors and KV bit patterns with the shapes and value distributions of the paper's
workloads (recipe: DESIGN.md section 5).  Both sides receive the same tensors.

Recipe (LM-like logits; the paper gives no logit statistics):
  target row  z^p_v = 2.5 g_v, g ~ N(0,1), plus h ~ U{1..8} "head" tokens raised by U(8,18)
  draft row   z^q   = z^p + sigma_d g'  (sigma_d = 0 identical models, 0.5 default, 1.5 low ESS)
  drafted token d_j ~ q (Gumbel-max on tau_q z^q; the draft model itself is out of scope)
  target tensor has K+1 rows per particle (K scored rows + the bonus row)
"""
from __future__ import annotations

import math

import torch

GEN_SEED_BASE = 20260415          # generator seed = GEN_SEED_BASE + config id
PHILOX_SEED = 0x5EED5EED          # resampling seed used by tests and bench


def padded_ld(V: int, dtype: torch.dtype) -> int:
    """Smallest row pitch >= V that keeps every row 16-byte aligned."""
    vec = 8 if dtype == torch.bfloat16 else 4
    return (V + vec - 1) // vec * vec


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def lm_logits(P: int, N: int, K: int, V: int, *, dtype=torch.bfloat16, seed: int = GEN_SEED_BASE,
              sigma_d: float = 0.5, tau_q: float = 1.0, ld: int | None = None, bonus: bool = True,
              pad_value: float = float("nan"), device="cpu", chunk_rows: int = 2048):
    """Returns (logits_p [P,N,K+bonus,ld], logits_q [P,N,K,ld], tokens [P,N,K] int32).

    Columns >= V are padding filled with ``pad_value`` (NaN by default, so any read of the
    padding poisons the result).  Generation is chunked so multi-GB configs fit.
    """
    ld = padded_ld(V, dtype) if ld is None else ld
    assert ld >= V
    rp = K + (1 if bonus else 0)
    g = _gen(seed, device)
    lp = torch.empty((P, N, rp, ld), dtype=dtype, device=device)
    lq = torch.empty((P, N, K, ld), dtype=dtype, device=device)
    tok = torch.empty((P, N, K), dtype=torch.int32, device=device)
    if ld > V:
        lp[..., V:] = pad_value
        lq[..., V:] = pad_value
    flat_p = lp.view(P * N, rp, ld)
    flat_q = lq.view(P * N, K, ld)
    flat_t = tok.view(P * N, K)
    pn_per_chunk = max(1, chunk_rows // rp)
    for s in range(0, P * N, pn_per_chunk):
        e = min(P * N, s + pn_per_chunk)
        rows = (e - s) * rp
        z = torch.randn((rows, V), generator=g, device=device, dtype=torch.float32) * 2.5
        h = torch.randint(1, 9, (rows, 1), generator=g, device=device)
        pos = torch.randint(0, V, (rows, 8), generator=g, device=device)
        amt = torch.rand((rows, 8), generator=g, device=device) * 10.0 + 8.0
        amt = amt * (torch.arange(8, device=device)[None, :] < h)
        z.scatter_add_(1, pos, amt)
        zp = z.view(e - s, rp, V)
        flat_p[s:e, :, :V] = zp.to(dtype)
        zq = zp[:, :K, :] + sigma_d * torch.randn((e - s, K, V), generator=g, device=device)
        zq_c = zq.to(dtype)
        flat_q[s:e, :, :V] = zq_c
        # draft phase stand-in: d ~ softmax(tau_q z^q) by Gumbel-max on the stored values
        gum = -torch.log(-torch.log(torch.rand((e - s, K, V), generator=g, device=device)
                                    .clamp_(1e-12, 1.0 - 1e-7)))
        flat_t[s:e] = torch.argmax(zq_c.float() * tau_q + gum, dim=-1).to(torch.int32)
        del z, zp, zq, zq_c, gum
    return lp, lq, tok


def uniform_prior(P: int, N: int, device="cpu") -> torch.Tensor:
    """lambda_prev = fl32(-ln N) for every particle (the state right after a reset)."""
    return torch.full((P, N), -math.log(N), dtype=torch.float32, device=device)


def random_logw(P: int, N: int, *, seed: int, sigma: float = 1.0, neg_inf_frac: float = 0.0,
                device="cpu") -> torch.Tensor:
    """Gaussian log-weights, optionally with a fraction of -inf (zero-weight) particles."""
    g = _gen(seed, device)
    lw = torch.randn((P, N), generator=g, device=device) * sigma
    if neg_inf_frac > 0:
        mask = torch.rand((P, N), generator=g, device=device) < neg_inf_frac
        lw[mask] = -float("inf")
    return lw.float()


def kv_bits(shape, *, seed: int, device="cpu") -> torch.Tensor:
    """Random 16-bit patterns (any bf16 bit pattern, NaN payloads included) as int16."""
    g = _gen(seed, device)
    return torch.randint(-32768, 32768, tuple(shape), generator=g, device=device, dtype=torch.int32) \
        .to(torch.int16)


def kv_bits_fast(shape, *, seed: int, device="cuda") -> torch.Tensor:
    """Same distribution as kv_bits for multi-GB caches: uniform int32 words viewed as int16."""
    g = _gen(seed, device)
    numel = 1
    for s in shape:
        numel *= s
    assert numel % 2 == 0
    w = torch.randint(-2 ** 31, 2 ** 31, (numel // 2,), generator=g, device=device, dtype=torch.int32)
    return w.view(torch.int16).view(tuple(shape))


def dirichlet_rows(n_rows: int, V: int, *, seed: int, conc: float = 1.0) -> torch.Tensor:
    """Random probability rows (fp64) for the tiny enumeration fixtures."""
    g = _gen(seed, "cpu")
    x = (-torch.log(torch.rand((n_rows, V), generator=g, dtype=torch.float64))) ** (1.0 / conc)
    return x / x.sum(dim=1, keepdim=True)
