"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Bars (north star): log-weights within 1e-4 absolute; ancestors,
offspring, slot plans, resampled flags, reset values and KV bytes bit-exact (ties flagged);
ESS / lse within 1e-12 relative when both sides start from the same fp32 log-weights."""
import math

import numpy as np
import pytest
import torch

import synth
from gpu_util import max_abs, np_, to_host

pytestmark = pytest.mark.gpu

TOL_LOGW = 1e-4          # north star: log-weights within 1e-4 absolute
TOL_ELL = 2e-5           # per-row log-prob (fp32 kernel vs fp64 oracle)


@pytest.fixture(scope="module")
def smc():
    import paper_2604_15672_b200 as m          # raises if libsmcsd.so is missing (no fallback)
    assert torch.cuda.is_available()
    return m


def _run_weights(smc, orc, lp, lq, tok, V, **kw):
    dev = torch.device("cuda")
    g = dict(n_drafted=kw.get("n_drafted"), logw_prev=kw.get("logw_prev"))
    gpu = smc.smcsd_weights(lp.to(dev), lq.to(dev), tok.to(dev), V=V,
                            n_drafted=None if g["n_drafted"] is None else g["n_drafted"].to(dev),
                            logw_prev=None if g["logw_prev"] is None else g["logw_prev"].to(dev),
                            alpha=kw.get("alpha", 1.0), inv_temp_p=kw.get("tp", 1.0),
                            inv_temp_q=kw.get("tq", 1.0))
    torch.cuda.synchronize()
    ref = orc.weights(to_host(lp), to_host(lq), tok.numpy(), V=V, n_drafted=np_(g["n_drafted"]),
                      logw_prev=np_(g["logw_prev"]), alpha=kw.get("alpha", 1.0),
                      tau_p=kw.get("tp", 1.0), tau_q=kw.get("tq", 1.0))
    return gpu, ref


CASES = [
    # (P, N, K, V, dtype, sigma_d)       -- tiles: 8192-element segments; ragged tails
    (1, 4, 4, 1000, torch.float32, 0.5),          # cfg1 tiny
    (1, 16, 8, 128256, torch.bfloat16, 0.5),      # cfg2 (full size, every row checked)
    (3, 5, 3, 8192, torch.bfloat16, 0.5),         # exactly one segment
    (2, 3, 2, 8193, torch.float32, 1.5),          # one element into a second segment
    (2, 7, 5, 20001, torch.bfloat16, 1.5),        # odd V (bf16 vector straddles V)
    (1, 1, 1, 3, torch.float32, 0.5),             # V < one vector, N = 1, K = 1
    (2, 33, 2, 50000, torch.float32, 0.5),        # N not a multiple of 32
    (2, 3, 33, 1000, torch.float32, 0.5),         # K > 32: chunks split particles (S3 in last CTA)
    (1, 7, 7, 3000, torch.bfloat16, 0.5),         # K = 7: 28-pair chunks of whole particles
    (2, 40, 8, 20001, torch.bfloat16, 0.5),       # 10 chunk CTAs per prompt: a 10-CTA cluster
    (1, 64, 8, 30000, torch.bfloat16, 0.5),       # 16 chunk CTAs: the largest (non-portable) cluster
    (1, 65, 8, 9000, torch.float32, 0.5),         # 17 chunks: the per-prompt counter path
]


@pytest.mark.parametrize("P,N,K,V,dtype,sd", CASES)
def test_weights_parity(smc, orc, P, N, K, V, dtype, sd):
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=dtype, sigma_d=sd, seed=1000 + V + N)
    prev = synth.random_logw(P, N, seed=7, sigma=0.5)
    gpu, ref = _run_weights(smc, orc, lp, lq, tok, V, logw_prev=prev)
    assert np.array_equal(np_(gpu.status).astype(np.uint32), ref["status"])
    assert max_abs(np_(gpu.logp_tok), ref["logp_tok"]) <= TOL_ELL
    assert max_abs(np_(gpu.logq_tok), ref["logq_tok"]) <= TOL_ELL
    assert max_abs(np_(gpu.logw), ref["logw"]) <= TOL_LOGW
    assert np.allclose(np_(gpu.lse), ref["lse"], rtol=0, atol=TOL_LOGW)
    assert np.allclose(np_(gpu.ess), ref["ess"], rtol=1e-3)
    assert np.allclose(np_(gpu.wnorm), ref["wnorm"], rtol=1e-3, atol=1e-6)


def test_temperature_and_power(smc, orc):
    lp, lq, tok = synth.lm_logits(2, 8, 4, 30000, dtype=torch.bfloat16, seed=5, tau_q=0.7)
    gpu, ref = _run_weights(smc, orc, lp, lq, tok, 30000, alpha=2.5, tp=1.0 / 0.6, tq=0.7)
    assert max_abs(np_(gpu.logw), ref["logw"]) <= TOL_LOGW
    assert max_abs(np_(gpu.logp_tok), ref["logp_tok"]) <= TOL_ELL * 2


def test_identical_models_exact_zero(smc):
    # p == q bitwise, tau_p == tau_q, alpha = 1  =>  Delta == 0.0 exactly and ESS == N exactly
    # (requires the fixed in-row reduction order, reading G17)
    lp, _, tok = synth.lm_logits(2, 16, 8, 128256, dtype=torch.bfloat16, seed=3)
    dev = torch.device("cuda")
    lpd = lp.to(dev)
    lqd = lpd[:, :, :8, :].contiguous()
    prev = torch.full((2, 16), -math.log(16), device=dev)
    out = smc.smcsd_weights(lpd, lqd, tok.to(dev), V=128256, logw_prev=prev)
    assert torch.equal(out.logw, prev)
    assert torch.equal(out.logp_tok, out.logq_tok)
    assert torch.all(out.ess == 16.0)


def test_status_flags_match_oracle(smc, orc):
    lp, lq, tok = synth.lm_logits(4, 4, 3, 9000, dtype=torch.float32, seed=9)
    tok[0, 1, 0] = 9000                                   # BAD_TOKEN
    lq[1, 2, 1, tok[1, 2, 1]] = -float("inf")             # NOT_ABSCONT
    lp[2, 3, 0, 8500] = float("nan")                      # NONFINITE (second segment)
    lp[3, 0, 2, tok[3, 0, 2]] = -float("inf")             # p(d) = 0: allowed, weight -inf
    nd = torch.tensor([[3, 3, 3, 3], [3, 3, 3, 3], [3, 3, 3, 3], [3, 3, 3, 3]], dtype=torch.int32)
    gpu, ref = _run_weights(smc, orc, lp, lq, tok, 9000, n_drafted=nd)
    assert np_(gpu.status).astype(np.uint32).tolist() == ref["status"].tolist() == [4, 2, 8, 0]
    assert np.array_equal(np.isneginf(np_(gpu.logw)), np.isneginf(ref["logw"]))
    assert max_abs(np_(gpu.logw), ref["logw"]) <= TOL_LOGW
    # all particles dead -> DEGENERATE
    dead = torch.full((4, 4), -float("inf"))
    gpu, ref = _run_weights(smc, orc, lp, lq, tok, 9000, logw_prev=dead)
    assert np.array_equal(np_(gpu.status).astype(np.uint32), ref["status"])
    assert np.all(np_(gpu.lse) == -np.inf) and np.all(np_(gpu.ess) == 0.0)


def test_n_drafted_rows_never_read(smc, orc):
    lp, lq, tok = synth.lm_logits(2, 5, 4, 10000, dtype=torch.bfloat16, seed=12)
    nd = torch.tensor([[4, 0, 2, 1, 3], [4, 4, 4, 4, 4]], dtype=torch.int32)
    for p in range(2):
        for n in range(5):
            k = int(nd[p, n])
            lp[p, n, k:, :] = float("nan")
            lq[p, n, k:, :] = float("nan")
            tok[p, n, k:] = 10 ** 6
    gpu, ref = _run_weights(smc, orc, lp, lq, tok, 10000, n_drafted=nd)
    assert np.all(np_(gpu.status) == 0) and np.all(ref["status"] == 0)
    assert max_abs(np_(gpu.logw), ref["logw"]) <= TOL_LOGW
    assert np_(gpu.logw)[0, 1] == np.float32(-math.log(5))


def test_large_n_weights_path(smc, orc):
    # N > 1024 takes the serial-normalisation tail; ESS-rate fixture from SPEC.md:203
    N = 4000
    rng = np.random.default_rng(31)
    row_p = torch.tensor([math.log(0.5), math.log(0.5), float("nan"), float("nan")])
    row_q = torch.tensor([math.log(0.25), math.log(0.75), float("nan"), float("nan")])
    lp = row_p.expand(1, N, 3, 4).contiguous()
    lq = row_q.expand(1, N, 2, 4).contiguous()
    tok = torch.from_numpy((rng.random((1, N, 2)) < 0.75).astype(np.int32))
    gpu, ref = _run_weights(smc, orc, lp, lq, tok, 2, logw_prev=torch.zeros(1, N))
    assert max_abs(np_(gpu.logw), ref["logw"]) <= 1e-6
    assert np_(gpu.ess)[0] == pytest.approx(ref["ess"][0], rel=1e-6)
    assert np_(gpu.ess)[0] / N == pytest.approx(0.5625, abs=0.03)


# ----------------------------------------------------------------------------- resampling
def _resample_both(smc, orc, lw, **kw):
    dev = torch.device("cuda")
    un = kw.get("uniforms")
    scheme = kw.get("scheme", 0)
    gpu = smc.smcsd_resample(torch.from_numpy(lw).to(dev), eta=kw.get("eta", math.inf),
                             seed=kw.get("seed", synth.PHILOX_SEED), step=kw.get("step", 0),
                             prompt_base=kw.get("prompt_base", 0), scheme=scheme,
                             uniforms=None if un is None else torch.from_numpy(un.view(np.int32)).to(dev))
    torch.cuda.synchronize()
    ref = orc.resample(lw, eta=kw.get("eta", math.inf), seed=kw.get("seed", synth.PHILOX_SEED),
                       step=kw.get("step", 0), prompt_base=kw.get("prompt_base", 0), uniforms=un,
                       scheme=scheme)
    return gpu, ref


def _assert_resample_equal(gpu, ref):
    assert np.array_equal(np_(gpu.resampled), ref["resampled"])
    assert np.array_equal(np_(gpu.status).astype(np.uint32), ref["status"])
    assert np.array_equal(np_(gpu.n_ties), ref["n_ties"])
    ok = ref["n_ties"] == 0
    assert np.array_equal(np_(gpu.ancestors)[ok], ref["ancestors"][ok])
    assert np.array_equal(np_(gpu.offspring)[ok], ref["offspring"][ok])
    assert np.array_equal(np_(gpu.slot_src)[ok], ref["slot_src"][ok])
    assert np_(gpu.logw)[ok].tobytes() == ref["logw"][ok].tobytes()
    fin = np.isfinite(ref["lse"])
    assert np.allclose(np_(gpu.lse)[fin], ref["lse"][fin], rtol=1e-12, atol=0)
    assert np.allclose(np_(gpu.ess), ref["ess"], rtol=1e-12, atol=0)
    assert np.array_equal(np_(gpu.lse)[~fin], ref["lse"][~fin])


@pytest.mark.parametrize("N", [1, 2, 16, 32, 64, 100, 1024])
def test_resample_bit_exact(smc, orc, N):
    P = 64
    lw = synth.random_logw(P, N, seed=N, sigma=2.0, neg_inf_frac=0.2).numpy()
    lw[0, :] = -np.inf                                    # degenerate prompt
    lw[1, :] = 0.0                                        # uniform: ESS = N
    lw[2, :] = -np.inf; lw[2, N // 2] = 1.5               # single survivor
    if N > 3:
        lw[3, 3] = np.nan                                 # non-finite input -> flagged, -inf
    for step in (0, 1, (1 << 40) + 3):
        gpu, ref = _resample_both(smc, orc, lw, step=step, prompt_base=1000)
        _assert_resample_equal(gpu, ref)
    gpu, ref = _resample_both(smc, orc, lw, eta=N / 2)    # threshold path: some prompts kept
    _assert_resample_equal(gpu, ref)


def test_resample_worked_examples(smc, orc):
    from conftest import read_golden
    for line in read_golden("systematic_worked.txt"):
        w, x, anc, off = [s.strip() for s in line.split(";")]
        lw = np.log(np.array([float(v) for v in w.split(",")]))[None, :].astype(np.float32)
        gpu, ref = _resample_both(smc, orc, lw, uniforms=np.array([int(x)], np.uint32))
        assert np_(gpu.ancestors)[0].tolist() == [int(v) for v in anc.split(",")]
        assert np_(gpu.offspring)[0].tolist() == [int(v) for v in off.split(",")]


def _tie_flagged(u, C, delta=2.0 ** -40):
    """Particles n whose u_n lies within the tie radius of some C_m (reading G7)."""
    return np.array([np.any(np.abs(un - C) <= delta) for un in u])


def _assert_ties_equal(gpu_a, ref, u):
    """n_ties equal and > 0; ancestors equal except at flagged particles (reading G7)."""
    assert np.array_equal(np_(gpu_a.n_ties), ref["n_ties"])
    for p in range(ref["n_ties"].shape[0]):
        flag = _tie_flagged(u[p], ref["cdf"][p])
        assert int(flag.sum()) > 0 and int(ref["n_ties"][p]) > 0
        ga, ra = np_(gpu_a.ancestors)[p], ref["ancestors"][p]
        assert np.array_equal(ga[~flag], ra[~flag])
        # at a flagged particle the ancestor may move only across the boundaries within the tie
        # radius: #{m : C_m < u_n - delta} <= a_n <= #{m : C_m <= u_n + delta}
        C = ref["cdf"][p]
        for n in np.nonzero(flag)[0]:
            lo = int(np.sum(C < u[p][n] - 2.0 ** -40))
            hi = int(np.sum(C <= u[p][n] + 2.0 ** -40))
            assert lo <= int(ga[n]) <= hi, (p, n, int(ga[n]), lo, hi)


def test_forced_ties_resample_and_step(smc, orc):
    """Forced scan-boundary ties (tests/golden/systematic_ties.txt, derived by hand): the GPU
    reports the same n_ties > 0 as the oracle through smcsd_resample and through the fused
    smcsd_step (p == q bitwise gives Delta = 0 exactly, so lam' = lam_prev and C is exact)."""
    from conftest import read_golden
    dev = torch.device("cuda")
    rows = []
    for line in read_golden("systematic_ties.txt"):
        w, x, anc, off, ties = [s.strip() for s in line.split(";")]
        wts = np.array([float(v) for v in w.split(",")])
        if int(ties) == 0:
            continue
        with np.errstate(divide="ignore"):
            rows.append((np.log(wts).astype(np.float32), int(x), [int(v) for v in anc.split(",")],
                         int(ties)))
    for lw1, x, anc, ties in rows:
        N = lw1.size
        lw = lw1[None, :]
        un = np.array([x], np.uint32)
        gpu, ref = _resample_both(smc, orc, lw, uniforms=un)
        u = ((np.arange(N) + x / 2 ** 32) / N)[None, :]
        assert int(ref["n_ties"][0]) == ties
        _assert_ties_equal(gpu, ref, u)
        assert np_(gpu.ancestors)[0].tolist() == anc            # C is exact here: no slack used
        # fused step: p == q (bitwise), logw_prev = the same log-weights -> lam' == lam_prev
        V, K = 1000, 2
        lp, _, tok = synth.lm_logits(1, N, K, V, dtype=torch.float32, seed=5 + N)
        lq = lp[:, :, :K].contiguous()
        out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V,
                             logw_prev=torch.from_numpy(lw).to(dev), eta=math.inf,
                             uniforms=torch.from_numpy(un.view(np.int32)).to(dev))
        torch.cuda.synchronize()
        assert np_(out.logw_pre).tobytes() == lw.tobytes()
        ref_s = orc.resample(np_(out.logw_pre), eta=math.inf, uniforms=un)
        _assert_ties_equal(out, ref_s, u)
        assert np_(out.ancestors)[0].tolist() == anc
    # N = 1024 at the radius boundary (test_oracle_resample.py::test_tie_threshold_boundary)
    lw = np.zeros((2, 1024), np.float32)
    un = np.array([4, 5], np.uint32)
    gpu = smc.smcsd_resample(torch.from_numpy(lw).to(dev), eta=math.inf,
                             uniforms=torch.from_numpy(un.view(np.int32)).to(dev))
    torch.cuda.synchronize()
    assert np_(gpu.n_ties).tolist() == [1023, 0]
    # multinomial: same rule over i.i.d. u_n
    words = np.array([[0, 1 << 30, 1 << 31, 3 << 30]], np.uint32)
    gpu, ref = _resample_both(smc, orc, np.zeros((1, 4), np.float32), uniforms=words, scheme=1)
    assert int(np_(gpu.n_ties)[0]) == int(ref["n_ties"][0]) == 3
    assert np_(gpu.ancestors)[0].tolist() == ref["ancestors"][0].tolist() == [0, 1, 2, 3]


def test_default_eta_is_half_n_and_inputs_validated(smc, orc):
    """The binding's default threshold is ESS < N/2 (reading G2), and wrongly
    typed / shaped / placed inputs raise instead of being read as raw bytes (int64 tokens,
    non-contiguous views, CPU tensors)."""
    dev = torch.device("cuda")
    P, N = 8, 16
    lw = synth.random_logw(P, N, seed=4, sigma=1.5).numpy()
    lw[0] = 0.0                                              # ESS = N: kept under N/2
    lw[1] = -np.inf; lw[1, 3] = 0.0                          # ESS = 1: resampled
    gpu = smc.smcsd_resample(torch.from_numpy(lw).to(dev))
    torch.cuda.synchronize()
    ref = orc.resample(lw, eta=N / 2)
    assert np.array_equal(np_(gpu.resampled), ref["resampled"])
    assert np_(gpu.resampled)[0] == 0 and np_(gpu.resampled)[1] == 1
    assert np.array_equal(np_(gpu.ancestors), ref["ancestors"])
    lp, lq, tok = synth.lm_logits(1, 4, 2, 1000, dtype=torch.float32, seed=8)
    lpd, lqd = lp.to(dev), lq.to(dev)
    with pytest.raises(ValueError):
        smc.smcsd_step(lpd, lqd, tok.to(dev).long(), V=1000)         # int64 tokens
    with pytest.raises(ValueError):
        smc.smcsd_step(lpd, lqd, tok.to(dev), V=1000, logw_prev=torch.zeros(1, 8, device=dev)[:, ::2])
    with pytest.raises(ValueError):
        smc.smcsd_step(lpd, lqd, tok, V=1000)                        # tokens on the host
    with pytest.raises(ValueError):
        smc.smcsd_resample(torch.zeros(2, 4, dtype=torch.float64, device=dev))


def test_reset_value_table(smc):
    # fl32(-ln N), N = 1..1024, bitwise equal to the oracle's and Python's
    dev = torch.device("cuda")
    for N in range(1, 1025):
        out = smc.smcsd_resample(torch.zeros(1, N, device=dev), eta=math.inf)
        got = out.logw[0, 0].item()
        assert np.float32(got).tobytes() == np.float32(-math.log(N)).tobytes(), N


def test_systematic_unbiased_sweep(smc):
    # deterministic exactness: mean over a stratified U sweep of o_m equals N*wbar_m to 2/M
    dev = torch.device("cuda")
    N, M = 32, 4096
    lw = synth.random_logw(1, N, seed=77, sigma=1.5).to(dev).expand(M, N).contiguous()
    xs = ((np.arange(M) + 0.5) / M * 2 ** 32).astype(np.uint64).astype(np.uint32)
    out = smc.smcsd_resample(lw, eta=math.inf, uniforms=torch.from_numpy(xs.view(np.int32)).to(dev))
    mean = out.offspring.double().mean(0).cpu().numpy()
    wbar = out.wnorm[0].double().cpu().numpy()
    assert np.max(np.abs(mean - N * wbar)) <= 2.0 / M + 1e-6


@pytest.mark.parametrize("N,scheme,eta", [(32, 0, math.inf), (33, 0, math.inf), (48, 1, math.inf),
                                           (64, 0, math.inf), (64, 1, None), (65, 0, math.inf)])
def test_step_staged_parity(smc, orc, N, scheme, eta):
    # fused S1-S7: logw_pre feeds the oracle's S4-S7 -> bit-exact ancestry (staged protocol);
    # N <= 32 / <= 64 / > 64 are the three S4-S7 routines (warp_tail<1>, warp_tail<2>, one lane)
    P, K, V = 4, 8, 40000
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=21 + N)
    dev = torch.device("cuda")
    prev = synth.uniform_prior(P, N)
    prev[1, ::3] = -math.inf                                  # zero-weight particles
    eta_v = N / 2 if eta is None else eta
    out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V, logw_prev=prev.to(dev),
                         eta=eta, scheme=scheme, seed=123, step=9, prompt_base=40)
    torch.cuda.synchronize()
    ref_w = orc.weights(to_host(lp), to_host(lq), tok.numpy(), V=V, logw_prev=prev.numpy())
    assert max_abs(np_(out.logw_pre), ref_w["logw"]) <= TOL_LOGW
    staged = orc.resample(np_(out.logw_pre), eta=eta_v, scheme=scheme, seed=123, step=9, prompt_base=40)
    _assert_resample_equal(out, staged)
    # determinism: a second run is bitwise identical
    out2 = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V, logw_prev=prev.to(dev),
                          eta=eta, scheme=scheme, seed=123, step=9, prompt_base=40)
    for f in ("logw", "logw_pre", "ancestors", "slot_src", "ess", "lse", "logp_tok"):
        assert torch.equal(getattr(out, f), getattr(out2, f)), f


def test_step_end_to_end_vs_oracle(smc, orc):
    # soft protocol: oracle from the logits; ancestor mismatches only where |u - C| is within
    # the CDF disagreement (none expected at these sizes)
    P, N, K, V = 2, 16, 8, 128256
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=22)
    dev = torch.device("cuda")
    out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V, eta=math.inf, seed=5, step=1)
    torch.cuda.synchronize()
    ref_w = orc.weights(to_host(lp), to_host(lq), tok.numpy(), V=V)
    ref = orc.resample(ref_w["logw"], eta=math.inf, seed=5, step=1)
    assert max_abs(np_(out.logw_pre), ref_w["logw"]) <= TOL_LOGW
    assert np.allclose(np_(out.ess), ref["ess"], rtol=1e-3)
    assert np.array_equal(np_(out.ancestors), ref["ancestors"])


def test_n_equals_one(smc):
    # N = 1 reduces to plain proposal sampling: a = [0], ESS = 1
    lp, lq, tok = synth.lm_logits(3, 1, 4, 5000, dtype=torch.bfloat16, seed=2)
    dev = torch.device("cuda")
    out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=5000, eta=math.inf)
    assert torch.all(out.ancestors == 0) and torch.all(out.ess == 1.0)
    assert torch.all(out.logw == 0.0)


def test_dp_prompt_sharding_is_bit_identical(smc):
    # prompt-sharded (data-parallel) runs use the global prompt index for Philox
    P, N, K, V = 8, 32, 8, 30000
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=33)
    dev = torch.device("cuda")
    lp, lq, tok = lp.to(dev), lq.to(dev), tok.to(dev)
    full = smc.smcsd_step(lp, lq, tok, V=V, eta=math.inf, seed=99, step=4)
    for G in (2, 4, 8):
        per = P // G
        for g in range(G):
            sl = slice(g * per, (g + 1) * per)
            part = smc.smcsd_step(lp[sl].contiguous(), lq[sl].contiguous(), tok[sl].contiguous(),
                                  V=V, eta=math.inf, seed=99, step=4, prompt_base=g * per)
            for f in ("logw", "ancestors", "slot_src", "ess", "lse"):
                assert torch.equal(getattr(part, f), getattr(full, f)[sl]), (G, g, f)


# ----------------------------------------------------------------------------- TP (cfg5)
@pytest.mark.parametrize("G", [2, 4, 8])
def test_tp_vocab_sharded_simulated(smc, orc, G):
    # cfg5 shapes: V = 128256 split G-way, N = 64, K = 8; shards run one after another on
    # one GPU, gathered in rank order, combined (bit-identical on every rank by construction)
    P, N, K, V = 1, 64, 8, 128256
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=55)
    dev = torch.device("cuda")
    lpd, lqd, tokd = lp.to(dev), lq.to(dev), tok.to(dev)
    bounds = [V * g // G // 8 * 8 for g in range(G)] + [V]
    parts = []
    for g in range(G):
        b0, b1 = bounds[g], bounds[g + 1]
        w = (b1 - b0 + 7) // 8 * 8
        sp = torch.full((P, N, K + 1, w), float("nan"), dtype=torch.bfloat16, device=dev)
        sq = torch.full((P, N, K, w), float("nan"), dtype=torch.bfloat16, device=dev)
        sp[..., :b1 - b0] = lpd[..., b0:b1]
        sq[..., :b1 - b0] = lqd[..., b0:b1]
        parts.append(smc.smcsd_weights_partial(sp, sq, tokd, v_begin=b0, v_len=b1 - b0))
    gathered = torch.stack(parts).contiguous()
    c1 = smc.smcsd_weights_combine(gathered, tokd, V=V)
    c2 = smc.smcsd_weights_combine(gathered.clone(), tokd, V=V)
    assert torch.equal(c1.logw, c2.logw) and torch.equal(c1.ess, c2.ess)
    full = smc.smcsd_weights(lpd, lqd, tokd, V=V)
    assert (c1.logw - full.logw).abs().max().item() <= 1e-5
    ref = orc.weights(to_host(lp), to_host(lq), tok.numpy(), V=V)
    assert max_abs(np_(c1.logw), ref["logw"]) <= TOL_LOGW
    assert np.array_equal(np_(c1.status).astype(np.uint32), ref["status"])
    # S10 all-reduce form (north-star literal): MAX over ranks (emulated by a stack max),
    # smcsd_partials_rescale on every rank, SUM over ranks, combine with G = 1
    mx = gathered.amax(dim=0)
    resc = [smc.smcsd_partials_rescale(parts[g], mx) for g in range(G)]
    merged = resc[0].clone()
    merged[..., 1] = torch.stack([r[..., 1] for r in resc]).sum(dim=0)
    assert all(torch.equal(r[..., 0], mx[..., 0]) and torch.equal(r[..., 2], mx[..., 2]) for r in resc)
    c3 = smc.smcsd_weights_combine(merged.unsqueeze(0).contiguous(), tokd, V=V)
    assert (c3.logw - c1.logw).abs().max().item() <= 1e-5
    assert max_abs(np_(c3.logw), ref["logw"]) <= TOL_LOGW
    assert np.array_equal(np_(c3.status).astype(np.uint32), ref["status"])


# ----------------------------------------------------------------------------- KV (S8/S9)
def _kv_case(smc, orc, L, P, N, H, S, d, seq_len, in_place, seed):
    dev = torch.device("cuda")
    kv = synth.kv_bits((L, 2, P, N, H, S, d), seed=seed)
    lw = synth.random_logw(P, N, seed=seed, sigma=2.0).numpy()
    r = orc.resample(lw, eta=np.inf, seed=seed)
    idx = r["slot_src"] if in_place else r["ancestors"]
    geom = smc.kv_geometry(kv, seq_len)
    src = kv.to(dev)
    dst = src if in_place else torch.zeros_like(src)
    smc.smcsd_kv_reindex(dst, src, torch.from_numpy(idx).to(dev), **geom)
    torch.cuda.synchronize()
    want = kv.numpy().copy()
    want_dst = want if in_place else np.zeros_like(want)
    orc.kv_reindex(want_dst, want, idx, **geom)
    assert np.array_equal(dst.cpu().numpy(), want_dst)


@pytest.mark.parametrize("in_place", [False, True])
def test_kv_reindex_toy_cfg1(smc, orc, in_place):
    _kv_case(smc, orc, L=2, P=1, N=4, H=2, S=64, d=16, seq_len=64, in_place=in_place, seed=1)


@pytest.mark.parametrize("in_place", [False, True])
def test_kv_reindex_ragged(smc, orc, in_place):
    # several chunks, partial fill of each head, P > 1, N not a power of two
    _kv_case(smc, orc, L=3, P=3, N=37, H=4, S=256, d=64, seq_len=200, in_place=in_place, seed=2)
    _kv_case(smc, orc, L=1, P=2, N=1024, H=1, S=8, d=8, seq_len=8, in_place=in_place, seed=3)


@pytest.mark.parametrize("N", [1, 2, 31, 32, 33, 256, 257])
@pytest.mark.parametrize("in_place", [False, True])
def test_kv_reindex_kernel_boundaries(smc, orc, N, in_place):
    # the three K3 kernels' ranges (one-warp bulk copy N <= 32, 256-thread bulk copy N <= 256,
    # register path above), segments of 4 KB + a ragged part (seq_len < S: non-contiguous)
    _kv_case(smc, orc, L=2, P=2, N=N, H=3, S=48, d=64, seq_len=40, in_place=in_place, seed=50 + N)


def test_token_history_reindex(smc, orc):
    # S9: tok'[p][n][:] = tok[p][a_n][:], int32 rows through the same entry point
    dev = torch.device("cuda")
    P, N, T = 4, 16, 100
    tok = torch.randint(0, 128256, (P, N, T), dtype=torch.int32)
    lw = synth.random_logw(P, N, seed=4, sigma=2.0).numpy()
    r = orc.resample(lw, eta=np.inf, seed=4)
    geom = dict(n_outer=1, outer_stride=0, prompt_stride=N * T * 4, particle_stride=T * 4,
                seg_count=1, seg_bytes=T * 4, seg_stride=T * 4)
    src = tok.to(dev)
    dst = torch.zeros_like(src)
    smc.smcsd_kv_reindex(dst, src, torch.from_numpy(r["ancestors"]).to(dev), **geom)
    want = np.stack([tok.numpy()[p][r["ancestors"][p]] for p in range(P)])
    assert np.array_equal(dst.cpu().numpy(), want)


@pytest.mark.parametrize("in_place", [False, True])
def test_kv_reindex_invalid_index_status(smc, orc, in_place):
    """ST_BAD_INDEX (reading G23) against the oracle, bytes included: out-of-range entries are
    skipped; an in-place plan that overwrites one of its sources is skipped whole."""
    dev = torch.device("cuda")
    kv = synth.kv_bits((2, 2, 4, 6, 2, 16, 16), seed=3)
    a = np.array([[1, 6, 2, -1, 4, 5], [0, 0, 1, 1, 4, 5], [5, 1, 2, 3, 4, 5],
                  [0, 1, 2, 3, 4, 5]], np.int32)
    geom = smc.kv_geometry(kv)
    src = kv.to(dev)
    dst = src if in_place else torch.zeros_like(src)
    want = kv.numpy().copy() if in_place else np.zeros_like(kv.numpy())
    st_ref = orc.kv_reindex(want, want if in_place else kv.numpy().copy(), a, **geom)
    st = torch.full((4,), -1, dtype=torch.int32, device=dev)
    smc.smcsd_kv_reindex(dst, src, torch.from_numpy(a).to(dev), status=st, **geom)
    torch.cuda.synchronize()
    assert np_(st).astype(np.uint32).tolist() == st_ref.tolist()
    assert st_ref.tolist() == ([64, 64, 0, 0] if in_place else [64, 0, 0, 0])
    assert np.array_equal(dst.cpu().numpy(), want)


def test_kv_reindex_multi_per_layer_tensors(smc, orc):
    """smcsd_kv_reindex_multi: per-layer K and V tensors (separate allocations, a serving
    engine's layout) + the token history in ONE launch, in place and out of place, against
    the oracle's gather of the equivalent single tensor."""
    dev = torch.device("cuda")
    L, P, N, H, S, d, T = 3, 2, 13, 2, 96, 32, 52          # token rows: 208 B (16-B multiple)
    kv = synth.kv_bits((L, 2, P, N, H, S, d), seed=21)
    tok = torch.randint(0, 128256, (P, N, T), dtype=torch.int32)
    lw = synth.random_logw(P, N, seed=21, sigma=2.0).numpy()
    r = orc.resample(lw, eta=np.inf, seed=21)
    for in_place in (True, False):
        idx = r["slot_src"] if in_place else r["ancestors"]
        layers = [kv[l, c].contiguous().to(dev) for l in range(L) for c in range(2)]  # [P][N][H][S][d]
        outs = layers if in_place else [torch.zeros_like(t) for t in layers]
        tsrc = tok.to(dev)
        tdst = tsrc if in_place else torch.zeros_like(tsrc)
        e = kv.element_size()
        g = dict(n_outer=1, outer_stride=0, prompt_stride=N * H * S * d * e, particle_stride=H * S * d * e,
                 seg_count=H, seg_bytes=70 * d * e, seg_stride=S * d * e)        # filled rows [0, 70)
        gt = dict(n_outer=1, outer_stride=0, prompt_stride=N * T * 4, particle_stride=T * 4,
                  seg_count=1, seg_bytes=T * 4, seg_stride=T * 4)
        ents = [smc.kv_tensor(o, i, **g) for o, i in zip(outs, layers)] + [smc.kv_tensor(tdst, tsrc, **gt)]
        smc.smcsd_kv_reindex_multi(ents, torch.from_numpy(idx).to(dev))
        torch.cuda.synchronize()
        want = kv.numpy().copy()
        want_dst = want if in_place else np.zeros_like(want)
        orc.kv_reindex(want_dst, want, idx, **smc.kv_geometry(kv, 70))
        got = np.stack([outs[2 * l + c].cpu().numpy() for l in range(L) for c in range(2)]).reshape(want.shape)
        assert np.array_equal(got, want_dst)
        want_t = np.stack([tok.numpy()[p][idx[p]] if not in_place else tok.numpy()[p][idx[p]] for p in range(P)])
        assert np.array_equal(tdst.cpu().numpy(), want_t)


def test_kv_identity_is_noop(smc):
    dev = torch.device("cuda")
    kv = synth.kv_bits((2, 2, 1, 8, 2, 32, 16), seed=5).to(dev)
    before = kv.clone()
    smc.smcsd_kv_reindex(kv, kv, torch.arange(8, dtype=torch.int32, device=dev)[None],
                         **smc.kv_geometry(kv))
    assert torch.equal(kv, before)


# ----------------------------------------------------------------------- NEXT #3: multinomial
@pytest.mark.parametrize("N", [1, 3, 16, 33, 64, 1024])
def test_multinomial_resample_bit_exact(smc, orc, N):
    P = 48
    lw = synth.random_logw(P, N, seed=500 + N, sigma=2.0, neg_inf_frac=0.2).numpy()
    lw[0, :] = -np.inf
    lw[1, :] = 0.0
    for step in (0, 7, (1 << 35) + 1):
        gpu, ref = _resample_both(smc, orc, lw, step=step, prompt_base=77, scheme=1)
        _assert_resample_equal(gpu, ref)
    words = np.random.default_rng(N).integers(0, 2 ** 32, size=(P, N), dtype=np.uint64).astype(np.uint32)
    gpu, ref = _resample_both(smc, orc, lw, uniforms=words, scheme=1)
    _assert_resample_equal(gpu, ref)


def test_step_multinomial_staged(smc, orc):
    P, N, K, V = 3, 32, 8, 20000
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=61)
    dev = torch.device("cuda")
    out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V, eta=math.inf, seed=3, step=4,
                         scheme=smc.SMCSD_MULTINOMIAL)
    torch.cuda.synchronize()
    staged = orc.resample(np_(out.logw_pre), eta=math.inf, seed=3, step=4, scheme=1)
    _assert_resample_equal(out, staged)


def test_terminal_selection(smc, orc):
    dev = torch.device("cuda")
    P, N = 500, 37
    lw = synth.random_logw(P, N, seed=8, sigma=2.0, neg_inf_frac=0.3).numpy()
    lw[3, :] = -np.inf
    sel, st = smc.smcsd_select(torch.from_numpy(lw).to(dev), seed=11, step=2, prompt_base=5)
    ref = orc.select(lw, seed=11, step=2, prompt_base=5)
    assert np.array_equal(np_(sel), ref["selected"])
    assert np.array_equal(np_(st).astype(np.uint32), ref["status"])
    words = np.random.default_rng(3).integers(0, 2 ** 32, size=P, dtype=np.uint64).astype(np.uint32)
    sel, _ = smc.smcsd_select(torch.from_numpy(lw).to(dev), uniforms=torch.from_numpy(words.view(np.int32)).to(dev))
    assert np.array_equal(np_(sel), orc.select(lw, uniforms=words)["selected"])


# ----------------------------------------------------------------------- NEXT #1: paged KV
def test_paged_reindex_bit_exact(smc, orc):
    import test_oracle_kv_tp as kvt
    dev = torch.device("cuda")
    rng = np.random.default_rng(3)
    for trial in range(6):
        P, N = int(rng.integers(1, 5)), int(rng.integers(1, 70))
        table, n_pages, rc = kvt._paged_fixture(P, N, 130, seed=trial)     # seq 2048 / page 16
        lw = (rng.standard_normal((P, N)) * 2).astype(np.float32)
        a = orc.resample(lw, eta=np.inf, seed=trial)["ancestors"]
        ref = orc.kv_reindex_paged(table, n_pages, rc, a)
        rcd = torch.from_numpy(rc).to(dev)
        freed = torch.zeros(rc.size, dtype=torch.uint8, device=dev)
        td, nd, st = smc.smcsd_kv_reindex_paged(torch.from_numpy(table).to(dev),
                                                torch.from_numpy(n_pages).to(dev), rcd,
                                                torch.from_numpy(a).to(dev), freed=freed)
        torch.cuda.synchronize()
        assert np.array_equal(np_(td), ref["table"])
        assert np.array_equal(np_(nd), ref["n_pages"])
        assert np.array_equal(np_(rcd), ref["refcount"])
        touched = np.zeros(rc.size, bool)
        for p in range(P):
            for n in range(N):
                touched[table[p, n, :n_pages[p, n]]] = True
        assert np.array_equal(np_(freed)[touched], ref["freed"][touched])
        assert np.all(np_(st) == 0)


# ------------------------------------------------------------- PowerSMC weights (NEXT #4)
def _power_both(smc, orc, lg, V, alpha, tau=1.0, prev=None):
    dev = torch.device("cuda")
    gpu = smc.smcsd_powersmc_weights(lg.to(dev), V=V, alpha=alpha, inv_temp=tau,
                                     logw_prev=None if prev is None else prev.to(dev))
    torch.cuda.synchronize()
    ref = orc.powersmc_weights(to_host(lg), V=V, alpha=alpha, tau=tau, logw_prev=np_(prev))
    return gpu, ref


# integer alpha (repeated products), half-integer alpha (one ex2 of t/2: 0.5 .. 3.5) and a
# general alpha (second exp): every K1 power variant
@pytest.mark.parametrize("alpha", [0.5, 1.5, 2.0, 2.5, 2.7, 3.0, 3.5, 4.0])
@pytest.mark.parametrize("P,N,V,dtype", [(1, 16, 128256, torch.bfloat16), (2, 33, 20001, torch.float32),
                                         (3, 5, 8193, torch.bfloat16), (1, 1, 3, torch.float32),
                                         (1, 8, 140001, torch.bfloat16)])   # 18 segments: 2 chunks
def test_powersmc_weights_parity(smc, orc, P, N, V, dtype, alpha):
    lg, _, _ = synth.lm_logits(P, N, 1, V, dtype=dtype, seed=4000 + V + N, bonus=False)
    prev = synth.random_logw(P, N, seed=8, sigma=0.5)
    gpu, ref = _power_both(smc, orc, lg, V, alpha, tau=1.0 / 0.8, prev=prev)
    assert np.array_equal(np_(gpu.status).astype(np.uint32), ref["status"])
    assert max_abs(np_(gpu.logp_tok), ref["inc"]) <= TOL_LOGW
    assert max_abs(np_(gpu.logw), ref["logw"]) <= TOL_LOGW
    assert np.allclose(np_(gpu.lse), ref["lse"], rtol=0, atol=TOL_LOGW)
    assert np.allclose(np_(gpu.ess), ref["ess"], rtol=1e-3)
    assert np.allclose(np_(gpu.wnorm), ref["wnorm"], rtol=1e-3, atol=1e-6)


def test_powersmc_alpha_one_is_exact_zero(smc):
    # alpha = 1: S2 and S1 are the same fp32 sum, so log w = ln2 (log2 S - log2 S) = 0 exactly
    lg, _, _ = synth.lm_logits(2, 16, 1, 128256, dtype=torch.bfloat16, seed=3, bonus=False)
    dev = torch.device("cuda")
    prev = torch.full((2, 16), -math.log(16), device=dev)
    out = smc.smcsd_powersmc_weights(lg.to(dev), V=128256, alpha=1.0, logw_prev=prev)
    assert torch.all(out.logp_tok == 0.0)
    assert torch.equal(out.logw, prev)
    assert torch.all(out.ess == 16.0)


@pytest.mark.parametrize("alpha", [2.0, 2.5, 2.7])
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_powersmc_status_and_masked_rows(smc, orc, alpha, dtype):
    lg, _, _ = synth.lm_logits(3, 4, 1, 9000, dtype=dtype, seed=21, bonus=False)
    lg[0, 2, 0, 8700] = float("nan")                   # NONFINITE, particle dead
    lg[1, :, 0, :] = -float("inf")                     # every row masked -> all dead, DEGENERATE
    lg[2, 1, 0, :8000] = -float("inf")                 # partially masked row: fine
    gpu, ref = _power_both(smc, orc, lg, 9000, alpha)
    assert np_(gpu.status).astype(np.uint32).tolist() == ref["status"].tolist()
    assert ref["status"].tolist() == [8, 9, 0]
    assert np.array_equal(np.isneginf(np_(gpu.logw)), np.isneginf(ref["logw"]))
    assert max_abs(np_(gpu.logw), ref["logw"]) <= TOL_LOGW


# ------------------------------------------------------------- bonus token (NEXT #2)
SEG_MARGIN_TOL = 1e-5      # |C_i/W - U| below this: segment choice is a rounding-order near-tie
KEY_MARGIN_TOL = 1e-4      # top-2 Gumbel keys (natural units) closer than this: near-tie
BONUS_SEG = 8192           # reading G22's segment width as the product path uses it


def _bonus_check(gpu_b, ref):
    """Draw-for-draw parity except at rounding-order near-ties, and there the GPU's draw must be
    one of the near-tied candidates the oracle names: at a segment near-tie the draw of the
    segment across the nearest CDF boundary (ref['alt']), at a key near-tie the runner-up column
    of the chosen segment (ref['second'])."""
    seg_tie = ref["seg_margin"] <= SEG_MARGIN_TOL
    key_tie = ref["key_margin"] <= KEY_MARGIN_TOL
    ok = ~seg_tie & ~key_tie
    assert ok.mean() > 0.9
    assert np.array_equal(gpu_b[ok], ref["bonus"][ok])
    for idx in zip(*np.nonzero(~ok)):
        g = gpu_b[idx]
        allowed = {int(ref["bonus"][idx])}
        if seg_tie[idx]:
            allowed.add(int(ref["alt"][idx]))
        if key_tie[idx]:
            allowed.add(int(ref["second"][idx]))
        allowed.discard(-1)
        assert int(g) in allowed, (idx, int(g), allowed)
    return ok


@pytest.mark.parametrize("P,N,K,V,dtype", [(1, 16, 8, 128256, torch.bfloat16),   # cfg2
                                           (2, 33, 3, 20001, torch.float32),     # ragged
                                           (3, 5, 2, 8192, torch.bfloat16),      # one segment
                                           (2, 4, 1, 7, torch.float32)])         # V < vector
def test_bonus_token_parity(smc, orc, P, N, K, V, dtype):
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=dtype, seed=6000 + V + N)
    dev = torch.device("cuda")
    kw = dict(V=V, eta=math.inf, seed=77, step=5, prompt_base=3, inv_temp_p=1.0 / 0.7)
    out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), bonus=True, **kw)
    plain = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), **kw)
    torch.cuda.synchronize()
    ref = orc.bonus(to_host(lp), K=K, V=V, tau=1.0 / 0.7, seed=77, step=5, prompt_base=3,
                    seg=BONUS_SEG)
    _bonus_check(np_(out.bonus), ref)
    assert np.all(np_(out.status) == 0) and np.all(ref["status"] == 0)
    # the bonus row never enters the weights or the resampling
    assert torch.equal(out.logw_pre, plain.logw_pre) and torch.equal(out.ancestors, plain.ancestors)


def test_bonus_token_n_drafted_and_flags(smc, orc):
    P, N, K, V = 2, 6, 4, 9000
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.float32, seed=61)
    nd = torch.tensor([[0, 1, 2, 3, 4, 4], [4, 4, 4, 4, 4, 4]], dtype=torch.int32)
    lp[1, 2, K, 4000] = float("nan")                       # bonus row NaN -> -1, NONFINITE
    lp[1, 4, K, :] = -float("inf")                         # all -inf bonus row -> -1, NONFINITE
    dev = torch.device("cuda")
    out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V, n_drafted=nd.to(dev),
                         eta=math.inf, step=2, bonus=True)
    torch.cuda.synchronize()
    ref = orc.bonus(to_host(lp), K=K, V=V, n_drafted=nd.numpy(), step=2, seg=BONUS_SEG)
    _bonus_check(np_(out.bonus), ref)
    assert np_(out.bonus)[1, 2] == -1 and np_(out.bonus)[1, 4] == -1
    assert int(np_(out.status)[1]) & 8


def test_bonus_token_frequencies(smc):
    # 8 hot columns over 3 segments (ragged tail): GPU draws follow the softmax (chi-square)
    from scipy import stats
    V, N = 3 * 8192 + 100, 1024
    hot = torch.tensor([5, 4000, 8191, 8192, 12000, 16383, 20000, 3 * 8192 + 99])
    z = torch.tensor([1.0, 0.3, -0.5, 0.8, 0.0, 1.2, -1.0, 0.6])
    lp = torch.full((1, N, 2, V + 4), -float("inf"))
    lp[:, :, :, hot] = z
    lq = lp[:, :, :1].contiguous()
    tok = torch.full((1, N, 1), 5, dtype=torch.int32)
    dev = torch.device("cuda")
    lpd, lqd, tokd = lp.to(dev), lq.to(dev), tok.to(dev)
    draws = []
    for s in range(16):
        draws.append(np_(smc.smcsd_step(lpd, lqd, tokd, V=V, step=s, bonus=True).bonus).ravel())
    b = np.concatenate(draws)
    cnt = np.array([(b == h).sum() for h in hot.tolist()])
    assert cnt.sum() == b.size
    p = np.exp(z.double().numpy()); p /= p.sum()
    chi2 = ((cnt - p * b.size) ** 2 / (p * b.size)).sum()
    assert stats.chi2.sf(chi2, len(hot) - 1) > 1e-3


# ------------------------------------------- TP with S10 fused into K1 over peer memory
def _shard(x, b0, b1, align, dev):
    w = (b1 - b0 + align - 1) // align * align
    s = torch.full(x.shape[:-1] + (w,), float("nan"), dtype=x.dtype, device=dev)
    s[..., :b1 - b0] = x[..., b0:b1]
    return s


@pytest.mark.parametrize("G,P,N,K,V,dtype", [(1, 1, 64, 8, 128256, torch.bfloat16),
                                             (2, 2, 8, 3, 50001, torch.float32),
                                             (4, 1, 64, 8, 128256, torch.bfloat16),
                                             (8, 1, 64, 8, 128256, torch.bfloat16)])
def test_tp_step_fused_exchange(smc, orc, G, P, N, K, V, dtype):
    # G simulated ranks on one GPU, each on its own stream: K1 of every rank pushes its
    # segment partials into every rank's exchange buffer and publishes the epoch; every
    # rank's tail waits on its flags and merges in rank order.  Two steps (both parity halves).
    from paper_2604_15672_b200.dist import TPExchange
    dev = torch.device("cuda")
    align = 8 if dtype == torch.bfloat16 else 4
    ex = TPExchange.local_group(P, N, K, V, G, device=dev)
    streams = [torch.cuda.Stream(dev) for _ in range(G)]
    for it in range(2):
        lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=dtype, seed=900 + 7 * G + it)
        prev = synth.random_logw(P, N, seed=11 + it, sigma=0.5)
        lpd, lqd, tokd, prevd = lp.to(dev), lq.to(dev), tok.to(dev), prev.to(dev)
        shards = [(_shard(lpd, e.v_begin, e.v_begin + e.v_len, align, dev),
                   _shard(lqd, e.v_begin, e.v_begin + e.v_len, align, dev)) for e in ex]
        torch.cuda.synchronize()
        outs = []
        for g, e in enumerate(ex):
            with torch.cuda.stream(streams[g]):
                outs.append(e.step(*shards[g], tokd, logw_prev=prevd, eta=math.inf, seed=3,
                                   step=it, workspace=smc.Workspace(dev), stream=streams[g]))
        torch.cuda.synchronize()
        for o in outs:
            assert np.all(np_(o.status) == 0)
            for f in ("logw_pre", "logw", "ancestors", "slot_src", "ess", "lse"):
                assert torch.equal(getattr(o, f), getattr(outs[0], f)), f
        ref = orc.weights(to_host(lp), to_host(lq), tok.numpy(), V=V, logw_prev=prev.numpy())
        assert max_abs(np_(outs[0].logw_pre), ref["logw"]) <= TOL_LOGW
        assert max_abs(np_(outs[0].logp_tok), ref["logp_tok"]) <= TOL_ELL
        rr = orc.resample(np_(outs[0].logw_pre), eta=np.inf, seed=3, step=it)
        assert np.array_equal(np_(outs[0].ancestors), rr["ancestors"])
        assert np.array_equal(np_(outs[0].logw), rr["logw"])


def _tp_check(outs, lp, lq, tok, prev, V, step, orc):
    for o in outs:
        assert np.all(np_(o.status) == 0)
        for f in ("logw_pre", "logw", "ancestors", "slot_src", "ess", "lse"):
            assert torch.equal(getattr(o, f), getattr(outs[0], f)), f
    ref = orc.weights(to_host(lp), to_host(lq), tok.numpy(), V=V, logw_prev=prev.numpy())
    assert max_abs(np_(outs[0].logw_pre), ref["logw"]) <= TOL_LOGW
    rr = orc.resample(np_(outs[0].logw_pre), eta=np.inf, seed=3, step=step)
    assert np.array_equal(np_(outs[0].ancestors), rr["ancestors"])


def test_tp_step_explicit_epoch(smc, orc):
    # the host-epoch mode of smcsd_tp_step (epoch >= 1 per call), three steps (both halves)
    from paper_2604_15672_b200.dist import TPExchange
    dev = torch.device("cuda")
    P, N, K, V, G = 1, 16, 4, 30001, 2
    ex = TPExchange.local_group(P, N, K, V, G, device=dev, device_epoch=False)
    streams = [torch.cuda.Stream(dev) for _ in range(G)]
    for it in range(3):
        lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=950 + it)
        prev = synth.random_logw(P, N, seed=21 + it, sigma=0.5)
        lpd, lqd, tokd, prevd = lp.to(dev), lq.to(dev), tok.to(dev), prev.to(dev)
        shards = [(_shard(lpd, e.v_begin, e.v_begin + e.v_len, 8, dev),
                   _shard(lqd, e.v_begin, e.v_begin + e.v_len, 8, dev)) for e in ex]
        torch.cuda.synchronize()
        outs = []
        for g, e in enumerate(ex):
            with torch.cuda.stream(streams[g]):
                outs.append(e.step(*shards[g], tokd, logw_prev=prevd, eta=math.inf, seed=3,
                                   step=it, workspace=smc.Workspace(dev), stream=streams[g]))
        torch.cuda.synchronize()
        assert ex[0].epoch == it + 1
        _tp_check(outs, lp, lq, tok, prev, V, it, orc)


@pytest.mark.parametrize("G", [1, 2])
def test_tp_step_graph_replay(smc, orc, G):
    # the device-resident epoch makes smcsd_tp_step capturable: each rank's step is captured
    # once into a CUDA graph on its own stream, then replayed for new inputs (copied into the
    # captured buffers); every replay is the next epoch, so flags and parity halves advance
    from paper_2604_15672_b200.dist import TPExchange
    dev = torch.device("cuda")
    P, N, K, V = 1, 32, 8, 128256
    ex = TPExchange.local_group(P, N, K, V, G, device=dev)
    streams = [torch.cuda.Stream(dev) for _ in range(G)]
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=970)
    prev = synth.random_logw(P, N, seed=31, sigma=0.5)
    tokd, prevd = tok.to(dev), prev.to(dev)
    shards = [(_shard(lp.to(dev), e.v_begin, e.v_begin + e.v_len, 8, dev),
               _shard(lq.to(dev), e.v_begin, e.v_begin + e.v_len, 8, dev)) for e in ex]
    outs = [smc.Outputs() for _ in range(G)]
    wss = [smc.Workspace(dev) for _ in range(G)]

    def run_all(step):
        for g, e in enumerate(ex):
            with torch.cuda.stream(streams[g]):
                e.step(*shards[g], tokd, logw_prev=prevd, eta=math.inf, seed=3, step=step,
                       out=outs[g], workspace=wss[g], stream=streams[g])

    for s_ in streams:
        s_.wait_stream(torch.cuda.current_stream())
    run_all(0)                                   # eager warm-up: outputs allocated, epoch 1
    torch.cuda.synchronize()
    _tp_check(outs, lp, lq, tok, prev, V, 0, orc)
    graphs = [torch.cuda.CUDAGraph() for _ in range(G)]
    for g, e in enumerate(ex):
        with torch.cuda.graph(graphs[g], stream=streams[g]):
            e.step(*shards[g], tokd, logw_prev=prevd, eta=math.inf, seed=3, step=7,
                   out=outs[g], workspace=wss[g], stream=streams[g])
    torch.cuda.synchronize()
    for it in range(3):                          # epochs 2, 3, 4: both parity halves
        lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=971 + it)
        prev = synth.random_logw(P, N, seed=32 + it, sigma=0.5)
        tokd.copy_(tok.to(dev))
        prevd.copy_(prev.to(dev))
        for g, e in enumerate(ex):
            a, b = _shard(lp.to(dev), e.v_begin, e.v_begin + e.v_len, 8, dev), \
                _shard(lq.to(dev), e.v_begin, e.v_begin + e.v_len, 8, dev)
            shards[g][0].copy_(a)
            shards[g][1].copy_(b)
        torch.cuda.synchronize()
        for g in range(G):
            with torch.cuda.stream(streams[g]):
                graphs[g].replay()
        torch.cuda.synchronize()
        _tp_check(outs, lp, lq, tok, prev, V, 7, orc)


def test_tp_step_many_epochs(smc, orc):
    # 600 graph replays of a G = 2 fused step (both ranks concurrently on their own streams):
    # epochs and parity halves advance on the device every replay; no rank ever times out and
    # the ranks stay bit-identical and equal to the oracle
    from paper_2604_15672_b200.dist import TPExchange
    dev = torch.device("cuda")
    P, N, K, V, G = 1, 16, 4, 30001, 2
    ex = TPExchange.local_group(P, N, K, V, G, device=dev)
    streams = [torch.cuda.Stream(dev) for _ in range(G)]
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=990)
    prev = synth.random_logw(P, N, seed=41, sigma=0.5)
    tokd, prevd = tok.to(dev), prev.to(dev)
    shards = [(_shard(lp.to(dev), e.v_begin, e.v_begin + e.v_len, 8, dev),
               _shard(lq.to(dev), e.v_begin, e.v_begin + e.v_len, 8, dev)) for e in ex]
    outs = [smc.Outputs() for _ in range(G)]
    wss = [smc.Workspace(dev) for _ in range(G)]
    for s_ in streams:
        s_.wait_stream(torch.cuda.current_stream())
    for g, e in enumerate(ex):                   # eager first step: outputs allocated
        with torch.cuda.stream(streams[g]):
            e.step(*shards[g], tokd, logw_prev=prevd, eta=math.inf, seed=3, step=5,
                   out=outs[g], workspace=wss[g], stream=streams[g])
    torch.cuda.synchronize()
    graphs = [torch.cuda.CUDAGraph() for _ in range(G)]
    for g, e in enumerate(ex):
        with torch.cuda.graph(graphs[g], stream=streams[g]):
            for _ in range(10):
                e.step(*shards[g], tokd, logw_prev=prevd, eta=math.inf, seed=3, step=5,
                       out=outs[g], workspace=wss[g], stream=streams[g])
    torch.cuda.synchronize()
    for _ in range(60):
        for g in range(G):
            with torch.cuda.stream(streams[g]):
                graphs[g].replay()
    torch.cuda.synchronize()
    word = [int(e.buf[48 * 4:49 * 4].view(torch.int32).item()) for e in ex]
    assert word == [601, 601]                    # device epoch: 1 eager + 600 replayed steps
    _tp_check(outs, lp, lq, tok, prev, V, 5, orc)


def test_extreme_and_masked_rows(smc, orc):
    # SURVEY 8(d) edge rows: +-60 extremes and -inf-masked tails (vocabulary masking), both
    # dtypes; the drafted token always keeps finite target and draft mass
    for dtype in (torch.float32, torch.bfloat16):
        P, N, K, V = 2, 8, 4, 20000
        lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=dtype, seed=4242)
        g = torch.Generator().manual_seed(5)
        ext = torch.rand(lp.shape[:-1] + (V,), generator=g) < 0.002
        sign = torch.where(torch.rand(ext.shape, generator=g) < 0.5, -60.0, 60.0).to(dtype)
        lp[..., :V] = torch.where(ext, sign, lp[..., :V])
        lq[..., :V] = torch.where(ext[:, :, :K], sign[:, :, :K], lq[..., :V])
        lp[0, :, :, 15000:V] = -float("inf")                # masked tail (prompt 0)
        lq[0, :, :, 15000:V] = -float("inf")
        tok[0] = tok[0] % 15000                             # drafted tokens stay unmasked
        gpu, ref = _run_weights(smc, orc, lp, lq, tok, V)
        assert np.array_equal(np_(gpu.status).astype(np.uint32), ref["status"])
        assert max_abs(np_(gpu.logp_tok), ref["logp_tok"]) <= TOL_ELL * 4
        assert max_abs(np_(gpu.logw), ref["logw"]) <= TOL_LOGW


def test_step_plan_matches_step(smc):
    """smc.StepPlan (prepared argument list) gives exactly smcsd_step's outputs, input swaps
    included, and rejects inputs of another shape."""
    dev = torch.device("cuda")
    sets = [synth.lm_logits(2, 8, 4, 20001, dtype=torch.bfloat16, seed=900 + r) for r in range(2)]
    sets = [tuple(t.to(dev) for t in s_) for s_ in sets]
    ws = smc.Workspace(dev)
    plan = smc.StepPlan(*sets[0], V=20001, out=smc.Outputs(), workspace=ws, bonus=True)
    for i in range(4):
        got = plan.run(*sets[i % 2], step=i)
        torch.cuda.synchronize()
        ref = smc.smcsd_step(*sets[i % 2], V=20001, step=i, bonus=True)
        torch.cuda.synchronize()
        for f in ("logw", "logw_pre", "ancestors", "slot_src", "ess", "bonus", "status"):
            assert torch.equal(getattr(got, f), getattr(ref, f)), (i, f)
    bad = synth.lm_logits(2, 8, 4, 20050, dtype=torch.bfloat16, seed=1)      # another row pitch
    with pytest.raises(ValueError):
        plan.run(*(t.to(dev) for t in bad), step=9)


# ------------------------------------------------------------- limits the ABI accepts
@pytest.mark.parametrize("P,N,K,V,dtype", [(2, 1024, 2, 3000, torch.float32),    # N at kTailMaxN
                                           (2, 8, 64, 5000, torch.bfloat16),     # K = 64 (paper max)
                                           (1, 100, 8, 20001, torch.bfloat16)])  # N between 64 and 1024
def test_step_at_abi_limits(smc, orc, P, N, K, V, dtype):
    dev = torch.device("cuda")
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=dtype, sigma_d=0.5, seed=700 + N + K)
    prev = synth.random_logw(P, N, seed=13, sigma=0.5)
    g = torch.Generator().manual_seed(3)
    ndr = torch.randint(0, K + 1, (P, N), generator=g, dtype=torch.int32)
    out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V, n_drafted=ndr.to(dev),
                         logw_prev=prev.to(dev), eta=math.inf, step=4, seed=synth.PHILOX_SEED)
    torch.cuda.synchronize()
    ref = orc.weights(to_host(lp), to_host(lq), tok.numpy(), V=V, n_drafted=ndr.numpy(),
                      logw_prev=prev.numpy())
    assert max_abs(np_(out.logw_pre), ref["logw"]) <= TOL_LOGW
    assert np.array_equal(np_(out.status).astype(np.uint32), ref["status"])
    rr = orc.resample(np_(out.logw_pre), eta=np.inf, seed=synth.PHILOX_SEED, step=4)
    assert rr["n_ties"].sum() == 0
    assert np.array_equal(np_(out.ancestors), rr["ancestors"])
    assert np.array_equal(np_(out.slot_src), rr["slot_src"])
    assert np.array_equal(np_(out.offspring), rr["offspring"])


def test_bonus_at_max_vocab(smc, orc):
    """Bonus token at V = 2^21 (256 segments: the sampler's shared-memory limit)."""
    dev = torch.device("cuda")
    P, N, K, V = 1, 4, 2, 1 << 21
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=71)
    out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V, step=1, bonus=True)
    torch.cuda.synchronize()
    assert int(out.status.abs().sum()) == 0
    ref = orc.bonus(to_host(lp), K=K, V=V, step=1, seg=BONUS_SEG)
    _bonus_check(np_(out.bonus), ref)
    w = orc.weights(to_host(lp), to_host(lq), tok.numpy(), V=V)
    assert max_abs(np_(out.logw_pre), w["logw"]) <= TOL_LOGW
