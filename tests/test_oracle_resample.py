"""Pins for the oracle's S5-S7 (resample test, systematic ancestors, slot plan, reset).

Pins: worked examples (tests/golden/systematic_worked.txt), the closed form of systematic
offspring counts o_m = ceil(N C_m - U) - ceil(N C_{m-1} - U), floor/ceil bounds, exact
unbiasedness over a stratified sweep of U (integral of ceil(x - U) dU = x), special cases
(SPEC.md:193, 210, 254), and the -ln N reset table.
"""
import math

import numpy as np
import pytest

from conftest import read_golden


def _logw(weights):
    with np.errstate(divide="ignore"):
        return np.log(np.asarray(weights, dtype=np.float64)).astype(np.float32)[None, :]


def test_worked_examples(orc):
    for line in read_golden("systematic_worked.txt"):
        w, x, anc, off = [s.strip() for s in line.split(";")]
        out = orc.resample(_logw([float(v) for v in w.split(",")]), eta=np.inf,
                           uniforms=np.array([int(x)], np.uint32))
        assert out["resampled"][0] == 1
        assert out["ancestors"][0].tolist() == [int(v) for v in anc.split(",")], line
        assert out["offspring"][0].tolist() == [int(v) for v in off.split(",")], line
        assert out["n_ties"][0] == 0


def test_tie_counts(orc):
    """Positive pins for the scan-boundary tie count (reading G7; Alg. 1 resample step,
    PAPER.md:326-331).  Hand derivations for tests/golden/systematic_ties.txt (U = x 2^-32):

    * N equal weights, x = 0: e_n = exp(0) = 1 exactly, P_m = m+1, C_m = fl((m+1)/N) and
      u_n = fl(n/N) -- the same correctly rounded quotient -- so u_n == C_{n-1} for n = 1..N-1:
      N-1 ties (N = 4: 3, N = 8: 7, N = 3: 2).  a_n = #{m : C_m <= u_n} = n (identity).
    * (.5, 0, 0, .5), x = 0: e = (1, 0, 0, 1), C = (.5, .5, .5, 1), u = (0, .25, .5, .75).
      u_2 = .5 meets the zero-weight plateau C_0 = C_1 = C_2: 3 ties (each pair counts once).
      a = (0, 0, 3, 3): the zero-weight particles 1, 2 are skipped.
    * (0, 0, 1, 1), x = 0: C = (0, 0, .5, 1); u_0 = 0 meets C_0 = C_1 (2 ties), u_2 = .5 meets
      C_2 (1 tie): 3.  a = (2, 2, 3, 3): the plateau at zero is never chosen even at u = 0.
    * N = 4 equal, x = 1: u_n - C_{n-1} = 2^-32/4 = 2^-34 > 2^-40: no tie.
    * N = 48 and 64 equal, x = 0: as above, N-1 ties (the GPU's two-particles-per-lane S6);
      N = 64, x = 1: none.
    * (.5, 0 x 38, .5), N = 40, x = 0: e = (1, 0, ..., 0, 1), C_0..C_38 = .5, C_39 = 1,
      u_n = n/40.  u_20 = .5 meets the 39-entry plateau: 39 ties.  a_n = 0 for n < 20 (u < .5)
      and 39 from n = 20 on (all 39 plateau entries are <= u): offspring 20 and 20.
    """
    for line in read_golden("systematic_ties.txt"):
        w, x, anc, off, ties = [s.strip() for s in line.split(";")]
        out = orc.resample(_logw([float(v) for v in w.split(",")]), eta=np.inf,
                           uniforms=np.array([int(x)], np.uint32))
        assert out["ancestors"][0].tolist() == [int(v) for v in anc.split(",")], line
        assert out["offspring"][0].tolist() == [int(v) for v in off.split(",")], line
        assert int(out["n_ties"][0]) == int(ties), line


def test_tie_threshold_boundary(orc):
    """The tie radius is 2^-40 inclusive (reading G7).  N = 1024 equal weights: C_{n-1} = n/1024
    and u_n = (n + x 2^-32)/1024 are exact in fp64, so u_n - C_{n-1} = x 2^-42.  x = 4 gives
    exactly 2^-40 (a tie at each of the 1023 interior boundaries); x = 5 gives 1.25 2^-40 (none).
    A strict '<', a wrong radius (2^-41 or 2^-39) or a one-sided count fails one of these."""
    lw = np.zeros((1, 1024), np.float32)
    for x, want in ((4, 1023), (5, 0), (0, 1023), (3, 1023)):
        out = orc.resample(lw, eta=np.inf, uniforms=np.array([x], np.uint32))
        assert int(out["n_ties"][0]) == want, x
        assert out["ancestors"][0].tolist() == list(range(1024))
    # radius 2^-39 would make x = 8 a tie; 2^-40 must not
    out = orc.resample(lw, eta=np.inf, uniforms=np.array([8], np.uint32))
    assert int(out["n_ties"][0]) == 0


def test_tie_count_multinomial(orc):
    """Multinomial uses the same tie rule over its i.i.d. u_n.  Equal weights (N = 4,
    C = (.25, .5, .75, 1)) with raw words 0, 2^30, 2^31, 3 2^30 (u = 0, .25, .5, .75) tie at
    u = .25, .5, .75: 3 ties; a_n = #{C_m <= u_n} = (0, 1, 2, 3)."""
    words = np.array([[0, 1 << 30, 1 << 31, 3 << 30]], np.uint32)
    out = orc.resample(np.zeros((1, 4), np.float32), eta=np.inf, scheme=1, uniforms=words)
    assert int(out["n_ties"][0]) == 3
    assert out["ancestors"][0].tolist() == [0, 1, 2, 3]


def _closed_form_offspring(C, U, N):
    o = np.zeros(N, np.int64)
    prev = 0.0
    for m in range(N):
        o[m] = math.ceil(N * C[m] - U) - math.ceil(N * prev - U)
        prev = C[m]
    return o


def test_closed_form_and_bounds(orc):
    rng = np.random.default_rng(17)
    for trial in range(200):
        N = int(rng.integers(1, 70))
        lw = (rng.standard_normal(N) * 2).astype(np.float32)[None, :]
        if trial % 3 == 0:
            lw[0, rng.random(N) < 0.3] = -np.inf
            lw[0, 0] = 0.0
        x = int(rng.integers(0, 2 ** 32))
        out = orc.resample(lw, eta=np.inf, uniforms=np.array([x], np.uint32))
        a, o, C = out["ancestors"][0], out["offspring"][0], out["cdf"][0]
        U = x / 2 ** 32
        assert o.sum() == N
        assert np.all(np.diff(a) >= 0)
        assert np.array_equal(np.bincount(a, minlength=N), o)
        if out["n_ties"][0] == 0:
            assert np.array_equal(_closed_form_offspring(C, U, N), o)
            wbar = out["wnorm"][0]
            assert np.all(o >= np.floor(N * wbar - 1e-9)) and np.all(o <= np.ceil(N * wbar + 1e-9))
        assert np.all(o[lw[0] == -np.inf] == 0)


def test_unbiased_over_stratified_sweep(orc):
    # o_m(U) has at most two unit jumps, so the midpoint rule over M strata gives
    # |mean_U o_m - N wbar_m| <= 2/M exactly (deterministic, no Monte Carlo).
    rng = np.random.default_rng(23)
    N, M = 32, 4096
    lw = (rng.standard_normal(N) * 1.5).astype(np.float32)[None, :]
    xs = ((np.arange(M) + 0.5) / M * 2 ** 32).astype(np.uint64).astype(np.uint32)
    tot = np.zeros(N)
    wbar = None
    for x in xs:
        out = orc.resample(lw, eta=np.inf, uniforms=np.array([x], np.uint32))
        tot += out["offspring"][0]
        wbar = out["wnorm"][0]
    assert np.max(np.abs(tot / M - N * wbar)) <= 2.0 / M


def test_special_cases(orc):
    # single surviving weight => every ancestor is that index
    lw = np.full((1, 9), -np.inf, np.float32); lw[0, 4] = -3.0
    out = orc.resample(lw, eta=np.inf, seed=1, step=2)
    assert np.all(out["ancestors"][0] == 4) and out["ess"][0] == 1.0
    # uniform weights => identity for any U
    for x in (0, 1, 2 ** 31, 2 ** 32 - 1):
        out = orc.resample(np.zeros((1, 13), np.float32), eta=np.inf, uniforms=np.array([x], np.uint32))
        assert out["ancestors"][0].tolist() == list(range(13)) and out["ess"][0] == 13.0
    # N = 1 reduces to plain proposal sampling: a = [0], ESS = 1, weight 1
    out = orc.resample(np.array([[-5.25]], np.float32), eta=np.inf, seed=3)
    assert out["ancestors"][0, 0] == 0 and out["ess"][0] == 1.0 and out["wnorm"][0, 0] == 1.0
    assert out["logw"][0, 0] == np.float32(-0.0)


def test_threshold_is_strict_and_no_resample_keeps_weights(orc):
    lw = np.zeros((1, 8), np.float32)                 # ESS = 8 exactly
    out = orc.resample(lw, eta=8.0)
    assert out["resampled"][0] == 0                   # ESS < eta is strict
    out = orc.resample(lw, eta=np.nextafter(8.0, 9.0))
    assert out["resampled"][0] == 1
    rng = np.random.default_rng(5)
    lw = (rng.standard_normal((3, 16))).astype(np.float32)
    out = orc.resample(lw, eta=0.0)
    assert np.all(out["resampled"] == 0)
    assert np.array_equal(out["logw"], lw)
    assert np.all(out["ancestors"] == np.arange(16)) and np.all(out["offspring"] == 1)


def test_reset_value_table(orc):
    # fl32(-ln N) for N = 1..1024 ("reset all weights to 1/N"; reading G8),
    # against Python's math.log, an independent libm call chain.
    for N in range(1, 1025):
        want = np.float32(-math.log(N))
        got = orc.neg_log_n(N)
        assert got.tobytes() == want.tobytes(), N


def test_slot_plan_is_a_hazard_free_permutation_of_ancestors(orc):
    rng = np.random.default_rng(41)
    for _ in range(300):
        N = int(rng.integers(1, 80))
        lw = (rng.standard_normal((1, N)) * 2.5).astype(np.float32)
        out = orc.resample(lw, eta=np.inf, seed=int(rng.integers(0, 2 ** 63)), step=7)
        a, o, s = out["ancestors"][0], out["offspring"][0], out["slot_src"][0]
        assert sorted(s.tolist()) == sorted(a.tolist())              # same multiset
        for m in range(N):
            if o[m] >= 1:
                assert s[m] == m                                      # survivors stay
            else:
                assert o[s[m]] >= 2                                   # dead <- duplicated source
        dsts = {n for n in range(N) if s[n] != n}
        srcs = {int(s[n]) for n in range(N) if s[n] != n}
        assert not (dsts & srcs)                                      # hazard-free in place
        dead = [m for m in range(N) if o[m] == 0]
        assert [int(s[m]) for m in dead] == sorted(int(s[m]) for m in dead)   # E ascending


def test_philox_stream_addressing(orc):
    # U is word 0 of Philox(key=seed, ctr=(step_lo, step_hi, prompt_base+p, 0)): the same
    # global prompt index gives the same ancestors whatever the local split (DP invariance).
    rng = np.random.default_rng(8)
    lw = (rng.standard_normal((6, 24)) * 2).astype(np.float32)
    full = orc.resample(lw, eta=np.inf, seed=0xABCDEF0123, step=(1 << 33) + 5)
    for base in (0, 2, 4):
        part = orc.resample(lw[base:base + 2], eta=np.inf, seed=0xABCDEF0123,
                            step=(1 << 33) + 5, prompt_base=base)
        assert np.array_equal(part["ancestors"], full["ancestors"][base:base + 2])
    w = orc.philox4x32_10([5, 2, 3, 0], [0x23, 0xAB])     # (step lo, step hi, prompt, 0)
    direct = orc.resample(lw[3:4], eta=np.inf, uniforms=np.array([w[0]], np.uint32))
    via = orc.resample(lw[3:4], eta=np.inf, seed=0xAB00000023, step=(2 << 32) + 5, prompt_base=3)
    assert np.array_equal(via["ancestors"], direct["ancestors"])


def test_degenerate_and_nonfinite(orc):
    lw = np.full((2, 5), -np.inf, np.float32)
    lw[1, 2] = np.nan
    out = orc.resample(lw, eta=np.inf)
    assert out["status"][0] == orc.ST_DEGENERATE
    assert out["status"][1] == orc.ST_DEGENERATE | orc.ST_NONFINITE
    assert np.all(out["lse"] == -np.inf) and np.all(out["ess"] == 0.0)
    assert np.all(out["resampled"] == 0) and np.all(out["ancestors"] == np.arange(5))


# ---------------------------------------------------------------- multinomial (NEXT #3)
def test_multinomial_frequencies(orc):
    # a_n ~ Cat(wbar) i.i.d. (Alg. 1): weights (.5,.3,.2), 1e5 draws, within
    # +-0.01 of the weights
    P = 33334
    lw = np.tile(np.log(np.array([0.5, 0.3, 0.2])).astype(np.float32), (P, 1))
    out = orc.resample(lw, eta=np.inf, scheme=1, seed=2024, step=1)
    freq = np.bincount(out["ancestors"].ravel(), minlength=3) / out["ancestors"].size
    assert np.allclose(freq, [0.5, 0.3, 0.2], atol=0.01)
    assert np.all(out["offspring"].sum(1) == 3)


def test_multinomial_uniform_chi_square(orc):
    from scipy.stats import chisquare
    P, N = 6250, 16
    out = orc.resample(np.zeros((P, N), np.float32), eta=np.inf, scheme=1, seed=7, step=3)
    counts = np.bincount(out["ancestors"].ravel(), minlength=N)
    assert chisquare(counts).pvalue > 1e-3


def test_multinomial_inverse_cdf_and_invariants(orc):
    rng = np.random.default_rng(12)
    for _ in range(50):
        N = int(rng.integers(1, 60))
        lw = (rng.standard_normal((1, N)) * 2).astype(np.float32)
        lw[0, rng.random(N) < 0.2] = -np.inf
        lw[0, int(rng.integers(0, N))] = 0.0
        words = rng.integers(0, 2 ** 32, size=(1, N), dtype=np.uint64).astype(np.uint32)
        out = orc.resample(lw, eta=np.inf, scheme=1, uniforms=words)
        C = out["cdf"][0]
        want = np.searchsorted(C, words[0].astype(np.float64) / 2 ** 32, side="right")
        if out["n_ties"][0] == 0:
            assert np.array_equal(out["ancestors"][0], want)
        a, o, s = out["ancestors"][0], out["offspring"][0], out["slot_src"][0]
        assert np.array_equal(np.bincount(a, minlength=N), o)
        assert sorted(s.tolist()) == sorted(a.tolist())
        assert np.all(o[lw[0] == -np.inf] == 0)
    # single surviving weight
    lw = np.full((1, 7), -np.inf, np.float32); lw[0, 2] = 1.0
    assert np.all(orc.resample(lw, eta=np.inf, scheme=1, seed=9)["ancestors"] == 2)


def test_multinomial_philox_addressing(orc):
    # u_n = word (n mod 4) of Philox(ctr = (step_lo, step_hi, prompt, 1 + n/4))
    lw = (np.random.default_rng(1).standard_normal((1, 9))).astype(np.float32)
    words = np.zeros((1, 9), np.uint32)
    for n in range(9):
        words[0, n] = orc.philox4x32_10([11, 0, 5, 1 + n // 4], [0x77, 0x0])[n % 4]
    direct = orc.resample(lw, eta=np.inf, scheme=1, uniforms=words)
    via = orc.resample(lw, eta=np.inf, scheme=1, seed=0x77, step=11, prompt_base=5)
    assert np.array_equal(direct["ancestors"], via["ancestors"])


def test_terminal_selection(orc):
    # one sequence sampled from the terminal normalised weights
    P = 40000
    lw = np.tile(np.log(np.array([0.1, 0.6, 0.3])).astype(np.float32), (P, 1))
    sel = orc.select(lw, seed=5, step=9)
    freq = np.bincount(sel["selected"], minlength=3) / P
    assert np.allclose(freq, [0.1, 0.6, 0.3], atol=0.01)
    dead = orc.select(np.full((2, 4), -np.inf, np.float32))
    assert np.all(dead["selected"] == -1) and np.all(dead["status"] == orc.ST_DEGENERATE)
    one = orc.select(np.array([[-np.inf, 3.0, -np.inf]], np.float32))
    assert one["selected"][0] == 1
