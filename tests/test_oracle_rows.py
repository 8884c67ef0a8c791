"""Pins for the oracle's Philox, logit decode and S1/S2 (row log-softmax at the drafted token).

Each test checks the oracle against something other than itself: published KATs,
closed forms, invariants, or an independent library routine (scipy) on random rows.
"""
import math

import numpy as np
import pytest
from scipy.special import log_softmax

from conftest import read_golden


def test_philox_kat(orc):
    rows = read_golden("philox_kat.txt")
    assert len(rows) == 3
    for r in rows:
        w = [int(x, 16) for x in r.split()]
        out = orc.philox4x32_10(w[0:4], w[4:6])
        assert [int(x) for x in out] == w[6:10]


def _bf16(values):
    """bf16 bit patterns by truncation of exactly-representable fp32 values."""
    a = np.asarray(values, dtype=np.float32)
    return (a.view(np.uint32) >> 16).astype(np.uint16)


def test_bf16_decode_known_bits(orc):
    # 0x3F80 = 1.0, 0xC000 = -2.0, 0x4049 = 3.140625 -> with a single-token row the
    # log-softmax is 0 and the only information is the flag; use V=2 rows instead:
    # ell_0 = z0 - ln(e^z0 + e^z1).
    bits = np.array([0x3F80, 0xC000], dtype=np.uint16)  # (1.0, -2.0)
    ell, flag = orc.row_logprob(bits, 0)
    assert flag == 0
    assert ell == pytest.approx(1.0 - math.log(math.exp(1.0) + math.exp(-2.0)), abs=1e-15)
    bits = np.array([0x4049, 0x0000], dtype=np.uint16)  # (3.140625, 0.0)
    ell, _ = orc.row_logprob(bits, 1)
    assert ell == pytest.approx(0.0 - math.log(math.exp(3.140625) + 1.0), abs=1e-15)


def test_uniform_row_is_minus_log_v(orc):
    for V in (1, 2, 3, 1000, 128256):
        row = np.full(V, 0.25, dtype=np.float32)
        ell, flag = orc.row_logprob(row, V // 2)
        assert flag == 0
        assert ell == pytest.approx(-math.log(V), rel=1e-13, abs=1e-13)


def test_two_token_closed_form(orc):
    # z = (0, ln 3): p = (1/4, 3/4)  (Eq. 1a normalisation)
    row = np.array([0.0, math.log(3.0)], dtype=np.float64).astype(np.float32)
    z1 = float(row[1])
    ell1, _ = orc.row_logprob(row, 1)
    ell0, _ = orc.row_logprob(row, 0)
    assert ell1 == pytest.approx(z1 - math.log(1.0 + math.exp(z1)), abs=1e-15)
    assert ell1 == pytest.approx(math.log(0.75), abs=1e-7)
    assert ell0 == pytest.approx(math.log(0.25), abs=1e-7)


def test_normalisation_sums_to_one(orc):
    rng = np.random.default_rng(1)
    for V in (5, 97, 1000):
        row = (rng.standard_normal(V) * 3).astype(np.float32)
        tot = sum(math.exp(orc.row_logprob(row, d)[0]) for d in range(V))
        assert tot == pytest.approx(1.0, abs=1e-12)


def test_matches_scipy_log_softmax_random_rows(orc):
    rng = np.random.default_rng(2)
    for V, tau in ((1000, 1.0), (4096, 0.5), (777, 2.0)):
        row = (rng.standard_normal(V) * 4).astype(np.float32)
        ref = log_softmax(tau * row.astype(np.float64))
        for d in (0, V // 3, V - 1):
            ell, flag = orc.row_logprob(row, d, tau=tau)
            assert flag == 0
            assert ell == pytest.approx(ref[d], abs=1e-12)


def test_shift_invariance(orc):
    rng = np.random.default_rng(3)
    z = (np.round(rng.standard_normal(300) * 64) / 64).astype(np.float32)  # exact in fp32 after +-1000
    for c in (1000.0, -1000.0):
        zc = (z + np.float32(c)).astype(np.float32)
        assert np.all(zc.astype(np.float64) - c == z.astype(np.float64))
        for d in (0, 150, 299):
            assert orc.row_logprob(zc, d)[0] == pytest.approx(orc.row_logprob(z, d)[0], abs=1e-12)


def test_dominant_logit(orc):
    V = 1000
    row = np.zeros(V, dtype=np.float32)
    row[17] = 60.0
    ell, _ = orc.row_logprob(row, 17)
    assert ell == pytest.approx(-(V - 1) * math.exp(-60.0), abs=1e-20)
    ell_other, _ = orc.row_logprob(row, 3)
    assert ell_other == pytest.approx(-60.0, abs=1e-12)


def test_temperature_two_token(orc):
    # y = tau z (reading G9, SPEC.md:94-102 temper): p_tau(1) = 3^tau / (1 + 3^tau)
    row = np.array([0.0, math.log(3.0)], dtype=np.float32)
    z1 = float(row[1])
    for tau in (0.2, 0.5, 2.0, 5.0):
        ell, _ = orc.row_logprob(row, 1, tau=tau)
        assert ell == pytest.approx(tau * z1 - math.log(1.0 + math.exp(tau * z1)), abs=1e-14)


def test_masked_entries_and_flags(orc):
    row = np.array([0.0, -np.inf, 1.0, -np.inf], dtype=np.float32)
    ell, flag = orc.row_logprob(row, 2)
    assert flag == 0 and ell == pytest.approx(1.0 - math.log(1.0 + math.e), abs=1e-15)
    ell, flag = orc.row_logprob(row, 1)        # drafted token with p = 0 -> -inf, no flag
    assert flag == 0 and ell == -np.inf
    for bad in ([0.0, np.nan], [0.0, np.inf], [-np.inf, -np.inf]):
        ell, flag = orc.row_logprob(np.array(bad, dtype=np.float32), 0)
        assert flag == orc.ST_NONFINITE and math.isnan(ell)
