"""Pins for the oracle merge (O2): W' = RNE_bf16(W + (alpha/r) B A).

The reference for 'correctly rounded' is exact rational arithmetic
(fractions.Fraction) with a hand-written round-half-even onto the bf16 grid —
independent of numpy and of the oracle's rounding helper.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle.merge import merge_bf16_bits, merge_f64
from oracle.numerics import bf16_bits_to_f64, f64_to_bf16_bits, rne_bf16


def rand_bf16(rng, shape, scale):
    x = rng.uniform(-scale, scale, size=shape)
    return f64_to_bf16_bits(x)


def frac_round_bf16(q: Fraction) -> Fraction:
    """Round a rational to the nearest bf16 value, ties to even (8 significant bits)."""
    if q == 0:
        return Fraction(0)
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = 0
    while a >= 2:
        a /= 2
        e += 1
    while a < 1:
        a *= 2
        e -= 1
    # a in [1, 2): 8 significant bits -> quantum 2^-7 on a
    scaled = a * 128
    n = scaled.numerator // scaled.denominator
    rem = scaled - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return sign * Fraction(n, 128) * (Fraction(2) ** e)


@pytest.mark.parametrize("shape", [(3, 1, 5), (4, 2, 3), (5, 4, 7), (2, 8, 2)])
def test_merge_correctly_rounded_bruteforce(shape):
    o, r, i = shape
    rng = np.random.default_rng(sum(shape))
    W = rand_bf16(rng, (o, i), 0.05)
    B = rand_bf16(rng, (o, r), 0.5)
    A = rand_bf16(rng, (r, i), 0.5)
    s = 2.0
    got = bf16_bits_to_f64(merge_bf16_bits(W, B, A, s))
    Wf, Bf, Af = (bf16_bits_to_f64(x) for x in (W, B, A))
    for a in range(o):
        for b in range(i):
            exact = Fraction(Wf[a, b]) + Fraction(s) * sum(Fraction(Bf[a, k]) * Fraction(Af[k, b]) for k in range(r))
            assert Fraction(got[a, b]) == frac_round_bf16(exact), (a, b)


def test_rne_bf16_ties_to_even():
    # 1 + 2^-8 is exactly halfway between 1 and 1+2^-7 -> even (1.0); 1 + 3*2^-8 -> 1 + 2^-6
    assert rne_bf16(np.array([1 + 2 ** -8]))[0] == 1.0
    assert rne_bf16(np.array([1 + 3 * 2 ** -8]))[0] == 1 + 2 ** -6
    assert rne_bf16(np.array([-(1 + 2 ** -8)]))[0] == -1.0
    # values already on the grid are unchanged
    x = bf16_bits_to_f64(np.arange(0, 65535, 97, dtype=np.uint16))
    x = x[np.isfinite(x)]
    assert np.array_equal(rne_bf16(x), x)


def test_zero_delta_is_identity():
    rng = np.random.default_rng(0)
    W = rand_bf16(rng, (16, 32), 0.05)
    A = rand_bf16(rng, (4, 32), 0.5)
    Bz = np.zeros((16, 4), dtype=np.uint16)
    assert np.array_equal(merge_bf16_bits(W, Bz, A, 2.0), W)            # B = 0
    B = rand_bf16(rng, (16, 4), 0.5)
    assert np.array_equal(merge_bf16_bits(W, B, A, 0.0), W)             # s = 0


def test_one_hot_A_closed_form():
    # A = e_k (row k is the unit vector e_j0) => delta = s * B[:, k] placed in column j0 only
    rng = np.random.default_rng(1)
    o, r, i = 8, 4, 6
    Wf = bf16_bits_to_f64(rand_bf16(rng, (o, i), 0.05))
    Bf = bf16_bits_to_f64(rand_bf16(rng, (o, r), 0.5))
    k, j0 = 2, 3
    Af = np.zeros((r, i)); Af[k, j0] = 1.0
    D = merge_f64(Wf, Bf, Af, 2.0) - Wf
    expect = np.zeros((o, i)); expect[:, j0] = 2.0 * Bf[:, k]
    assert np.array_equal(D, expect)


def test_rank_one_outer_product():
    rng = np.random.default_rng(2)
    Wf = bf16_bits_to_f64(rand_bf16(rng, (5, 7), 0.05))
    b = bf16_bits_to_f64(rand_bf16(rng, (5, 1), 0.5))
    a = bf16_bits_to_f64(rand_bf16(rng, (1, 7), 0.5))
    D = merge_f64(Wf, b, a, 2.0) - Wf
    for x in range(5):
        for y in range(7):
            assert D[x, y] == 2.0 * b[x, 0] * a[0, y]


def test_delta_rank_at_most_r():
    rng = np.random.default_rng(3)
    for r in (1, 2, 5):
        Wf = bf16_bits_to_f64(rand_bf16(rng, (20, 24), 0.05))
        Bf = bf16_bits_to_f64(rand_bf16(rng, (20, r), 0.5))
        Af = bf16_bits_to_f64(rand_bf16(rng, (r, 24), 0.5))
        D = merge_f64(Wf, Bf, Af, 2.0) - Wf
        assert np.linalg.matrix_rank(D) <= r


def test_transpose_identity():
    # (W + sBA)^T == W^T + s A^T B^T : merging the transposed problem gives the transposed result
    rng = np.random.default_rng(4)
    W = rand_bf16(rng, (9, 11), 0.05)
    B = rand_bf16(rng, (9, 3), 0.5)
    A = rand_bf16(rng, (3, 11), 0.5)
    assert np.array_equal(merge_bf16_bits(W, B, A, 2.0).T, merge_bf16_bits(W.T.copy(), A.T.copy(), B.T.copy(), 2.0))


# ---------------------------------------------------------------------------------------------------
# fp32 debug-parity models (SURVEY.md §8(c) "Tolerances", 1e-4 gate): W' = RNE_f32(W + s B A)
# ---------------------------------------------------------------------------------------------------

def frac_round_sig(q: Fraction, bits: int) -> Fraction:
    """Round a rational to `bits` significant bits, ties to even (no exponent limits: normal range only)."""
    if q == 0:
        return Fraction(0)
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = 0
    while a >= 2:
        a /= 2
        e += 1
    while a < 1:
        a *= 2
        e -= 1
    scaled = a * (2 ** (bits - 1))
    n = scaled.numerator // scaled.denominator
    rem = scaled - n
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and n % 2 == 1):
        n += 1
    return sign * Fraction(n, 2 ** (bits - 1)) * (Fraction(2) ** e)


@pytest.mark.parametrize("shape", [(3, 1, 5), (4, 2, 3), (5, 8, 7), (2, 16, 3)])
def test_merge_f32_correctly_rounded_bruteforce(shape):
    """Exact rationals + hand-written round-half-even to 24 significant bits: the fp32 oracle merge is the
    correctly rounded value (its fp64 accumulation cannot move a result across an fp32 rounding boundary
    at these sizes unless the exact value sits within 2^-50 of a tie, which these random draws do not)."""
    from oracle.merge import merge_f32_values
    o, r, i = shape
    rng = np.random.default_rng(100 + sum(shape))
    W = rng.uniform(-0.05, 0.05, (o, i)).astype(np.float32)
    B = rng.uniform(-0.5, 0.5, (o, r)).astype(np.float32)
    A = rng.uniform(-0.5, 0.5, (r, i)).astype(np.float32)
    s = 2.0
    got = merge_f32_values(W, B, A, s)
    assert got.dtype == np.float32
    for a in range(o):
        for b in range(i):
            exact = Fraction(float(W[a, b])) + Fraction(s) * sum(
                Fraction(float(B[a, k])) * Fraction(float(A[k, b])) for k in range(r))
            assert Fraction(float(got[a, b])) == frac_round_sig(exact, 24), (a, b)


def test_merge_f32_identity_and_one_hot():
    from oracle.merge import merge_f32_values
    rng = np.random.default_rng(7)
    W = rng.uniform(-0.05, 0.05, (6, 9)).astype(np.float32)
    B = rng.uniform(-0.5, 0.5, (6, 4)).astype(np.float32)
    assert np.array_equal(merge_f32_values(W, np.zeros_like(B), rng.uniform(-1, 1, (4, 9)).astype(np.float32), 2.0), W)
    A = np.zeros((4, 9), dtype=np.float32)
    A[2, 5] = 1.0                                             # one-hot A: delta = s * B[:, 2] e_5^T
    got = merge_f32_values(W, B, A, 2.0)
    want = W.copy()
    want[:, 5] = (W[:, 5].astype(np.float64) + 2.0 * B[:, 2].astype(np.float64)).astype(np.float32)
    assert np.array_equal(got, want)
