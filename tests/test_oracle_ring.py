"""Pins for the oracle's ring layer: primes, negacyclic product, automorphism.

Everything here is checked against mathematics independent of the oracle code:
Python big-integer Miller-Rabin, schoolbook negacyclic convolution, monomial identities.
"""
import math
import random

import numpy as np
import pytest

# BASELINE.json configs[0]: "Q={58-bit,40-bit} + P={60-bit} NTT-friendly primes (largest below
# 2^k with q = 1 mod 16384), logPQ ~ 158"; values recomputed in SURVEY.md Appendix A.
APPENDIX_A = {58: 288230376150876161, 40: 1099511480321, 60: 1152921504606830593}


def _mr(n):
    """Independent deterministic Miller-Rabin (bases: first 13 primes, exact for n < 3.3e24)."""
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41]
    for p in small:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def test_primes_match_definition(O):
    q0, q1, P = O.primes()
    for bits, q in ((58, q0), (40, q1), (60, P)):
        assert q == APPENDIX_A[bits]
        assert q < 2 ** bits and q % 16384 == 1
        assert _mr(q)
        # "largest": every larger candidate below 2^bits with q = 1 mod 16384 is composite
        c = q + 16384
        while c < 2 ** bits:
            assert not _mr(c)
            c += 16384
    # PAPER.md:533 "log PQ ~ 158"
    assert abs(math.log2(q0 * q1 * P) - 158.0) < 0.01
    # 2N | q - 1 for N = 8192: negacyclic NTT exists for every N <= 8192
    assert all((q - 1) % 16384 == 0 for q in (q0, q1, P))


def test_oracle_primality_agrees(O):
    rnd = random.Random(5)
    L = O.lib()
    for _ in range(2000):
        n = rnd.getrandbits(rnd.choice([8, 20, 40, 61]))
        assert bool(L.or_is_prime(n)) == _mr(n)
    for q in APPENDIX_A.values():
        assert L.or_is_prime(q) == 1


def _schoolbook(a, b, q):
    n = len(a)
    c = [0] * n
    for i in range(n):
        for j in range(n):
            if i + j < n:
                c[i + j] += a[i] * b[j]
            else:
                c[i + j - n] -= a[i] * b[j]
    return [x % q for x in c]


@pytest.mark.parametrize("logN", [1, 2, 4, 5, 6])
@pytest.mark.parametrize("which", [0, 1, 2])
def test_poly_mul_equals_schoolbook(O, logN, which):
    q = O.primes()[which]
    n = 1 << logN
    rnd = random.Random(100 * logN + which)
    for _ in range(3):
        a = [rnd.randrange(q) for _ in range(n)]
        b = [rnd.randrange(q) for _ in range(n)]
        got = O.poly_mul(logN, q, np.array(a, np.uint64), np.array(b, np.uint64))
        assert [int(x) for x in got] == _schoolbook(a, b, q)


@pytest.mark.parametrize("which", [0, 1, 2])
def test_monomial_products_N8192(O, which):
    """X^a * X^b = (-1)^[a+b >= N] X^((a+b) mod N) in Z_q[X]/(X^N+1) at the real N = 8192."""
    q = O.primes()[which]
    N = 8192
    rnd = random.Random(which)
    for _ in range(4):
        a, b = rnd.randrange(N), rnd.randrange(N)
        ca, cb = rnd.randrange(1, q), rnd.randrange(1, q)
        A = np.zeros(N, np.uint64)
        B = np.zeros(N, np.uint64)
        A[a] = ca
        B[b] = cb
        got = O.poly_mul(13, q, A, B)
        exp = np.zeros(N, dtype=object)
        v = ca * cb % q
        exp[(a + b) % N] = v if a + b < N else (q - v) % q
        assert [int(x) for x in got] == list(exp)


def test_poly_mul_identity_and_linearity_N8192(O):
    q = O.primes()[0]
    rng = np.random.default_rng(3)
    a = rng.integers(0, q, 8192, dtype=np.uint64)
    one = np.zeros(8192, np.uint64)
    one[0] = 1
    assert np.array_equal(O.poly_mul(13, q, a, one), a)
    b = rng.integers(0, q, 8192, dtype=np.uint64)
    c = rng.integers(0, q, 8192, dtype=np.uint64)
    lhs = O.poly_mul(13, q, a, (b.astype(object) + c.astype(object)) % q)
    rhs = (O.poly_mul(13, q, a, b).astype(object) + O.poly_mul(13, q, a, c).astype(object)) % q
    assert list(lhs.astype(object)) == list(rhs)


@pytest.mark.parametrize("logN", [3, 6])
def test_automorphism_is_ring_map(O, logN):
    """sigma_g(a) defined by X -> X^g: matches direct substitution and is multiplicative."""
    q = O.primes()[0]
    n = 1 << logN
    rnd = random.Random(logN)
    a = [rnd.randrange(q) for _ in range(n)]
    b = [rnd.randrange(q) for _ in range(n)]
    for g in (5, 25, 2 * n - 1, pow(5, 3, 2 * n)):
        # direct substitution: a_k X^(k g), reduced with X^N = -1
        exp = [0] * n
        for k, v in enumerate(a):
            e = k * g % (2 * n)
            if e < n:
                exp[e] = (exp[e] + v) % q
            else:
                exp[e - n] = (exp[e - n] - v) % q
        got = O.automorphism(logN, q, np.array(a, np.uint64), g)
        assert [int(x) for x in got] == exp
        ab = O.poly_mul(logN, q, np.array(a, np.uint64), np.array(b, np.uint64))
        lhs = O.automorphism(logN, q, ab, g)
        rhs = O.poly_mul(logN, q, got, O.automorphism(logN, q, np.array(b, np.uint64), g))
        assert np.array_equal(lhs, rhs)
