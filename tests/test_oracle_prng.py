"""Pins for the oracle's randomness: ChaCha20 against RFC 8439, and the samplers against
their distributions (reading R14)."""
import json
import math
import os
from decimal import Decimal, getcontext

import numpy as np

GOLD = os.path.join(os.path.dirname(__file__), "golden", "chacha20_rfc8439.json")


def _golden():
    with open(GOLD) as f:
        return json.load(f)


def test_chacha_quarter_round_rfc8439(O):
    g = _golden()["quarter_round"]
    got = O.chacha_quarter(*[int(x, 16) for x in g["in"]])
    assert got == [int(x, 16) for x in g["out"]]


def test_chacha_block_rfc8439(O):
    g = _golden()["block"]
    kb = bytes.fromhex(g["key_bytes"])
    nb = bytes.fromhex(g["nonce_bytes"])
    key = [int.from_bytes(kb[4 * i:4 * i + 4], "little") for i in range(8)]
    nonce = [int.from_bytes(nb[4 * i:4 * i + 4], "little") for i in range(3)]
    got = O.chacha20_block(key, g["counter"], nonce)
    assert [int(x) for x in got] == [int(x, 16) for x in g["state_out"]]


def test_draw_addresses_stream_words(O):
    seed, purpose, obj, sub = 0x0123456789ABCDEF, 9, (5 << 32) + 7, 2
    key = [seed & 0xFFFFFFFF, seed >> 32, purpose, 0, 0, 0, 0, 0]
    nonce = [obj & 0xFFFFFFFF, obj >> 32, sub]
    for n in (0, 1, 7, 8, 1000, 16383):
        blk = O.chacha20_block(key, n // 8, nonce)
        w = 2 * (n % 8)
        assert O.draw(seed, purpose, obj, sub, n) == int(blk[w]) | (int(blk[w + 1]) << 32)


def test_uniform_sampler(O):
    q = O.primes()[2]
    x = O.sample(11, 2, 0, 2, O.KIND_UNIFORM, 4096, q)
    # value = (draw(2k+1) << 64 | draw(2k)) mod q
    for k in (0, 1, 4095):
        v = (O.draw(11, 2, 0, 2, 2 * k + 1) << 64 | O.draw(11, 2, 0, 2, 2 * k)) % q
        assert int(x[k]) == v
    xf = x.astype(np.float64) / q
    assert (x < np.uint64(q)).all()
    assert abs(xf.mean() - 0.5) < 0.02
    hist = np.histogram(xf, bins=16, range=(0, 1))[0]
    chi2 = ((hist - 256) ** 2 / 256).sum()
    assert chi2 < 45  # 15 dof, p ~ 1e-4


def test_ternary_sampler(O):
    x = O.sample(3, 1, 0, 0, O.KIND_TERNARY, 60000)
    assert set(np.unique(x)) <= {-1, 0, 1}
    c = np.bincount(x + 1, minlength=3) / len(x)
    assert np.all(np.abs(c - 1 / 3) < 0.01)
    assert int(x[5]) == O.draw(3, 1, 0, 0, 5) % 3 - 1


def _exact_cdt():
    getcontext().prec = 80
    sig2 = Decimal("3.2") ** 2
    rho = [(-(Decimal(k) ** 2) / (2 * sig2)).exp() for k in range(20)]
    Z = rho[0] + 2 * sum(rho[1:])
    out, acc = [], rho[0]
    for k in range(19):
        if k > 0:
            acc += 2 * rho[k]
        out.append(int((Decimal(2) ** 63 * acc / Z).to_integral_value(rounding="ROUND_FLOOR")))
    return out


def test_gaussian_sampler_matches_exact_cdt(O):
    """Sampler output = #{k: v >= CDT_k} with sign from the top bit, where CDT_k is the exact
    floor(2^63 * Pr(|X|<=k)) of the sigma=3.2 discrete Gaussian (recomputed here at 80 digits
    with a symmetric-sum formulation)."""
    cdt = _exact_cdt()
    x = O.sample(7, 3, 0, 0, O.KIND_GAUSS, 3000)
    for k in range(3000):
        r = O.draw(7, 3, 0, 0, k)
        v = r & (2 ** 63 - 1)
        mag = sum(1 for t in cdt if v >= t)
        assert int(x[k]) == (-mag if r >> 63 else mag)


def test_gaussian_sampler_distribution(O):
    x = O.sample(8, 3, 1, 0, O.KIND_GAUSS, 200000).astype(np.float64)
    assert np.abs(x).max() <= 19
    assert abs(x.mean()) < 0.05
    assert abs(x.std() - 3.2) < 0.03
    # P(0) of a discrete Gaussian with sigma 3.2 ~ 1 / (sigma sqrt(2 pi)) (theta-function error < 1e-30)
    p0 = (x == 0).mean()
    assert abs(p0 - 1 / (3.2 * math.sqrt(2 * math.pi))) < 0.003
