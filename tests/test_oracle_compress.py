"""Pins for the oracle's f1 row: output compression (
SPEC.md:321-329), with HE-C^3 run one level higher on the chain extended by q2 (reading R28):
level 2 -> tensor, 3-digit relin, Res by q2 -> level 1 -> ladder at level 1 -> per set t:
Res_q1(Mul(P)(C_t, M)) at level 0, right rotation by t mod s, added into packed ciphertext t // s.

Pins used (each independent of the oracle code path it checks):
  * the 3-digit relinearization key satisfies its gadget relation exactly (big integers)
  * relin + Res by q2: q2 (c0' + c1' s) = d0 + d1 s + d2 s^2 + (rounding terms) on the CRT lifts
  * trivial ciphertexts (c1 = 0): the whole compressed scan equals a big-integer closed form
  * SPEC.md:327's worked example (T = 2, s = 2, B = 4, S = 8) in real CKKS at N = 16
  * T = 1: the packed ciphertext holds the scores at slots k s and ZEROS elsewhere (the garbage
    partial sums of the uncompressed output are masked away)
  * end to end at N = 8192: the packed scores of two sets equal the plaintext cosines, top-1
"""
import json
import os
import random

import numpy as np
import pytest

from paper_2408_06167_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def _crt(res, mods):
    M = 1
    for m in mods:
        M *= m
    x = 0
    for r, m in zip(res, mods):
        Mi = M // m
        x += int(r) * Mi * pow(Mi, -1, m)
    return x % M


def _cent(x, m):
    x %= m
    return x - m if x > m // 2 else x


def _negacyclic_big(a, b):
    n = len(a)
    c = [0] * n
    for i in range(n):
        if a[i] == 0:
            continue
        for j in range(n):
            if i + j < n:
                c[i + j] += a[i] * b[j]
            else:
                c[i + j - n] -= a[i] * b[j]
    return c


def _sigma_int(a, g):
    n = len(a)
    out = [0] * n
    for k, v in enumerate(a):
        t = k * g % (2 * n)
        if t < n:
            out[t] += v
        else:
            out[t - n] -= v
    return out


def _rnd_div(x, m):          # (X - c_m(X)) / m: the rescale rounding on true integers
    return (x - _cent(x, m)) // m


def test_rlk2_relation(O):
    """rlk2[j]: b + a s = [l = j] (P mod q_l) s^2 in limbs q0, q1, q2 and 0 in limb P (zero errors)."""
    logN = 5
    N = 1 << logN
    q0, q1, P = O.primes()
    q2 = O.q2()
    sk, pk, rlk, gk = O.keygen(logN, 9, 0)
    rlk2, gkl, gkc = O.keygen_cmp(logN, 9, 8, 2, zero_error=True)
    s = [int(v) for v in sk]
    s2 = _negacyclic_big(s, s)
    for j in range(3):
        for l, q in enumerate((q0, q1, q2, P)):
            b = [int(v) for v in rlk2[j, 0, l]]
            asum = _negacyclic_big([int(v) for v in rlk2[j, 1, l]], s)
            lhs = [(b[k] + asum[k]) % q for k in range(N)]
            rhs = [((P % q) * s2[k]) % q if l == j else 0 for k in range(N)]
            assert lhs == rhs, (j, l)


def test_relin_rescale_l2_identity(O):
    """q2 (c0' + c1' s) = d0 + d1 s + d2 s^2 + e (mod q0 q1 q2), |e| <= (N+1)(q2/2 + 1): the ModDown
    rounding plus the Res rounding z0 + z1 s -- a wrong digit, limb or gadget constant gives e ~ Q."""
    logN = 5
    N = 1 << logN
    q0, q1, P = O.primes()
    q2 = O.q2()
    mods = (q0, q1, q2)
    Q2 = q0 * q1 * q2
    sk, pk, rlk, gk = O.keygen(logN, 3, 0)
    rlk2, _, _ = O.keygen_cmp(logN, 3, 8, 2, zero_error=True)
    rnd = random.Random(41)
    d = np.array([[[rnd.randrange(m) for _ in range(N)] for m in mods] for _ in range(3)], np.uint64)
    out = O.relin_rescale_l2(logN, d, rlk2)
    s = [int(v) for v in sk]
    D = [[_crt([d[i][0][k], d[i][1][k], d[i][2][k]], mods) for k in range(N)] for i in range(3)]
    C = [[_crt([out[c][0][k], out[c][1][k]], (q0, q1)) for k in range(N)] for c in range(2)]
    lhs = [q2 * (C[0][k] + v) for k, v in enumerate(_negacyclic_big(C[1], s))]
    rhs1, rhs2 = _negacyclic_big(D[1], s), _negacyclic_big(D[2], _negacyclic_big(s, s))
    e = [_cent(lhs[k] - D[0][k] - rhs1[k] - rhs2[k], Q2) for k in range(N)]
    assert max(abs(v) for v in e) <= (N + 1) * (q2 // 2 + 1)
    assert max(abs(v) for v in e) > 0


@pytest.mark.parametrize("T", [3, 5])
def test_trivial_compressed_scan_closed_form(O, T):
    """c1 = 0 everywhere: packed g = sum_{u} sigma_{5^(S-u)}(round(M L_t / q1)), t = g s + u, with
    L_t = sum_{delta < s} sigma_{5^delta}(round(sum_i pu_i ps_{t,i} / q2)) (Res q2, the level-1 ladder)."""
    logN, d, p = 6, 8, 2                  # N = 64, S = 32, s = 4, B = 8
    N = 1 << logN
    S, s, B = O.layout(logN, d, p)
    q0, q1, P = O.primes()
    q2 = O.q2()
    rlk2, gkl, gkc = O.keygen_cmp(logN, 6, d, p)
    rnd = random.Random(70 + T)
    r30 = lambda: [rnd.randrange(-2 ** 30, 2 ** 30) for _ in range(N)]
    pu = [r30() for _ in range(p)]
    ps = [[r30() for _ in range(p)] for _ in range(T)]
    mask = [rnd.randrange(-2 ** 40, 2 ** 40) for _ in range(N)]

    def trivial(pt):
        ct = np.zeros((2, 3, N), np.uint64)
        for l, m in enumerate((q0, q1, q2)):
            ct[0, l] = [v % m for v in pt]
        return ct
    q = np.stack([trivial(v) for v in pu])[None]
    db = np.stack([np.stack([trivial(v) for v in ps[t]]) for t in range(T)])
    out = O.match_cmp(logN, d, p, rlk2, gkl, gkc, np.array(mask, np.int64), db, q)
    G = -(-T // s)
    assert out.shape[:2] == (1, G)
    for g in range(G):
        acc = [0] * N
        for u in range(s):
            t = g * s + u
            if t >= T:
                break
            prod = [sum(x) for x in zip(*[_negacyclic_big(pu[i], ps[t][i]) for i in range(p)])]
            C = [_rnd_div(v, q2) for v in prod]
            L = [0] * N
            for delta in range(s):
                L = [a + b for a, b in zip(L, _sigma_int(C, pow(5, delta, 2 * N)))]
            K = [_rnd_div(v, q1) for v in _negacyclic_big(mask, L)]
            R = _sigma_int(K, pow(5, S - u, 2 * N)) if u else K
            acc = [a + b for a, b in zip(acc, R)]
        assert [int(v) for v in out[0, g, 0, 0]] == [v % q0 for v in acc], g
        assert not out[0, g, 1].any()


def _cmp_scan(O, logN, d, p, T, qv, key_seed=1, n_threads=4):
    S, s, B = O.layout(logN, d, p)
    n_sets = -(-T.shape[0] // B)
    sk, pk, rlk, gk = O.keygen(logN, key_seed, 0)
    pk_q2, _ = O.keygen_exp(logN, key_seed, d, p)
    rlk2, gkl, gkc = O.keygen_cmp(logN, key_seed, d, p)
    zdb = O.pack_db(T, logN, d, p, 0, n_sets)
    db = O.encrypt_l2(logN, pk, pk_q2, O.encode(zdb.reshape(-1, S), logN), 0, 2).reshape(n_sets, p, 2, 3, -1)
    zq = O.pack_query(qv, logN, d, p)
    qc = O.encrypt_l2(logN, pk, pk_q2, O.encode(zq.reshape(-1, S), logN), 0, 3).reshape(len(qv), p, 2, 3, -1)
    out = O.match_cmp(logN, d, p, rlk2, gkl, gkc, O.cmp_mask(logN, d, p), db, qc, n_threads=n_threads)
    return out, sk, n_sets


def test_spec_compression_example_N16(O):
    """T = 2, s = 2, B = 4, S = 8: packed = [a0, b0, a1, b1, a2, b2, a3, b3] with a_k, b_k
    the scores of set 0 / set 1 block k -- in real CKKS at N = 16 (d = 4, p = 2)."""
    logN, d, p = 4, 4, 2
    T = I.random_unit(8, d, 4)
    qv = I.random_unit(1, d, 5)
    out, sk, n_sets = _cmp_scan(O, logN, d, p, T, qv)
    assert n_sets == 2 and out.shape[1] == 1
    q0 = O.primes()[0]
    m = O.decrypt(logN, sk, out[0, 0], 1)[0]
    z = O.decode_slots(O.centred_i64(m, q0), logN, O.DELTA ** 2 / O.q2())
    cos = (qv @ T.T)[0]
    want = np.empty(8)
    want[0::2], want[1::2] = cos[:4], cos[4:]           # [a0, b0, a1, b1, ...]
    assert np.abs(z - want).max() < 1e-6


def test_single_set_compression_masks_the_garbage(O):
    """T = 1: mask + rescale only; the packed ciphertext decrypts to the scores at slots
    k s and to zero at every other slot (the uncompressed output carries partial sums there)."""
    logN, d, p = 8, 16, 2                  # S = 128, s = 8, B = 16
    T = I.random_unit(16, d, 6)
    qv = I.random_unit(1, d, 7)
    out, sk, n_sets = _cmp_scan(O, logN, d, p, T, qv)
    q0 = O.primes()[0]
    m = O.decrypt(logN, sk, out[0, 0], 1)[0]
    z = O.decode_slots(O.centred_i64(m, q0), logN, O.DELTA ** 2 / O.q2())
    S, s, B = O.layout(logN, d, p)
    assert np.abs(z[0::s] - (qv @ T.T)[0]).max() < 1e-6
    other = np.delete(z, np.arange(0, S, s))
    assert np.abs(other).max() < 1e-6


def test_compressed_scan_end_to_end(O):
    """N = 8192, d = 16, p = 4 (s = 4, B = 1024): 1500 templates in two sets packed into one ciphertext;
    decrypted packed scores equal the plaintext cosines (1e-6) and the argmax is the genuine template."""
    logN, d, p = 13, 16, 4
    T = I.random_unit(1500, d, 13)
    qv = T[1234:1235] + 0.05 * np.random.default_rng(8).standard_normal((1, d))
    qv /= np.linalg.norm(qv)
    out, sk, n_sets = _cmp_scan(O, logN, d, p, T, qv)
    assert n_sets == 2 and out.shape[1] == 1
    sc = O.packed_scores(logN, d, p, sk, out[0], n_sets)[:1500]
    ref = (qv @ T.T)[0]
    assert np.abs(sc - ref).max() < 1e-6
    assert sc.argmax() == ref.argmax() == 1234
