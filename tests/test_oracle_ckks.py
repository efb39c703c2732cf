"""Pins for the oracle's CKKS layer and for Algorithm 2 (HE-C^3).

Pins used (each independent of the oracle code path it checks):
  * encode: direct O(N*S) definition at small N; decode(encode(z)) ~ z; slot j <-> zeta^(5^j)
  * Dec(Enc(m)) ~ m
  * ModDown / rescale: Python big-integer closed forms on the CRT lift
  * relinearization: Dec(relin(d)) - (d0 + d1 s + d2 s^2) is the ModDown rounding term,
    bounded by (N+1)/2 for error-free keys (exact algebra, see DESIGN.md sec. Oracle)
  * automorphism == slot rotation: decode(sigma_{5^r}(encode(z))) = rot_left(z, r)
  * trivial ciphertexts (c1 = 0): the whole scan equals a big-integer closed form
  * end-to-end: decrypted scores vs float64 cosine (north_star 1e-4, internal guard 1e-6)
  * SPEC.md worked examples at S = 8 in real CKKS at N = 16
"""
import json
import os
import random

import numpy as np
import pytest

from paper_2408_06167_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def _rot_left(z, r):
    return np.roll(z, -r, axis=-1)


# ----------------------------------------------------------------------------- encoding
@pytest.mark.parametrize("logN", [3, 5, 7])
def test_encode_fft_equals_direct_definition(O, logN):
    S = (1 << logN) // 2
    z = np.random.default_rng(logN).uniform(-1, 1, S)
    assert np.array_equal(O.encode(z, logN), O.encode_direct(z, logN))


@pytest.mark.parametrize("logN", [4, 13])
def test_decode_encode_roundtrip(O, logN):
    S = (1 << logN) // 2
    z = np.random.default_rng(1).uniform(-1, 1, S)
    pt = O.encode(z, logN)
    back = O.decode_slots(pt, logN, O.DELTA)
    assert np.abs(back - z).max() < 1e-9


def test_encoding_evaluates_at_5_power_roots(O):
    """m(zeta^(5^j)) = z_j: evaluate the real polynomial at the slot roots with complex numbers."""
    logN = 5
    N = 1 << logN
    z = np.random.default_rng(2).uniform(-1, 1, N // 2)
    m = O.encode(z, logN).astype(np.float64) / O.DELTA
    for j in range(N // 2):
        root = np.exp(1j * np.pi * pow(5, j, 2 * N) / N)
        val = np.polyval(m[::-1], root)
        assert abs(val.real - z[j]) < 1e-9 and abs(val.imag) < 1e-9


# ----------------------------------------------------------------------------- rotation semantics
@pytest.mark.parametrize("r", [1, 2, 3, 8])
def test_automorphism_rotates_slots_left(O, r):
    logN = 6
    S = 32
    q0 = O.primes()[0]
    z = np.random.default_rng(r).uniform(-1, 1, S)
    pt = O.encode(z, logN)
    res = np.array([int(x) % q0 for x in pt], np.uint64)
    g = pow(5, r, 2 << logN)
    rot = O.automorphism(logN, q0, res, g)
    back = O.decode_slots(O.centred_i64(rot, q0), logN, O.DELTA)
    assert np.abs(back - _rot_left(z, r)).max() < 1e-9
    # rotation by S is the identity (ord(5) = S mod 2N)
    assert pow(5, S, 2 << logN) == 1


# ----------------------------------------------------------------------------- enc / dec
def test_encrypt_decrypt_roundtrip(O):
    logN = 13
    S = 4096
    sk, pk, rlk, gk = O.keygen(logN, 1, 0)
    z = np.random.default_rng(4).uniform(-1, 1, (2, S))
    ct = O.encrypt(logN, pk, O.encode(z, logN), 0, 9)
    q0 = O.primes()[0]
    for i in range(2):
        m = O.decrypt(logN, sk, ct[i], 2)
        back = O.decode_slots(O.centred_i64(m[0], q0), logN, O.DELTA)
        assert np.abs(back - z[i]).max() < 1e-6


def test_public_key_relation(O):
    """pk = (b, a) with b + a s = e small (RLWE sample)."""
    logN = 8
    sk, pk, rlk, gk = O.keygen(logN, 5, 2)
    for l in range(2):
        q = O.primes()[l]
        s = np.array([int(x) % q for x in sk], np.uint64)
        e = (pk[0, l].astype(object) + O.poly_mul(logN, q, pk[1, l], s).astype(object)) % q
        e = [int(x) - q if int(x) > q // 2 else int(x) for x in e]
        assert max(abs(x) for x in e) <= 19


# ----------------------------------------------------------------------------- ModDown / rescale closed forms
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


def test_moddown_closed_form(O):
    """ModDown(X) = (X - c_P(X)) / P mod Q for the CRT lift X (SURVEY.md sec. 8c pins)."""
    q0, q1, P = O.primes()
    logN = 4
    N = 16
    rnd = random.Random(7)
    KS = np.array([[rnd.randrange(m) for _ in range(N)] for m in (q0, q1, P)], np.uint64)
    got = O.moddown(logN, 2, KS)
    for k in range(N):
        X = _crt([KS[0, k], KS[1, k], KS[2, k]], [q0, q1, P])
        y = (X - _cent(X, P)) // P
        assert (X - _cent(X, P)) % P == 0
        assert int(got[0, k]) == y % q0 and int(got[1, k]) == y % q1


def test_rescale_closed_form(O):
    """Res: (X - c_q1(X)) / q1 mod q0 for X = CRT(c[q0], c[q1]) (round to nearest, reading R5)."""
    q0, q1, P = O.primes()
    logN = 4
    N = 16
    rnd = random.Random(8)
    ct = np.array([[[rnd.randrange(m) for _ in range(N)] for m in (q0, q1)] for _ in range(2)], np.uint64)
    got = O.rescale(logN, ct)
    for c in range(2):
        for k in range(N):
            X = _crt([ct[c, 0, k], ct[c, 1, k]], [q0, q1])
            y = (X - _cent(X, q1)) // q1
            assert int(got[c, 0, k]) == y % q0
            # same thing as round(X / q1) on the centred integer (no ties: q1 odd)
            Xc = _cent(X, q0 * q1)
            assert (Xc - _cent(Xc, q1)) // q1 % q0 == y % q0


# ----------------------------------------------------------------------------- key switching
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


@pytest.mark.parametrize("zero_error,bound", [(True, None), (False, 2 ** 20)])
def test_relinearization_identity(O, zero_error, bound):
    """c0' + c1' s = d0 + d1 s + d2 s^2 + e (mod Q) with e the ModDown rounding term:
    |e| <= (N+1)/2 exactly for error-free keys; small for sigma = 3.2 keys."""
    logN = 5
    N = 32
    q0, q1, P = O.primes()
    sk, pk, rlk, gk = O.keygen(logN, 3, 0, zero_error=zero_error)
    rnd = random.Random(9)
    d = np.array([[[rnd.randrange(m) for _ in range(N)] for m in (q0, q1)] for _ in range(3)], np.uint64)
    out = O.relinearize(logN, d, rlk)
    Q = q0 * q1
    lift = lambda arr: [_crt([arr[0][k], arr[1][k]], [q0, q1]) for k in range(N)]
    s = [int(x) for x in sk]
    s2 = _negacyclic_big(s, s)
    D = [lift(d[i]) for i in range(3)]
    C = [lift(out[i]) for i in range(2)]
    lhs = [(C[0][k] + v) for k, v in enumerate(_negacyclic_big(C[1], s))]
    rhs_1 = _negacyclic_big(D[1], s)
    rhs_2 = _negacyclic_big(D[2], s2)
    e = [_cent(lhs[k] - D[0][k] - rhs_1[k] - rhs_2[k], Q) for k in range(N)]
    lim = (N + 1) // 2 if bound is None else bound
    assert max(abs(x) for x in e) <= lim
    # a plausible mistake (wrong gadget digit / sign) makes e of size ~Q: make sure e is not trivially 0
    assert any(x != 0 for x in e) or zero_error


def test_rotation_keyswitch_decrypts_to_rotated_slots(O):
    logN = 6
    S = 32
    q0 = O.primes()[0]
    sk, pk, rlk, gk = O.keygen(logN, 4, 3)
    z = np.random.default_rng(5).uniform(-1, 1, S)
    ct = O.encrypt(logN, pk, O.encode(z[None], logN), 0, 1)[0]
    # drop to level 0 by keeping the q0 limb (valid ciphertext mod q0 at scale Delta)
    ct0 = np.ascontiguousarray(ct[:, :1, :])
    for i, r in enumerate((1, 2, 4)):
        rot = O.rotate(logN, ct0, r, gk[i])
        m = O.decrypt(logN, sk, rot, 1)[0]
        back = O.decode_slots(O.centred_i64(m, q0), logN, O.DELTA)
        assert np.abs(back - _rot_left(z, r)).max() < 1e-6


# ----------------------------------------------------------------------------- exact level-0 key-switch identities
def _sigma_signed(a, g):
    """sigma_g on integer coefficients: X^k -> X^(k g mod 2N), negated past N (direct substitution)."""
    n = len(a)
    out = [0] * n
    for k, v in enumerate(a):
        t = k * g % (2 * n)
        if t < n:
            out[t] += v
        else:
            out[t - n] -= v
    return out


def _moddown_round(x_P, key_P, P):
    """y^ = centred_P(x key mod P): the ModDown rounding term, recomputed with big integers from the
    digit lifted to P and the key's P limb (SURVEY.md sec. 8c "Key switch" pin)."""
    return [_cent(v % P, P) for v in _negacyclic_big(x_P, key_P)]


@pytest.mark.parametrize("r", [1, 2, 4])
def test_rotate_level0_keyswitch_identity(O, r):
    """Level-0 rotation (reading R3: one digit x = sigma_g(c1) in [0, q0), lifted to P as is; Galois key
    over {q0, P}): with error-free keys, EXACTLY
        c0' + c1' s = sigma(c0) + sigma(c1) sigma(s) - P^-1 (y^_0 + y^_1 s)   (mod q0),
    y^_c = centred_P(x gk[c][P]) recomputed here from the key's P limb (big integers); |e| <= (N+1)/2.
    A dropped term, a wrong sign, the wrong Galois element or a centred lift all break the equality."""
    logN = 5
    N = 1 << logN
    q0, q1, P = O.primes()
    sk, pk, rlk, gk = O.keygen(logN, 3, 3, zero_error=True)
    g = pow(5, r, 2 * N)
    rnd = random.Random(31 + r)
    ct = np.array([[[rnd.randrange(q0) for _ in range(N)]] for _ in range(2)], np.uint64)
    out = O.rotate(logN, ct, r, gk[r.bit_length() - 1])
    s = [int(v) for v in sk]
    c0, c1 = [int(v) for v in ct[0, 0]], [int(v) for v in ct[1, 0]]
    x = [v % q0 for v in _sigma_signed(c1, g)]                    # the digit, canonical mod q0
    y0 = _moddown_round(x, [int(v) for v in gk[r.bit_length() - 1][0][1]], P)
    y1 = _moddown_round(x, [int(v) for v in gk[r.bit_length() - 1][1][1]], P)
    Pinv = pow(P, -1, q0)
    lhs = [(int(out[0, 0, k]) + v) % q0 for k, v in enumerate(_negacyclic_big([int(v) for v in out[1, 0]], s))]
    xs = _negacyclic_big(x, _sigma_signed(s, g))
    corr = [y0[k] + v for k, v in enumerate(_negacyclic_big(y1, s))]
    sc0 = _sigma_signed(c0, g)
    rhs = [(sc0[k] + xs[k] - Pinv * corr[k]) % q0 for k in range(N)]
    assert lhs == rhs
    e = [_cent((lhs[k] - sc0[k] - xs[k]) % q0, q0) for k in range(N)]
    assert max(abs(v) for v in e) <= (N + 1) // 2 and any(v != 0 for v in e)


@pytest.mark.parametrize("s_len", [2, 4, 8])
def test_hoisted_rot_sum_keyswitch_identity(O, s_len):
    """f2's hoisted rotation sum (reading R23): with error-free keys, EXACTLY
        o0 + o1 s = sum_{r<s} sigma_r(c0) + c1 s + sum_{0<r<s} sigma_r(c1) sigma_r(s)
                    - P^-1 (Y_0 + Y_1 s)   (mod q0),
    Y_c = centred_P(sum_{0<r<s} sigma_r(x~)_P hgk_r[c][P]) with the digit x = c1 in [0, q0) lifted to P
    ONCE and permuted in the P limb as a signed permutation (negation mod P), big integers."""
    logN = 5
    N = 1 << logN
    q0, q1, P = O.primes()
    sk, pk, rlk, gk = O.keygen(logN, 5, 0, zero_error=True)
    hgk = O.keygen_hoisted(logN, 5, s_len, zero_error=True)
    rnd = random.Random(40 + s_len)
    ct = np.array([[[rnd.randrange(q0) for _ in range(N)]] for _ in range(2)], np.uint64)
    out = O.hoisted_rot_sum(logN, s_len, hgk, ct)
    s = [int(v) for v in sk]
    c0, c1 = [int(v) for v in ct[0, 0]], [int(v) for v in ct[1, 0]]
    acc = [0] * N   # the Q-limb message part
    Y = [[0] * N, [0] * N]
    for r in range(s_len):
        g = pow(5, r, 2 * N)
        sc0 = _sigma_signed(c0, g)
        acc = [acc[k] + sc0[k] for k in range(N)]
        if r == 0:
            acc = [acc[k] + v for k, v in enumerate(_negacyclic_big(c1, s))]
            continue
        xg = _sigma_signed(c1, g)                           # sigma_r of the lifted digit (integers)
        ss = _negacyclic_big(xg, _sigma_signed(s, g))
        acc = [acc[k] + ss[k] for k in range(N)]
        for c in range(2):
            kp = [int(v) for v in hgk[r - 1][c][1]]
            prod = _negacyclic_big([v % P for v in xg], kp)
            Y[c] = [Y[c][k] + prod[k] for k in range(N)]
    Yc = [[_cent(v % P, P) for v in Y[c]] for c in range(2)]
    Pinv = pow(P, -1, q0)
    corr = [Yc[0][k] + v for k, v in enumerate(_negacyclic_big(Yc[1], s))]
    lhs = [(int(out[0, 0, k]) + v) % q0 for k, v in enumerate(_negacyclic_big([int(v) for v in out[1, 0]], s))]
    rhs = [(acc[k] - Pinv * corr[k]) % q0 for k in range(N)]
    assert lhs == rhs
    e = [_cent((lhs[k] - acc[k]) % q0, q0) for k in range(N)]
    assert max(abs(v) for v in e) <= (N + 1) // 2 and any(v != 0 for v in e)


# ----------------------------------------------------------------------------- trivial-ciphertext closed form
def _trivial(pt_list, q0, q1, N):
    """(pt, 0) as a level-1 ciphertext."""
    ct = np.zeros((len(pt_list), 2, 2, N), np.uint64)
    for i, pt in enumerate(pt_list):
        ct[i, 0, 0] = [int(v) % q0 for v in pt]
        ct[i, 0, 1] = [int(v) % q1 for v in pt]
    return ct


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


@pytest.mark.parametrize("order", [0, 1, 2])
def test_trivial_ciphertext_scan_closed_form(O, order):
    """With c1 = 0 every key switch vanishes, so HE-C^3 reduces to integer arithmetic:
    hoisted:  C = round(sum_i pt_u,i * pt_s,i / q1) mod q0   (orders 0 and 2)
    paper:    C = sum_i round(pt_u,i * pt_s,i / q1) mod q0
    then      out = sum_{delta < s} sigma_{5^delta}(C) mod q0      (the ladder's
    doubling steps and the f2 hoisted rotation sum both add every rotation delta < s once)"""
    logN, d, p = 6, 16, 2              # N = 64, S = 32, s = 8, B = 4
    N = 1 << logN
    q0, q1, P = O.primes()
    s = d // p
    sk, pk, rlk, gk = O.keygen(logN, 6, O.n_rot_for(d, p))
    if order == 2:
        gk = O.keygen_hoisted(logN, 6, s)
    rnd = random.Random(11)
    pu = [[rnd.randrange(-2 ** 40, 2 ** 40) for _ in range(N)] for _ in range(p)]
    ps = [[rnd.randrange(-2 ** 40, 2 ** 40) for _ in range(N)] for _ in range(p)]
    qct = _trivial(pu, q0, q1, N)[None]
    sct = _trivial(ps, q0, q1, N)[None]
    out, _ = O.match(logN, d, p, order, rlk, gk, sct, qct)

    def rnd_div(x, m):  # (X - c_m(X)) / m, the rescale rounding on true integers (|X| < Q/2)
        return (x - _cent(x, m)) // m

    prods = [_negacyclic_big(pu[i], ps[i]) for i in range(p)]
    if order in (0, 2):
        tot = [sum(pr[k] for pr in prods) for k in range(N)]
        C = [rnd_div(v, q1) for v in tot]
    else:
        C = [sum(rnd_div(pr[k], q1) for pr in prods) for k in range(N)]
    acc = [0] * N
    for delta in range(s):
        sg = _sigma_int(C, pow(5, delta, 2 * N))
        acc = [a + b for a, b in zip(acc, sg)]
    exp = [v % q0 for v in acc]
    assert [int(x) for x in out[0, 0, 0]] == exp
    assert not out[0, 1].any()


# ----------------------------------------------------------------------------- f2: hoisted rotation sum
def test_hoisted_rotation_sum_decrypts_to_window_sums(O):
    """f2: sum_{r<s} Rot(ct, r) with one hoisted key switch decrypts to the sum of
    the s left rotations of the slots (SPEC.md:82 rotation semantics), for s = 1, 2, 8."""
    logN = 6
    S = 32
    q0 = O.primes()[0]
    sk, pk, rlk, gk = O.keygen(logN, 4, 3)
    z = np.random.default_rng(7).uniform(-1, 1, S)
    ct = O.encrypt(logN, pk, O.encode(z[None], logN), 0, 1)[0]
    ct0 = np.ascontiguousarray(ct[:, :1, :])
    for s in (1, 2, 8):
        hgk = O.keygen_hoisted(logN, 4, s)
        out = O.hoisted_rot_sum(logN, s, hgk, ct0)
        m = O.decrypt(logN, sk, out, 1)[0]
        back = O.decode_slots(O.centred_i64(m, q0), logN, O.DELTA)
        want = sum(_rot_left(z, r) for r in range(s))
        assert np.abs(back - want).max() < 1e-6, s
    if True:  # s = 1 is the identity (no key switch at all)
        assert np.array_equal(O.hoisted_rot_sum(logN, 1, O.keygen_hoisted(logN, 4, 1), ct0), ct0)


def test_bsgs_rotation_sum_decrypts_to_window_sums(O):
    """f2 baby-step giant-step sum (b = 2^ceil(log2 s / 2) baby rotations, g = s / b giant ones, each a
    hoisted key switch) decrypts to the sum of the s left rotations of the slots, s = 2..32
    (s = 2: b = 2, g = 1 -- the plain hoisted sum, bit for bit)."""
    logN = 6
    S = 32
    q0 = O.primes()[0]
    sk, pk, rlk, gk = O.keygen(logN, 4, 3)
    z = np.random.default_rng(8).uniform(-1, 1, S)
    ct = O.encrypt(logN, pk, O.encode(z[None], logN), 0, 1)[0]
    ct0 = np.ascontiguousarray(ct[:, :1, :])
    for s in (2, 4, 8, 16, 32):
        hgk = O.keygen_hoisted(logN, 4, s)
        out = O.bsgs_rot_sum(logN, s, hgk, ct0)
        m = O.decrypt(logN, sk, out, 1)[0]
        back = O.decode_slots(O.centred_i64(m, q0), logN, O.DELTA)
        want = sum(_rot_left(z, r) for r in range(s))
        assert np.abs(back - want).max() < 1e-6, s
        if s == 2:
            assert np.array_equal(out, O.hoisted_rot_sum(logN, s, hgk, ct0))
        else:
            assert not np.array_equal(out, O.hoisted_rot_sum(logN, s, hgk, ct0))


@pytest.mark.parametrize("s_len", [4, 8, 16])
def test_bsgs_rotation_sum_exact_error_bound(O, s_len):
    """With error-free keys the baby-step giant-step sum is the window sum of the decryption up to the
    two ModDowns' rounding: o0 + o1 s - sum_{r<s} sigma_r(c0 + c1 s) = g e_b' + e_g with every
    |coefficient| <= (g + 1)(N + 1)/2 (each hoisted ModDown adds |e| <= (N + 1)/2, the baby one is
    rotated g times), big integers, random level-0 ciphertext.  A wrong key (amount, index) or a wrong
    giant stride leaves an error of order q0."""
    logN = 5
    N = 1 << logN
    q0 = O.primes()[0]
    sk, pk, rlk, gk = O.keygen(logN, 6, 0, zero_error=True)
    hgk = O.keygen_hoisted(logN, 6, s_len, zero_error=True)
    rnd = random.Random(90 + s_len)
    ct = np.array([[[rnd.randrange(q0) for _ in range(N)]] for _ in range(2)], np.uint64)
    out = O.bsgs_rot_sum(logN, s_len, hgk, ct)
    sv = [int(v) for v in sk]
    m = [int(a) + b for a, b in zip(ct[0, 0], _negacyclic_big([int(v) for v in ct[1, 0]], sv))]
    want = [0] * N
    for r in range(s_len):
        want = [a + b for a, b in zip(want, _sigma_signed(m, pow(5, r, 2 * N)))]
    got = [int(a) + b for a, b in zip(out[0, 0], _negacyclic_big([int(v) for v in out[1, 0]], sv))]
    e = [_cent((x - y) % q0, q0) for x, y in zip(got, want)]
    log_s = s_len.bit_length() - 1
    g = s_len // (1 << ((log_s + 1) // 2))
    assert max(abs(v) for v in e) <= (g + 1) * (N + 1) // 2 and any(v != 0 for v in e)


def test_hoisted_keys_are_galois_keys_of_their_rotation(O):
    """hgk[r-1] satisfies the Galois-key relation of rotation r: with zero-error keys,
    b + a s = (P mod q0) sigma_{5^r}(s) in q0 and 0 in P -- an independent big-integer check of the
    key generator (a wrong rotation amount, limb or sign fails it)."""
    logN = 5
    N = 1 << logN
    q0, q1, P = O.primes()
    sk, pk, rlk, gk = O.keygen(logN, 9, 2)
    hgk = O.keygen_hoisted(logN, 9, 6, zero_error=True)
    s_int = [int(v) for v in sk]
    for r in range(1, 6):
        g = pow(5, r, 2 * N)
        ss = _sigma_int(s_int, g)
        for li, q in ((0, q0), (1, P)):
            b = [int(v) for v in hgk[r - 1, 0, li]]
            a = [int(v) for v in hgk[r - 1, 1, li]]
            asum = _negacyclic_big(a, s_int)
            lhs = [(b[k] + asum[k]) % q for k in range(N)]
            rhs = [((P % q0) * ss[k]) % q if li == 0 else 0 for k in range(N)]
            assert lhs == rhs, (r, li)


# ----------------------------------------------------------------------------- end to end
def _run_scan(O, logN, d, p, tmpl, qv, order=0, key_seed=1, n_threads=4):
    S, s, B = O.layout(logN, d, p)
    n_sets = -(-tmpl.shape[0] // B)
    sk, pk, rlk, gk = O.keygen(logN, key_seed, O.n_rot_for(d, p))
    if order == 2:
        gk = O.keygen_hoisted(logN, key_seed, s)
    zdb = O.pack_db(tmpl, logN, d, p, 0, n_sets)
    zq = O.pack_query(qv, logN, d, p)
    db = O.encrypt(logN, pk, O.encode(zdb.reshape(-1, S), logN), 0, 2).reshape(n_sets, p, 2, 2, -1)
    qc = O.encrypt(logN, pk, O.encode(zq.reshape(-1, S), logN), 0, 3).reshape(len(qv), p, 2, 2, -1)
    out, pairs = O.match(logN, d, p, order, rlk, gk, db, qc, n_threads=n_threads)
    q0 = O.primes()[0]
    scores = np.zeros((len(qv), n_sets * B))
    for i, (j, t) in enumerate(pairs):
        scores[j, t * B:(t + 1) * B] = O.scores_from_output(logN, d, p, sk, out[i], q0)
    return scores[:, :tmpl.shape[0]], out


def test_config1_end_to_end(O):
    """BASELINE.json configs[0]: d=16, p=1, 256 templates, query = T[17] + noise -> top-1 17."""
    T = I.templates(1)
    Q, exp = I.queries(1)
    sc, _ = _run_scan(O, 13, 16, 1, T, Q)
    ref = Q @ T.T
    assert np.abs(sc - ref).max() < 1e-6      # internal guard (north_star contract: 1e-4)
    assert sc.argmax() == ref.argmax() == 17


def test_config1_end_to_end_hoisted_rotations(O):
    """configs[0] through the f2 order (hoisted rotation sum): same scores within 1e-6, top-1 17."""
    T = I.templates(1)
    Q, exp = I.queries(1)
    sc, _ = _run_scan(O, 13, 16, 1, T, Q, order=2)
    ref = Q @ T.T
    assert np.abs(sc - ref).max() < 1e-6
    assert sc.argmax() == 17


def test_orders_coincide_for_p1_and_agree_in_value(O):
    logN, d = 8, 8                          # N = 256, S = 128
    T = I.random_unit(40, d, 1)
    Q = I.random_unit(2, d, 2)
    a, oa = _run_scan(O, logN, d, 1, T, Q, order=0)
    b, ob = _run_scan(O, logN, d, 1, T, Q, order=1)
    assert np.array_equal(oa, ob)           # p = 1: one relin + rescale either way
    c, oc = _run_scan(O, logN, d, 4, T, Q, order=0)
    e, oe = _run_scan(O, logN, d, 4, T, Q, order=1)
    ref = Q @ T.T
    for x in (a, c, e):
        assert np.abs(x - ref).max() < 1e-6
    assert not np.array_equal(oc, oe)       # residues differ across orders (reading R8)


def _spec():
    with open(GOLD) as f:
        return json.load(f)


def test_spec_layout_examples(O):
    g = _spec()
    lay = g["layout"]
    S, s, B = O.layout(4, lay["m"], lay["N_in"])
    assert (S, s, B) == (lay["S"], lay["s"], lay["B"])
    en = g["enroll"]
    tm = np.zeros((2, 4))
    tm[en["index"]] = en["vector"]
    z = O.pack_db(tm, 4, 4, 2, 0, 1)[0]
    assert np.allclose(z[0], en["ct0"]) and np.allclose(z[1], en["ct1"])
    ex = g["expand"]
    w = O.pack_query(np.array([ex["query"]]), 4, 4, 2)[0]
    assert np.allclose(w[0], ex["out0"]) and np.allclose(w[1], ex["out1"])
    pc = g["paper_capacity"]
    assert pc["paper_slots"] * pc["N_in"] // pc["m"] == pc["B_paper"]
    # reading R1: standard ring, S = N/2 slots -> half the paper's capacity
    assert O.layout(13, pc["m"], pc["N_in"])[2] == pc["B_paper"] // 2


def test_spec_match_example_N16(O):
    g = _spec()["match"]
    T = np.array(g["enrolled"], np.float64)
    Q = np.array([g["query"]], np.float64)
    sc, out = _run_scan(O, 4, 4, 2, T, Q)
    # slot 0 = block 0 (template 0), slot 2 = block 1 (template 1)
    assert abs(sc[0, 0] - g["slot0"]) < 1e-6 and abs(sc[0, 1] - g["slot2"]) < 1e-6


# ----------------------------------------------------------------------------- f2: relin-free degree-2 output
def test_deg2_scan_big_integer_closed_form(O):
    """f2's relin-free output for p = d: per pair, every component of
    sum_i tensor(C_u,i, C_s,i) rescaled by q1.  Recomputed here with big integers on random (not
    trivial) ciphertexts: per limb the negacyclic products summed over the parts (Karatsuba-free
    schoolbook d0 = sum a0 b0, d1 = sum a0 b1 + a1 b0, d2 = sum a1 b1), the CRT lift of the two limbs,
    and (X - centred_q1(X)) / q1 mod q0."""
    logN, d = 4, 4
    p = d
    N = 1 << logN
    q0, q1, P = O.primes()
    rnd = random.Random(71)
    ct = lambda: np.array([[[[rnd.randrange(m) for _ in range(N)] for m in (q0, q1)] for _ in range(2)]
                           for _ in range(p)], np.uint64)
    qct, sct = ct()[None], ct()[None]
    out, _ = O.match_deg2(logN, d, p, sct, qct)
    for comp, terms in ((0, [(0, 0)]), (1, [(0, 1), (1, 0)]), (2, [(1, 1)])):
        lim = []
        for li, m in enumerate((q0, q1)):
            acc = [0] * N
            for i in range(p):
                for a, b in terms:
                    pr = _negacyclic_big([int(v) for v in qct[0, i, a, li]], [int(v) for v in sct[0, i, b, li]])
                    acc = [x + y for x, y in zip(acc, pr)]
            lim.append([v % m for v in acc])
        X = [_crt([lim[0][k], lim[1][k]], [q0, q1]) for k in range(N)]
        exp = [((x - _cent(x, q1)) // q1) % q0 for x in X]
        assert [int(v) for v in out[0, comp, 0]] == exp, comp


def test_deg2_scan_decrypts_with_s_squared(O):
    """The degree-2 output decrypts with (1, s, s^2) to the cosines of every template (s = 1: every
    slot is a score, B = 4096) at N = 8192; top-1 is the genuine template.  Tolerance 1e-5 (north_star
    contract 1e-4): unlike the relinearised output, the rounding of the third component's rescale is
    multiplied by s^2 (dense ternary s: coefficients of s^2 ~ sqrt(2N/3) ~ 74), a slot error of
    sigma ~ sqrt(N) 0.29 74 sqrt(N) / 2^40 ~ 1.6e-7 (f2 degree-2 output)."""
    logN, d = 13, 16
    p = d
    T = I.random_unit(300, d, 72)
    q = T[123] + 0.05 * np.random.default_rng(73).standard_normal(d)
    Q = (q / np.linalg.norm(q))[None]
    S, s, B = O.layout(logN, d, p)
    sk, pk, rlk, gk = O.keygen(logN, 1, 0)
    db = O.encrypt(logN, pk, O.encode(O.pack_db(T, logN, d, p, 0, 1).reshape(-1, S), logN), 0, 2).reshape(1, p, 2, 2, -1)
    qc = O.encrypt(logN, pk, O.encode(O.pack_query(Q, logN, d, p).reshape(-1, S), logN), 0, 3).reshape(1, p, 2, 2, -1)
    out, _ = O.match_deg2(logN, d, p, db, qc)
    q0, q1, P = O.primes()
    m = O.decrypt_deg2(logN, sk, out[0].reshape(3, -1))
    slots = O.decode_slots(O.centred_i64(m, q0), logN, 2.0 ** 80 / q1)
    sc = slots[:T.shape[0]]
    assert np.abs(sc - T @ Q[0]).max() < 1e-5
    assert int(np.argmax(sc)) == 123
