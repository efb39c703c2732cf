"""Pins for the oracle's f3 row: server-side query expansion, Algorithm 1
"Input Ciphertext Expansion", on the prime chain extended by one 40-bit
prime q2 (readings R24-R26).

Pins used (each independent of the oracle code path it checks):
  * q2: an independent Miller-Rabin in Python; every NTT-friendly candidate between q2 and q1
    is composite; log2(q0 q1 q2 P) stays below the 218-bit bound
  * keys: b + a s = e small (public key limb q2, same error as pk); the level-1 Galois keys
    satisfy the gadget relation of their rotation exactly (big integers, zero-error keys)
  * Mul(P) + Res by q2: Python big-integer closed form on the CRT lift over {q0, q1, q2}
  * level-1 rotation: the key-switch identity c0' + c1' s = sigma(c0) + sigma(c1) sigma(s) + e,
    |e| <= (N+1)/2 for error-free keys; decryption equals the left-rotated slots
  * trivial ciphertexts (c1 = 0): the whole expansion equals a big-integer closed form
  * decryption of every expanded part equals SPEC.md:297's post-condition w_i[x] = q[i s + x mod s]
  * SPEC.md:300's worked example (S = 8, m = 4, N_in = 2) in real CKKS at N = 16
  * end to end: expanded queries through HE-C^3 give the plaintext cosines and top-1
f4 (server-side enrollment packing, Fig. 3 / PAPER.md:251-269, same chain; reading R27):
  * trivial ciphertexts: every set part equals a big-integer closed form (signed permutations
    of round(E_i pt / q2) by the right rotations (k - i) s)
  * SPEC.md:291's worked example at N = 16; decryption equals the client-side packing layout
     for two sets covering every rotation amount; the enrolled DB scans to the
    plaintext cosines and top-1
"""
import json
import os
import random

import numpy as np
import pytest

from paper_2408_06167_b200 import inputs as I

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")


def _mr_prime(n):
    """Deterministic Miller-Rabin for n < 3.3e24 (bases 2..41), written here independently."""
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)
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


def _rot_left(z, r):
    return np.roll(z, -r, axis=-1)


# ----------------------------------------------------------------------------- the extra prime
def test_q2_is_the_next_ntt_prime_below_q1(O):
    q0, q1, P = O.primes()
    q2 = O.q2()
    assert q2 == 1099510890497 == 2 ** 40 - 45 * 2 ** 14 + 1
    assert _mr_prime(q2) and q2 % 16384 == 1 and q2 < q1
    for k in range(1, (q1 - q2) // 16384):           # every candidate strictly between is composite
        assert not _mr_prime(q1 - k * 16384)
    bits = (q0 * q1 * q2 * P).bit_length()
    assert bits == 198 and bits <= 218                 # SPEC.md:159 bound at N = 8192
    assert O.find_prime_below(q1, 16384) == q2


# ----------------------------------------------------------------------------- keys
def test_level2_public_key_limb(O):
    """pk_q2 = (b, a) with b + a s = e mod q2, e the SAME small error as pk's q0/q1 limbs."""
    logN = 6
    N = 1 << logN
    q0 = O.primes()[0]
    q2 = O.q2()
    sk, pk, rlk, gk = O.keygen(logN, 5, 0)
    pk_q2, _ = O.keygen_exp(logN, 5, 8, 2)
    s = [int(v) for v in sk]
    e2 = [_cent(int(b) + x, q2) for b, x in zip(pk_q2[0], _negacyclic_big([int(v) for v in pk_q2[1]], s))]
    e0 = [_cent(int(b) + x, q0) for b, x in zip(pk[0, 0], _negacyclic_big([int(v) for v in pk[1, 0]], s))]
    assert max(abs(v) for v in e2) <= 19 and e2 == e0
    assert len(set(int(v) for v in pk_q2[1])) > N // 2   # a is uniform, not a copy of a small poly


def test_level1_galois_keys_relation(O):
    """gk1[t][j]: b + a s = [l = j] (P mod q_l) sigma_{5^(s 2^t)}(s) in limb q_l and 0 in limb P,
    exactly, for error-free keys (a wrong rotation, digit, limb or sign fails it)."""
    logN, d, p = 5, 16, 4
    N = 1 << logN
    q0, q1, P = O.primes()
    sk, pk, rlk, gk = O.keygen(logN, 9, 0)
    _, gk1 = O.keygen_exp(logN, 9, d, p, zero_error=True)
    assert gk1.shape[:4] == (2, 2, 2, 3)
    s_int = [int(v) for v in sk]
    for t in range(2):
        g = pow(5, (d // p) << t, 2 * N)
        ss = _sigma_int(s_int, g)
        for j in range(2):
            for l, q in enumerate((q0, q1, P)):
                b = [int(v) for v in gk1[t, j, 0, l]]
                asum = _negacyclic_big([int(v) for v in gk1[t, j, 1, l]], s_int)
                lhs = [(b[k] + asum[k]) % q for k in range(N)]
                rhs = [((P % q) * ss[k]) % q if l == j else 0 for k in range(N)]
                assert lhs == rhs, (t, j, l)


# ----------------------------------------------------------------------------- enc / Mul(P) + Res
def test_encrypt_l2_extends_level1_encryption_and_decrypts(O):
    logN = 13
    S = 4096
    q0 = O.primes()[0]
    sk, pk, rlk, gk = O.keygen(logN, 1, 0)
    pk_q2, _ = O.keygen_exp(logN, 1, 128, 8)
    z = np.random.default_rng(4).uniform(-1, 1, (2, S))
    pt = O.encode(z, logN)
    c2 = O.encrypt_l2(logN, pk, pk_q2, pt, 7, 9)
    c1 = O.encrypt(logN, pk, pt, 7, 9)
    assert np.array_equal(c2[:, :, :2, :], c1)         # same streams: level 2 = level 1 + one limb
    for i in range(2):
        m = O.decrypt_l2(logN, sk, c2[i])
        for l, q in ((0, q0), (2, O.q2())):
            back = O.decode_slots(O.centred_i64(m[l], q), logN, O.DELTA)
            assert np.abs(back - z[i]).max() < 1e-6


def test_mul_plain_rescale_q2_closed_form(O):
    """Res(Mul(P)(ct, pt)) = (T - c_{q2}(T)) / q2 mod q_k, T = CRT lift over {q0,q1,q2} of ct * pt."""
    logN = 4
    N = 16
    q0, q1, P = O.primes()
    q2 = O.q2()
    mods = (q0, q1, q2)
    Q2 = q0 * q1 * q2
    rnd = random.Random(21)
    ct = np.array([[[rnd.randrange(m) for _ in range(N)] for m in mods] for _ in range(2)], np.uint64)
    pt = [rnd.randrange(-2 ** 45, 2 ** 45) for _ in range(N)]
    got = O.mul_plain_rescale_q2(logN, ct, np.array(pt, np.int64))
    for c in range(2):
        X = [_crt([ct[c, 0, k], ct[c, 1, k], ct[c, 2, k]], mods) for k in range(N)]
        T = [v % Q2 for v in _negacyclic_big(X, pt)]
        for k in range(N):
            y = (T[k] - _cent(T[k], q2)) // q2
            assert (T[k] - _cent(T[k], q2)) % q2 == 0
            assert int(got[c, 0, k]) == y % q0 and int(got[c, 1, k]) == y % q1


# ----------------------------------------------------------------------------- level-1 rotation
def test_rotate1_keyswitch_identity(O):
    """c0' + c1' s = sigma(c0) + sigma(c1) sigma(s) + e (mod q0 q1), |e| <= (N+1)/2 with
    error-free keys (e = -(y0 + y1 s)/P, the ModDown rounding), e != 0 somewhere."""
    logN, d, p = 5, 16, 2
    N = 1 << logN
    q0, q1, P = O.primes()
    Q = q0 * q1
    sk, pk, rlk, gk = O.keygen(logN, 3, 0)
    _, gk1 = O.keygen_exp(logN, 3, d, p, zero_error=True)
    r = d // p
    g = pow(5, r, 2 * N)
    rnd = random.Random(23)
    ct = np.array([[[rnd.randrange(m) for _ in range(N)] for m in (q0, q1)] for _ in range(2)], np.uint64)
    out = O.rotate1(logN, ct, r, gk1[0])
    lift = lambda arr: [_crt([arr[0][k], arr[1][k]], [q0, q1]) for k in range(N)]
    s = [int(v) for v in sk]
    C0, C1 = lift(out[0]), lift(out[1])
    A0, A1 = _sigma_int(lift(ct[0]), g), _sigma_int(lift(ct[1]), g)
    lhs = [C0[k] + v for k, v in enumerate(_negacyclic_big(C1, s))]
    rhs = [A0[k] + v for k, v in enumerate(_negacyclic_big(A1, _sigma_int(s, g)))]
    e = [_cent(lhs[k] - rhs[k], Q) for k in range(N)]
    assert max(abs(v) for v in e) <= (N + 1) // 2
    assert any(v != 0 for v in e)


def test_rotate1_decrypts_to_rotated_slots(O):
    logN = 6
    S = 32
    q0 = O.primes()[0]
    d, p = 8, 4                                          # rotations by s 2^t = 2, 4
    sk, pk, rlk, gk = O.keygen(logN, 4, 0)
    pk_q2, gk1 = O.keygen_exp(logN, 4, d, p)
    z = np.random.default_rng(5).uniform(-1, 1, S)
    ct = O.encrypt(logN, pk, O.encode(z[None], logN), 0, 1)[0]
    for t in range(2):
        r = (d // p) << t
        rot = O.rotate1(logN, ct, r, gk1[t])
        m = O.decrypt(logN, sk, rot, 2)
        back = O.decode_slots(O.centred_i64(m[0], q0), logN, O.DELTA)
        assert np.abs(back - _rot_left(z, r)).max() < 1e-6


# ----------------------------------------------------------------------------- Algorithm 1
def _trivial_l2(pt, mods, N):
    ct = np.zeros((2, 3, N), np.uint64)
    for l, m in enumerate(mods):
        ct[0, l] = [int(v) % m for v in pt]
    return ct


@pytest.mark.parametrize("p", [1, 2, 4])
def test_trivial_expansion_closed_form(O, p):
    """With c1 = 0 every key switch vanishes: part i = sum_{u < p} sigma_{5^(s u)}(round(X_i pt / q2))
    mod q_k (the doubling ladder adds every stride s u once), c1 = 0."""
    logN, d = 6, 16
    N = 1 << logN
    s = d // p
    q0, q1, P = O.primes()
    q2 = O.q2()
    sk, pk, rlk, gk = O.keygen(logN, 6, 0)
    _, gk1 = O.keygen_exp(logN, 6, d, p)
    rnd = random.Random(30 + p)
    pt = [rnd.randrange(-2 ** 40, 2 ** 40) for _ in range(N)]
    masks = np.array([[rnd.randrange(-2 ** 40, 2 ** 40) for _ in range(N)] for _ in range(p)], np.int64)
    out = O.expand(logN, d, p, masks, gk1, _trivial_l2(pt, (q0, q1, q2), N))[0]
    for i in range(p):
        prod = _negacyclic_big([int(v) for v in masks[i]], pt)
        C = [(v - _cent(v, q2)) // q2 for v in prod]
        acc = [0] * N
        for u in range(p):
            acc = [a + b for a, b in zip(acc, _sigma_int(C, pow(5, s * u, 2 * N)))]
        assert [int(v) for v in out[i, 0, 0]] == [v % q0 for v in acc], i
        assert [int(v) for v in out[i, 0, 1]] == [v % q1 for v in acc], i
        assert not out[i, 1].any()


def test_p1_expansion_is_mask_and_rescale_only(O):
    """N_in = 1: the single output is the masked, rescaled input, no rotation."""
    logN, d = 6, 8
    sk, pk, rlk, gk = O.keygen(logN, 2, 0)
    pk_q2, gk1 = O.keygen_exp(logN, 2, d, 1)
    assert len(gk1) == 0
    masks = O.expand_masks(logN, d, 1)
    z = O.tile_query(I.random_unit(1, d, 3), logN, d)
    ct = O.encrypt_l2(logN, pk, pk_q2, O.encode(z, logN), 0, 3)
    out = O.expand(logN, d, 1, masks, gk1, ct)
    assert np.array_equal(out[0, 0], O.mul_plain_rescale_q2(logN, ct[0], masks[0]))


def _expand_and_decrypt(O, logN, d, p, qv, key_seed=1):
    sk, pk, rlk, gk = O.keygen(logN, key_seed, 0)
    pk_q2, gk1 = O.keygen_exp(logN, key_seed, d, p)
    masks = O.expand_masks(logN, d, p)
    ct = O.encrypt_l2(logN, pk, pk_q2, O.encode(O.tile_query(qv, logN, d), logN), 0, 3)
    out = O.expand(logN, d, p, masks, gk1, ct)
    q0 = O.primes()[0]
    z = np.zeros((len(qv), p, (1 << logN) // 2))
    for j in range(len(qv)):
        for i in range(p):
            m = O.decrypt(logN, sk, out[j, i], 2)
            z[j, i] = O.decode_slots(O.centred_i64(m[0], q0), logN, O.DELTA)
    return z, out


@pytest.mark.parametrize("d,p", [(128, 8), (32, 4)])
def test_expansion_meets_spec_postcondition(O, d, p):
    """part i decrypts (at scale exactly 2^40) to w_i[x] = q[i s + (x mod s)]."""
    qv = I.random_unit(1, d, 40 + p)
    z, _ = _expand_and_decrypt(O, 13, d, p, qv)
    want = O.pack_query(qv, 13, d, p)
    assert np.abs(z - want).max() < 1e-6


def test_spec_expand_example_N16(O):
    ex = json.load(open(GOLD))["expand"]
    z, _ = _expand_and_decrypt(O, 4, 4, 2, np.array([ex["query"]]))
    assert np.abs(z[0, 0] - ex["out0"]).max() < 1e-6
    assert np.abs(z[0, 1] - ex["out1"]).max() < 1e-6


def test_expanded_queries_through_he_c3(O):
    """configs[0]'s data with p = 4 (s = 4): Enc_l2(tiled query) -> Algorithm 1 -> Algorithm 2 gives
    the plaintext cosines (internal guard 1e-6; north_star 1e-4) and top-1 = 17."""
    logN, d, p = 13, 16, 4
    T = I.templates(1)
    Q, _ = I.queries(1)
    S, s, B = O.layout(logN, d, p)
    n_sets = -(-T.shape[0] // B)
    sk, pk, rlk, gk = O.keygen(logN, 1, O.n_rot_for(d, p))
    pk_q2, gk1 = O.keygen_exp(logN, 1, d, p)
    zdb = O.pack_db(T, logN, d, p, 0, n_sets)
    db = O.encrypt(logN, pk, O.encode(zdb.reshape(-1, S), logN), 0, 2).reshape(n_sets, p, 2, 2, -1)
    ct = O.encrypt_l2(logN, pk, pk_q2, O.encode(O.tile_query(Q, logN, d), logN), 0, 3)
    qx = O.expand(logN, d, p, O.expand_masks(logN, d, p), gk1, ct)
    out, pairs = O.match(logN, d, p, 0, rlk, gk, db, qx, n_threads=4)
    q0 = O.primes()[0]
    sc = np.concatenate([O.scores_from_output(logN, d, p, sk, out[i], q0) for i in range(len(pairs))])
    sc = sc[:T.shape[0]]
    ref = (Q @ T.T)[0]
    assert np.abs(sc - ref).max() < 1e-6
    assert sc.argmax() == ref.argmax() == 17


# ----------------------------------------------------------------------------- f4: server-side enrollment
def test_enrollment_keys_extend_the_expansion_keys(O):
    """The enrollment's log2 B strides s 2^t include the expansion's log2 p ones (same objects)."""
    logN, d, p = 6, 16, 4
    _, g_exp = O.keygen_exp(logN, 7, d, p)
    nb = O.n_rot_enroll(logN, d, p)
    _, g_enr = O.keygen_exp(logN, 7, d, p, n_rot=nb)
    assert nb == 3 and g_enr.shape[0] == nb and np.array_equal(g_enr[:g_exp.shape[0]], g_exp)


@pytest.mark.parametrize("first_u,n", [(0, 3), (5, 6)])
def test_trivial_enrollment_closed_form(O, first_u, n):
    """With c1 = 0 the key switches vanish: set[t][i] = sum over its templates u = tB + k of
    sigma_{5^(s m)}(round(E_i pt_u / q2)), m = (i - k) mod B (a right rotation by (k - i) s)."""
    logN, d, p = 5, 8, 2                  # N = 32, S = 16, s = 4, B = 4
    N = 1 << logN
    S, s, B = O.layout(logN, d, p)
    q0, q1, P = O.primes()
    q2 = O.q2()
    _, gk1 = O.keygen_exp(logN, 8, d, p, n_rot=O.n_rot_enroll(logN, d, p))
    rnd = random.Random(50 + first_u)
    pts = [[rnd.randrange(-2 ** 40, 2 ** 40) for _ in range(N)] for _ in range(n)]
    em = np.array([[rnd.randrange(-2 ** 40, 2 ** 40) for _ in range(N)] for _ in range(p)], np.int64)
    n_sets = -(-(first_u + n) // B)
    db = np.zeros((n_sets, p, 2, 2, N), np.uint64)
    ct = np.stack([_trivial_l2(pt, (q0, q1, q2), N) for pt in pts])
    O.enroll(logN, d, p, em, gk1, ct, first_u, db)
    for t in range(n_sets):
        for i in range(p):
            acc = [0] * N
            for c in range(n):
                u = first_u + c
                if u // B != t:
                    continue
                m = (i - u % B) % B
                C = [(v - _cent(v, q2)) // q2 for v in _negacyclic_big([int(x) for x in em[i]], pts[c])]
                acc = [a + b for a, b in zip(acc, _sigma_int(C, pow(5, s * m, 2 * N)))]
            assert [int(v) for v in db[t, i, 0, 0]] == [v % q0 for v in acc]
            assert [int(v) for v in db[t, i, 0, 1]] == [v % q1 for v in acc]
            assert not db[t, i, 1].any()


def _enroll_and_decrypt(O, logN, d, p, T, first_u=0, key_seed=1):
    S, s, B = O.layout(logN, d, p)
    sk, pk, rlk, gk = O.keygen(logN, key_seed, O.n_rot_for(d, p))
    pk_q2, gk1 = O.keygen_exp(logN, key_seed, d, p, n_rot=O.n_rot_enroll(logN, d, p))
    ct = O.encrypt_l2(logN, pk, pk_q2, O.encode(O.enroll_vector(T, logN, d), logN), first_u, 5)
    n_sets = -(-(first_u + len(T)) // B)
    db = np.zeros((n_sets, p, 2, 2, 1 << logN), np.uint64)
    O.enroll(logN, d, p, O.enroll_masks(logN, d, p), gk1, ct, first_u, db)
    q0 = O.primes()[0]
    z = np.zeros((n_sets, p, S))
    for t in range(n_sets):
        for i in range(p):
            m = O.decrypt(logN, sk, db[t, i], 2)
            z[t, i] = O.decode_slots(O.centred_i64(m[0], q0), logN, O.DELTA)
    return z, db, (sk, pk, rlk, gk)


def test_spec_enroll_example_N16(O):
    """S = 8, m = 4, N_in = 2, enroll [a,b,c,d] at index 1 -> store ct 0 = [0,0,a,b,0,0,0,0],
    ct 1 = [0,0,c,d,0,0,0,0], in real CKKS at N = 16."""
    en = json.load(open(GOLD))["enroll"]
    z, _, _ = _enroll_and_decrypt(O, 4, 4, 2, np.array([en["vector"]]), first_u=en["index"])
    assert np.abs(z[0, 0] - en["ct0"]).max() < 1e-6
    assert np.abs(z[0, 1] - en["ct1"]).max() < 1e-6


def test_enrollment_meets_the_packing_layout(O):
    """SPEC.md:282-289 post-condition: after enrolling templates 0..n-1, set t part i decrypts to the
    client-side packing (template u = tB + k at slots k s .. k s + s - 1 of part i), two sets, the
    second partial (N = 256, d = 16, p = 4: s = 4, B = 32, every rotation amount m < 32 occurs)."""
    logN, d, p = 8, 16, 4
    T = I.random_unit(45, d, 9)
    z, _, _ = _enroll_and_decrypt(O, logN, d, p, T)
    want = O.pack_db(T, logN, d, p, 0, z.shape[0])
    assert np.abs(z - want).max() < 1e-6


def test_server_enrolled_db_scans_to_cosines(O):
    """f4 enrollment + Algorithm 2: the server-packed DB gives the plaintext cosines (1e-6) and top-1."""
    logN, d, p = 9, 16, 4
    T = I.random_unit(100, d, 12)
    qv = T[37:38] + 0.05 * np.random.default_rng(3).standard_normal((1, d))
    qv /= np.linalg.norm(qv)
    z, db, (sk, pk, rlk, gk) = _enroll_and_decrypt(O, logN, d, p, T)
    S, s, B = O.layout(logN, d, p)
    qc = O.encrypt(logN, pk, O.encode(O.pack_query(qv, logN, d, p).reshape(-1, S), logN), 0, 3).reshape(1, p, 2, 2, -1)
    out, pairs = O.match(logN, d, p, 0, rlk, gk, db, qc, n_threads=4)
    q0 = O.primes()[0]
    sc = np.concatenate([O.scores_from_output(logN, d, p, sk, out[i], q0) for i in range(len(pairs))])[:len(T)]
    ref = (qv @ T.T)[0]
    assert np.abs(sc - ref).max() < 1e-6
    assert sc.argmax() == ref.argmax() == 37
