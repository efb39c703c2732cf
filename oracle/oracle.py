"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and --impl reference)
may import this module.  It loads oracle/liboracle.so (plain C, ckks_oracle.c) and adds
the floating-point client-side steps in plain numpy:

  * encode  (CKKS canonical embedding, "encrypts ... feature vector";
             slot j <-> root zeta^(5^j), zeta = exp(i pi / N); readings R1, R15)
  * decode  (direct formula z_j = sum_k m_k cos(pi k e_j / N) / scale)
  * packing of templates into sets and of the query into p replicated parts
             (readings R10, R11)
  * score extraction at slot k*s and argmax

Nothing here is shared with the product package; the only common module is the seeded
input generator paper_2408_06167_b200/inputs.py (no CKKS arithmetic in it).
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_san.so" if os.environ.get("ORACLE_SANITIZE") else "liboracle.so")

DELTA = 2.0 ** 40          # encoding scale (BASELINE.json configs[0]: "scale 2^40")
ORDER_HOISTED = 0
ORDER_PAPER = 1

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i8p = ctypes.POINTER(ctypes.c_int8)
_u32p = ctypes.POINTER(ctypes.c_uint32)


def build(force=False):
    """Compile liboracle.so (plain C, no optimisation flags beyond -O2).  ORACLE_SANITIZE=1 builds an
    ASan + UBSan instrumented copy instead (tools/oracle_sanitize.sh)."""
    src = os.path.join(HERE, "ckks_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        san = ["-fsanitize=address,undefined", "-fno-omit-frame-pointer", "-g"] if os.environ.get(
            "ORACLE_SANITIZE") else []
        subprocess.check_call(["gcc", "-O2", "-Wall", "-fPIC", "-shared", *san, "-o", LIB_PATH, src, "-lpthread"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.or_is_prime.argtypes = [ctypes.c_uint64]
        L.or_is_prime.restype = ctypes.c_int
        L.or_find_prime.argtypes = [ctypes.c_int, ctypes.c_uint64]
        L.or_find_prime.restype = ctypes.c_uint64
        L.or_primes.argtypes = [_u64p]
        L.or_poly_mul.argtypes = [ctypes.c_int, ctypes.c_uint64, _u64p, _u64p, _u64p]
        L.or_automorphism.argtypes = [ctypes.c_int, ctypes.c_uint64, _u64p, ctypes.c_uint64, _u64p]
        L.or_chacha_quarter.argtypes = [_u32p, _u32p, _u32p, _u32p]
        L.or_chacha20_block.argtypes = [_u32p, ctypes.c_uint32, _u32p, _u32p]
        L.or_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64]
        L.or_draw.restype = ctypes.c_uint64
        L.or_sample.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int,
                                ctypes.c_int, ctypes.c_uint64, _u64p]
        L.or_keygen.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _i8p, _u64p, _u64p, _u64p]
        L.or_keygen.restype = ctypes.c_int
        L.or_encrypt.argtypes = [ctypes.c_int, _u64p, _i64p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, _u64p]
        L.or_decrypt.argtypes = [ctypes.c_int, _i8p, _u64p, ctypes.c_int, _u64p]
        L.or_relinearize.argtypes = [ctypes.c_int, _u64p, _u64p, _u64p]
        L.or_rescale.argtypes = [ctypes.c_int, _u64p, _u64p]
        L.or_rotate.argtypes = [ctypes.c_int, _u64p, ctypes.c_uint64, _u64p, _u64p]
        L.or_moddown.argtypes = [ctypes.c_int, ctypes.c_int, _u64p, _u64p]
        L.or_match.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _u64p, _u64p, _u64p,
                               ctypes.c_int64, _u64p, ctypes.c_int64, _i64p, ctypes.c_int64, _u64p, ctypes.c_int]
        L.or_match_deg2.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _u64p, ctypes.c_int64, _u64p,
                                    ctypes.c_int64, _i64p, ctypes.c_int64, _u64p, ctypes.c_int]
        L.or_match_deg2.restype = ctypes.c_int
        L.or_decrypt_deg2.argtypes = [ctypes.c_int, _i8p, _u64p, _u64p]
        L.or_match.restype = ctypes.c_int
        L.or_keygen_hoisted.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _u64p]
        L.or_keygen_hoisted.restype = ctypes.c_int
        L.or_hoisted_rot_sum.argtypes = [ctypes.c_int, ctypes.c_int, _u64p, _u64p, _u64p]
        L.or_bsgs_rot_sum.argtypes = [ctypes.c_int, ctypes.c_int, _u64p, _u64p, _u64p]
        # f3: server-side query expansion on the chain extended by q2
        L.or_find_prime_below.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.or_find_prime_below.restype = ctypes.c_uint64
        L.or_q2.restype = ctypes.c_uint64
        L.or_keygen_exp.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _u64p, _u64p]
        L.or_keygen_exp.restype = ctypes.c_int
        L.or_encrypt_l2.argtypes = [ctypes.c_int, _u64p, _u64p, _i64p, ctypes.c_int64, ctypes.c_uint64,
                                    ctypes.c_uint64, _u64p]
        L.or_decrypt_l2.argtypes = [ctypes.c_int, _i8p, _u64p, _u64p]
        L.or_mul_plain_rescale_q2.argtypes = [ctypes.c_int, _u64p, _i64p, _u64p]
        L.or_rotate1.argtypes = [ctypes.c_int, _u64p, ctypes.c_uint64, _u64p, _u64p]
        L.or_expand.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, _u64p, _u64p, ctypes.c_int64, _u64p]
        L.or_expand.restype = ctypes.c_int
        L.or_enroll.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, _u64p, _u64p, ctypes.c_int64,
                                ctypes.c_int64, _u64p, ctypes.c_int64]
        L.or_enroll.restype = ctypes.c_int
        # f1: compression, with HE-C^3 one level up
        L.or_keygen_cmp.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _u64p,
                                    _u64p, _u64p]
        L.or_keygen_cmp.restype = ctypes.c_int
        L.or_relin_rescale_l2.argtypes = [ctypes.c_int, _u64p, _u64p, _u64p]
        L.or_match_cmp.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _u64p, _u64p, _u64p, _i64p, _u64p,
                                   ctypes.c_int64, _u64p, ctypes.c_int64, _u64p, ctypes.c_int]
        L.or_match_cmp.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a, t):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


def primes():
    out = np.zeros(3, np.uint64)
    lib().or_primes(_p(out, _u64p))
    return [int(x) for x in out]


def poly_mul(logN, q, a, b):
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    c = np.zeros(1 << logN, np.uint64)
    lib().or_poly_mul(logN, q, _p(a, _u64p), _p(b, _u64p), _p(c, _u64p))
    return c


def automorphism(logN, q, a, g):
    a = np.ascontiguousarray(a, np.uint64)
    c = np.zeros(1 << logN, np.uint64)
    lib().or_automorphism(logN, q, _p(a, _u64p), g, _p(c, _u64p))
    return c


def chacha20_block(key, counter, nonce):
    k = np.array(key, np.uint32)
    n = np.array(nonce, np.uint32)
    out = np.zeros(16, np.uint32)
    lib().or_chacha20_block(_p(k, _u32p), counter, _p(n, _u32p), _p(out, _u32p))
    return out


def chacha_quarter(a, b, c, d):
    v = [ctypes.c_uint32(x) for x in (a, b, c, d)]
    lib().or_chacha_quarter(*[ctypes.byref(x) for x in v])
    return [x.value for x in v]


def draw(seed, purpose, obj, sub, n):
    return int(lib().or_draw(seed, purpose, obj, sub, n))


KIND_UNIFORM, KIND_TERNARY, KIND_GAUSS = 0, 1, 2


def sample(seed, purpose, obj, sub, kind, n, q=0):
    out = np.zeros(n, np.uint64)
    lib().or_sample(seed, purpose, obj, sub, kind, n, q, _p(out, _u64p))
    return out if q else out.view(np.int64)


# ---------------------------------------------------------------------------- keys / enc / dec
def n_rot_for(d, p):
    s = d // p
    return max(0, s.bit_length() - 1)   # rotations 2^i, i < log2 s


def keygen(logN, seed, n_rot, zero_error=False):
    N = 1 << logN
    sk = np.zeros(N, np.int8)
    pk = np.zeros((2, 2, N), np.uint64)
    rlk = np.zeros((2, 2, 3, N), np.uint64)
    gk = np.zeros((max(n_rot, 1), 2, 2, N), np.uint64)
    lib().or_keygen(logN, seed, n_rot, int(zero_error), _p(sk, _i8p), _p(pk, _u64p), _p(rlk, _u64p), _p(gk, _u64p))
    return sk, pk, rlk, gk[:n_rot]


def keygen_hoisted(logN, seed, s, zero_error=False):
    """f2: Galois keys for every rotation r = 1..s-1 (hgk[r-1]), same secret as keygen(seed)."""
    N = 1 << logN
    hgk = np.zeros((max(s - 1, 1), 2, 2, N), np.uint64)
    lib().or_keygen_hoisted(logN, seed, s, int(zero_error), _p(hgk, _u64p))
    return hgk[:max(s - 1, 0)]


def hoisted_rot_sum(logN, s, hgk, ct):
    """f2: sum_{r<s} Rot(ct, r) with one hoisted key switch; ct [2][1][N] level 0."""
    ct = np.ascontiguousarray(ct, np.uint64)
    out = np.zeros((2, 1, 1 << logN), np.uint64)
    h = np.ascontiguousarray(hgk if len(hgk) else np.zeros((1, 2, 2, 1 << logN), np.uint64), np.uint64)
    lib().or_hoisted_rot_sum(logN, s, _p(h, _u64p), _p(ct, _u64p), _p(out, _u64p))
    return out


def bsgs_rot_sum(logN, s, hgk, ct):
    """f2: sum_{r<s} Rot(ct, r) as baby steps (b = 2^ceil(log2(s)/2)) then giant steps (g = s / b), each
    one hoisted key switch; ct [2][1][N] level 0."""
    ct = np.ascontiguousarray(ct, np.uint64)
    out = np.zeros((2, 1, 1 << logN), np.uint64)
    h = np.ascontiguousarray(hgk if len(hgk) else np.zeros((1, 2, 2, 1 << logN), np.uint64), np.uint64)
    lib().or_bsgs_rot_sum(logN, s, _p(h, _u64p), _p(ct, _u64p), _p(out, _u64p))
    return out


def encrypt(logN, pk, pt, first_obj, seed):
    """pt int64 [n][N] -> level-1 cts [n][2][2][N] (coefficient domain)."""
    pt = np.ascontiguousarray(pt, np.int64)
    n = pt.shape[0]
    out = np.zeros((n, 2, 2, 1 << logN), np.uint64)
    lib().or_encrypt(logN, _p(np.ascontiguousarray(pk), _u64p), _p(pt, _i64p), n, first_obj, seed, _p(out, _u64p))
    return out


def decrypt(logN, sk, ct, n_limbs):
    """ct [2][n_limbs][N] -> m residues [n_limbs][N]."""
    ct = np.ascontiguousarray(ct, np.uint64)
    m = np.zeros((n_limbs, 1 << logN), np.uint64)
    lib().or_decrypt(logN, _p(np.ascontiguousarray(sk), _i8p), _p(ct, _u64p), n_limbs, _p(m, _u64p))
    return m


def relinearize(logN, d, rlk):
    d = np.ascontiguousarray(d, np.uint64)
    out = np.zeros((2, 2, 1 << logN), np.uint64)
    lib().or_relinearize(logN, _p(d, _u64p), _p(np.ascontiguousarray(rlk), _u64p), _p(out, _u64p))
    return out


def rescale(logN, ct):
    ct = np.ascontiguousarray(ct, np.uint64)
    out = np.zeros((2, 1, 1 << logN), np.uint64)
    lib().or_rescale(logN, _p(ct, _u64p), _p(out, _u64p))
    return out


def rotate(logN, ct, r, gkr):
    ct = np.ascontiguousarray(ct, np.uint64)
    out = np.zeros((2, 1, 1 << logN), np.uint64)
    lib().or_rotate(logN, _p(ct, _u64p), r, _p(np.ascontiguousarray(gkr), _u64p), _p(out, _u64p))
    return out


def moddown(logN, n_q, KS):
    KS = np.ascontiguousarray(KS, np.uint64)
    out = np.zeros((n_q, 1 << logN), np.uint64)
    lib().or_moddown(logN, n_q, _p(KS, _u64p), _p(out, _u64p))
    return out


def match_deg2(logN, d, p, db, q, pairs=None, n_threads=1):
    """f2: the relin-free degree-2 scan for p = d (no rotations): per pair sum_i tensor, then Res of
    each of the three components.  db [T][p][2][2][N], q [Q][p][2][2][N] -> out [n_pairs][3][1][N]."""
    N = 1 << logN
    db = np.ascontiguousarray(db, np.uint64)
    q = np.ascontiguousarray(q, np.uint64)
    T, Q = db.shape[0], q.shape[0]
    if pairs is None:
        pairs = np.array([(j, t) for j in range(Q) for t in range(T)], np.int64).reshape(-1, 2)
    pairs = np.ascontiguousarray(pairs, np.int64)
    out = np.zeros((pairs.shape[0], 3, 1, N), np.uint64)
    rc = lib().or_match_deg2(logN, d, p, _p(db, _u64p), T, _p(q, _u64p), Q, _p(pairs, _i64p), pairs.shape[0],
                             _p(out, _u64p), n_threads)
    assert rc == 0, rc
    return out, pairs


def decrypt_deg2(logN, sk, ct):
    """m = c0 + c1 s + c2 s^2 mod q0 of a level-0 degree-2 ciphertext [3][N] (residues)."""
    ct = np.ascontiguousarray(ct, np.uint64)
    m = np.zeros(1 << logN, np.uint64)
    lib().or_decrypt_deg2(logN, _p(np.ascontiguousarray(sk), _i8p), _p(ct, _u64p), _p(m, _u64p))
    return m


def match(logN, d, p, order, rlk, gk, db, q, pairs=None, n_threads=1):
    """Algorithm 2 over (query, set) pairs. db [T][p][2][2][N], q [Q][p][2][2][N].
    order 0 hoisted relin, 1 paper order, 2 f2 hoisted rotation sum, 4 f2 baby-step giant-step rotation
    sum (2 and 4: gk = keygen_hoisted keys).
    Returns out [n_pairs][2][1][N] and the pairs array."""
    N = 1 << logN
    db = np.ascontiguousarray(db, np.uint64)
    q = np.ascontiguousarray(q, np.uint64)
    T, Q = db.shape[0], q.shape[0]
    if pairs is None:
        pairs = np.array([(j, t) for j in range(Q) for t in range(T)], np.int64).reshape(-1, 2)
    pairs = np.ascontiguousarray(pairs, np.int64)
    out = np.zeros((pairs.shape[0], 2, 1, N), np.uint64)
    gk = np.ascontiguousarray(gk if len(gk) else np.zeros((1, 2, 2, N), np.uint64), np.uint64)
    rc = lib().or_match(logN, d, p, order, _p(np.ascontiguousarray(rlk), _u64p), _p(gk, _u64p), _p(db, _u64p), T,
                        _p(q, _u64p), Q, _p(pairs, _i64p), pairs.shape[0], _p(out, _u64p), n_threads)
    if rc != 0:
        raise ValueError(f"or_match failed: {rc}")
    return out, pairs


# ---------------------------------------------------------------------------- encode / decode
def slot_exponents(logN):
    """e_j = 5^j mod 2N for the S = N/2 slots."""
    N = 1 << logN
    e = np.empty(N // 2, np.int64)
    x = 1
    for j in range(N // 2):
        e[j] = x
        x = (x * 5) % (2 * N)
    return e


def encode(z, logN, scale=DELTA):
    """Real slot vector(s) z [..., S] -> integer plaintext [..., N] (int64).

    m_k = (2/N) sum_j z_j cos(pi k e_j / N) = (2/N) Re(sum_t X[t] zeta^(k t)), X[e_j] = z_j,
    evaluated with a 2N-point inverse FFT (library primitive); pt_k = round(scale * m_k),
    halves away from zero (reading R15)."""
    N = 1 << logN
    z = np.asarray(z, np.float64)
    X = np.zeros(z.shape[:-1] + (2 * N,), np.complex128)
    X[..., slot_exponents(logN)] = z
    m = 4.0 * np.fft.ifft(X, axis=-1).real[..., :N]      # (2/N) * 2N * ifft
    v = scale * m
    return (np.sign(v) * np.floor(np.abs(v) + 0.5)).astype(np.int64)


def encode_direct(z, logN, scale=DELTA):
    """The same encoding by the O(N*S) direct formula (for small-N pins)."""
    N = 1 << logN
    e = slot_exponents(logN)
    k = np.arange(N)
    C = np.cos(np.pi * ((k[:, None] * e[None, :]) % (2 * N)) / N)
    v = scale * (2.0 / N) * (C @ np.asarray(z, np.float64))
    return (np.sign(v) * np.floor(np.abs(v) + 0.5)).astype(np.int64)


def decode_slots(m_centred, logN, scale, slots=None):
    """z_j = sum_k m_k cos(pi k e_j / N) / scale for the requested slots j (default all)."""
    N = 1 << logN
    e = slot_exponents(logN)
    if slots is not None:
        e = e[np.asarray(slots)]
    k = np.arange(N)
    C = np.cos(np.pi * ((e[:, None] * k[None, :]) % (2 * N)) / N)
    return (C @ np.asarray(m_centred, np.float64)) / scale


def centred(x, q):
    x = np.asarray(x, np.uint64).astype(object)
    return np.array([int(v) - q if int(v) > q // 2 else int(v) for v in x.ravel()], dtype=object).reshape(x.shape)


def centred_i64(x, q):
    x = np.asarray(x, np.uint64)
    half = np.uint64(q // 2)
    out = x.astype(np.int64)
    neg = x > half
    out[neg] = (x[neg] - np.uint64(q)).astype(np.int64)
    return out


# ---------------------------------------------------------------------------- packing (client side)
def layout(logN, d, p):
    S = (1 << logN) // 2
    s = d // p
    B = S // s
    return S, s, B


def pack_db(tmpl, logN, d, p, first_set, n_sets):
    """Slot vectors z[t][i][k*s + j] = v_{tB+k}[i*s + j]; zeros past n."""
    S, s, B = layout(logN, d, p)
    tmpl = np.asarray(tmpl, np.float64)
    n = tmpl.shape[0]
    z = np.zeros((n_sets, p, S))
    for t in range(n_sets):
        u0 = (first_set + t) * B
        cnt = max(0, min(B, n - u0))
        if cnt == 0:
            continue
        blk = tmpl[u0:u0 + cnt].reshape(cnt, p, s)          # [k][i][j]
        z[t, :, :cnt * s] = blk.transpose(1, 0, 2).reshape(p, cnt * s)
    return z


def pack_query(qv, logN, d, p):
    """w_i[x] = q[i*s + (x mod s)] for x < S."""
    S, s, B = layout(logN, d, p)
    qv = np.asarray(qv, np.float64).reshape(-1, p, s)
    return np.tile(qv, (1, 1, B))                            # [Q][p][S]


def scores_from_output(logN, d, p, sk, out_ct, q0):
    """Decrypt a level-0 result [2][1][N] and read slot k*s for k < B."""
    S, s, B = layout(logN, d, p)
    m = decrypt(logN, sk, out_ct, 1)[0]
    P = primes()
    scale = DELTA * DELTA / P[1]
    return decode_slots(centred_i64(m, q0), logN, scale, slots=np.arange(B) * s)


# ---------------------------------------------------------------------------- f3: query expansion
# Algorithm 1 "Input Ciphertext Expansion" with SPEC.md:297's post-condition
# on the chain extended by one 40-bit prime q2 (readings R24-R26): the client encrypts
# the query tiled S/d times at level 2 = {q0, q1, q2}; the server multiplies by mask X_i (scale q2),
# rescales by q2 (level 1, scale exactly 2^40) and adds log2(p) left rotations by s 2^t.
def q2():
    return int(lib().or_q2())


def find_prime_below(below, m):
    return int(lib().or_find_prime_below(below, m))


def log2_exact(x):
    k = x.bit_length() - 1
    assert 1 << k == x
    return k


def keygen_exp(logN, seed, d, p, zero_error=False, n_rot=None):
    """Expansion keys of keygen(seed)'s secret: pk_q2 [2][N] (pk's q2 limb) and the level-1
    Galois keys gk1 [n_rot][2 digits][2 comps][3 limbs q0,q1,P][N] of rotations s 2^t
    (n_rot: log2 p by default, the expansion's; log2 B covers the enrollment too)."""
    N = 1 << logN
    lp = log2_exact(p) if n_rot is None else n_rot
    pk_q2 = np.zeros((2, N), np.uint64)
    gk1 = np.zeros((max(lp, 1), 2, 2, 3, N), np.uint64)
    rc = lib().or_keygen_exp(logN, seed, d, p, lp, int(zero_error), _p(pk_q2, _u64p), _p(gk1, _u64p))
    if rc:
        raise ValueError(f"or_keygen_exp: {rc}")
    return pk_q2, gk1[:lp]


def encrypt_l2(logN, pk, pk_q2, pt, first_obj, seed):
    """pt int64 [n][N] -> level-2 cts [n][2][3][N] (coefficient domain)."""
    pt = np.ascontiguousarray(pt, np.int64)
    n = pt.shape[0]
    out = np.zeros((n, 2, 3, 1 << logN), np.uint64)
    lib().or_encrypt_l2(logN, _p(np.ascontiguousarray(pk, np.uint64), _u64p),
                        _p(np.ascontiguousarray(pk_q2, np.uint64), _u64p), _p(pt, _i64p), n, first_obj, seed,
                        _p(out, _u64p))
    return out


def decrypt_l2(logN, sk, ct):
    """ct [2][3][N] -> m residues [3][N] (limbs q0, q1, q2)."""
    ct = np.ascontiguousarray(ct, np.uint64)
    m = np.zeros((3, 1 << logN), np.uint64)
    lib().or_decrypt_l2(logN, _p(np.ascontiguousarray(sk), _i8p), _p(ct, _u64p), _p(m, _u64p))
    return m


def mul_plain_rescale_q2(logN, ct, pt):
    """Res(Mul(P)(ct, pt)): ct [2][3][N] level 2, pt int64 [N] -> [2][2][N] level 1."""
    ct = np.ascontiguousarray(ct, np.uint64)
    pt = np.ascontiguousarray(pt, np.int64)
    out = np.zeros((2, 2, 1 << logN), np.uint64)
    lib().or_mul_plain_rescale_q2(logN, _p(ct, _u64p), _p(pt, _i64p), _p(out, _u64p))
    return out


def rotate1(logN, ct, r, gkr):
    """Rot at level 1 with a 2-digit Galois key gkr [2][2][3][N]: ct [2][2][N] -> [2][2][N]."""
    ct = np.ascontiguousarray(ct, np.uint64)
    out = np.zeros((2, 2, 1 << logN), np.uint64)
    lib().or_rotate1(logN, _p(ct, _u64p), r, _p(np.ascontiguousarray(gkr, np.uint64), _u64p), _p(out, _u64p))
    return out


def expand_masks_slots(logN, d, p):
    """X_i[x] = 1 if (x mod d) lies in [i s, (i+1) s), else 0, for x < S."""
    S, s, _ = layout(logN, d, p)
    x = np.arange(S) % d
    return np.stack([((x >= i * s) & (x < (i + 1) * s)).astype(np.float64) for i in range(p)])


def expand_masks(logN, d, p):
    """The p mask plaintexts at scale q2 (so that Res by q2 leaves the query's scale at 2^40)."""
    return encode(expand_masks_slots(logN, d, p), logN, scale=float(q2()))


def tile_query(qv, logN, d):
    """The client's single query vector: q_hat tiled S/d times."""
    S = (1 << logN) // 2
    qv = np.asarray(qv, np.float64).reshape(-1, d)
    return np.tile(qv, (1, S // d))


def expand(logN, d, p, masks, gk1, ct):
    """Algorithm 1: level-2 cts [n][2][3][N] -> expanded level-1 parts [n][p][2][2][N]."""
    ct = np.ascontiguousarray(ct, np.uint64).reshape(-1, 2, 3, 1 << logN)
    n = ct.shape[0]
    out = np.zeros((n, p, 2, 2, 1 << logN), np.uint64)
    g = np.ascontiguousarray(gk1 if len(gk1) else np.zeros((1, 2, 2, 3, 1 << logN), np.uint64), np.uint64)
    rc = lib().or_expand(logN, d, p, _p(np.ascontiguousarray(masks, np.int64), _i64p), _p(g, _u64p), _p(ct, _u64p),
                         n, _p(out, _u64p))
    if rc:
        raise ValueError(f"or_expand: {rc}")
    return out


# ---------------------------------------------------------------------------- f4: server-side enrollment
# Fig. 3 / PAPER.md:251-269 with SPEC.md:282-293's semantics (reading R27), same chain as f3.
def n_rot_enroll(logN, d, p):
    """Galois keys the enrollment needs: strides s 2^t for t < log2 B."""
    return log2_exact(layout(logN, d, p)[2])


def enroll_masks_slots(logN, d, p):
    """E_i[x] = 1 if x lies in [i s, (i+1) s), else 0."""
    S, s, _ = layout(logN, d, p)
    x = np.arange(S)
    return np.stack([((x >= i * s) & (x < (i + 1) * s)).astype(np.float64) for i in range(p)])


def enroll_masks(logN, d, p):
    return encode(enroll_masks_slots(logN, d, p), logN, scale=float(q2()))


def enroll_vector(v, logN, d):
    """The client's enrollment slots: the template in slots [0, d), zeros elsewhere."""
    S = (1 << logN) // 2
    v = np.asarray(v, np.float64).reshape(-1, d)
    z = np.zeros((v.shape[0], S))
    z[:, :d] = v
    return z


def enroll(logN, d, p, emasks, gk1, ct, first_u, db):
    """Accumulates the level-2 template cts ct [n][2][3][N] (templates first_u..) into db
    [n_sets][p][2][2][N] (level 1, modified in place and returned)."""
    ct = np.ascontiguousarray(ct, np.uint64).reshape(-1, 2, 3, 1 << logN)
    assert db.flags["C_CONTIGUOUS"] and db.dtype == np.uint64
    g = np.ascontiguousarray(gk1 if len(gk1) else np.zeros((1, 2, 2, 3, 1 << logN), np.uint64), np.uint64)
    rc = lib().or_enroll(logN, d, p, _p(np.ascontiguousarray(emasks, np.int64), _i64p), _p(g, _u64p), _p(ct, _u64p),
                         ct.shape[0], first_u, _p(db, _u64p), db.shape[0])
    if rc:
        raise ValueError(f"or_enroll: {rc}")
    return db


# ---------------------------------------------------------------------------- f1: output compression
# PAPER.md:273, 343-345 and SPEC.md:321-329 (reading R28), same extended chain: HE-C^3 runs at
# level 2 (Res by q2), its ladder at level 1, and the compression's Mul(P) + Res by q1 ends at level 0.
def keygen_cmp(logN, seed, d, p, zero_error=False):
    """rlk2 [3][2][4 limbs q0,q1,q2,P][N]; gkl [log2 s][2][2][3][N] (level-1 ladder keys 2^i);
    gkc [s-1][2][2 limbs q0,P][N] (level-0 right rotations by u = 1..s-1)."""
    N = 1 << logN
    S, s, _ = layout(logN, d, p)
    ls = log2_exact(s)
    rlk2 = np.zeros((3, 2, 4, N), np.uint64)
    gkl = np.zeros((max(ls, 1), 2, 2, 3, N), np.uint64)
    gkc = np.zeros((max(s - 1, 1), 2, 2, N), np.uint64)
    rc = lib().or_keygen_cmp(logN, seed, d, p, int(zero_error), _p(rlk2, _u64p), _p(gkl, _u64p), _p(gkc, _u64p))
    if rc:
        raise ValueError(f"or_keygen_cmp: {rc}")
    return rlk2, gkl[:ls], gkc[:s - 1]


def relin_rescale_l2(logN, d3, rlk2):
    """(d0, d1, d2) at level 2 [3][3][N] -> relinearized, Res by q2: [2][2][N] (level 1)."""
    d3 = np.ascontiguousarray(d3, np.uint64)
    out = np.zeros((2, 2, 1 << logN), np.uint64)
    lib().or_relin_rescale_l2(logN, _p(d3, _u64p), _p(np.ascontiguousarray(rlk2, np.uint64), _u64p), _p(out, _u64p))
    return out


def cmp_mask(logN, d, p):
    """M[x] = [x mod s = 0] at scale q1 (the compression's score mask)."""
    S, s, _ = layout(logN, d, p)
    z = (np.arange(S) % s == 0).astype(np.float64)
    return encode(z, logN, scale=float(primes()[1]))


def match_cmp(logN, d, p, rlk2, gkl, gkc, mask, db, q, n_threads=1):
    """Compressed scan: db [T][p][2][3][N], q [Q][p][2][3][N] (level 2) -> [Q][ceil(T/s)][2][1][N]."""
    N = 1 << logN
    S, s, _ = layout(logN, d, p)
    db = np.ascontiguousarray(db, np.uint64)
    q = np.ascontiguousarray(q, np.uint64)
    T, Q = db.shape[0], q.shape[0]
    G = -(-T // s)
    out = np.zeros((Q, G, 2, 1, N), np.uint64)
    pad = lambda a, shape: np.ascontiguousarray(a if len(a) else np.zeros(shape, np.uint64), np.uint64)
    rc = lib().or_match_cmp(logN, d, p, _p(np.ascontiguousarray(rlk2, np.uint64), _u64p),
                            _p(pad(gkl, (1, 2, 2, 3, N)), _u64p), _p(pad(gkc, (1, 2, 2, N)), _u64p),
                            _p(np.ascontiguousarray(mask, np.int64), _i64p), _p(db, _u64p), T, _p(q, _u64p), Q,
                            _p(out, _u64p), n_threads)
    if rc:
        raise ValueError(f"or_match_cmp: {rc}")
    return out


def packed_scores(logN, d, p, sk, packed, n_sets):
    """Decrypt packed results [G][2][1][N] -> scores [n_sets * B] (set t = g s + u, block k at slot
    k s + u of packed g), scale 2^80 / q2."""
    S, s, B = layout(logN, d, p)
    q0, q1, P = primes()
    scale = DELTA * DELTA / q2()
    sc = np.zeros(n_sets * B)
    for g in range(packed.shape[0]):
        m = decrypt(logN, sk, packed[g], 1)[0]
        z = decode_slots(centred_i64(m, q0), logN, scale)
        for u in range(s):
            t = g * s + u
            if t < n_sets:
                sc[t * B:(t + 1) * B] = z[u::s][:B]
    return sc
