"""Worst-case residues and full-grid parity (GPU vs the CPU oracle, bit-exact).

The kernels rely on lazy-reduction bounds (ntt2.cuh: forward q0 grows to < 53 q0 < 2^64 without a
reduction, inverse q1 to < 2^15 q1; k_tensor folds its 128-bit sums every 512 parts; k_hrot folds
every 64 rotations) that uniform ciphertexts rarely approach.  Here the inputs are the extremes the
definitions allow, built from the definitions (never from the CUDA path):
  * "qm1":  every coefficient of every limb and component = q - 1;
  * "alt":  coefficients alternating 0 / q - 1 (component 1 in the opposite phase);
  * "ntt":  the constant polynomial -1 (coefficient 0 = q - 1, the rest 0), whose NTT-domain
            value is q - 1 in EVERY slot whatever the evaluation order: the tensor's worst case,
            products (q - 1)^2 summed over all p parts.
Ciphertexts enter the GPU through bm_ct_from_coeff (itself pinned against the oracle's encryption in
test_gpu_parity.py::test_encrypt_parity); the oracle takes the coefficient-domain arrays as they are.
The last test runs the whole bench grid of configs[1] (9,216 pairs) against the oracle."""
import os

import numpy as np
import pytest

from paper_2408_06167_b200 import inputs as I

pytestmark = pytest.mark.gpu

LOGN = 13
N = 1 << LOGN
NTH = max(1, os.cpu_count() or 1)


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the GPU tests need a B200 (there is no CPU fallback)")
    from paper_2408_06167_b200 import build
    build.build(verbose=False)
    from paper_2408_06167_b200 import bm
    return torch, bm


def pattern_ct(pattern, n, mods):
    """[n][2][len(mods)][N] coefficient-domain residues of the given extreme pattern."""
    L = len(mods)
    out = np.zeros((n, 2, L, N), np.uint64)
    for li, q in enumerate(mods):
        qm1 = np.uint64(q - 1)
        if pattern == "qm1":
            out[:, :, li, :] = qm1
        elif pattern == "alt":
            out[:, 0, li, 1::2] = qm1
            out[:, 1, li, 0::2] = qm1
        elif pattern == "ntt":
            out[:, :, li, 0] = qm1
        else:
            raise ValueError(pattern)
    return out


def to_dev(torch, B, prm, ct, n_limbs):
    t = torch.from_numpy(np.ascontiguousarray(ct).view(np.int64)).cuda()
    out = torch.empty_like(t)
    B.bm_ct_from_coeff(prm, t, n_limbs, out)
    return out


@pytest.mark.parametrize("d,p,order,pattern", [
    (128, 8, 0, "qm1"), (128, 8, 0, "alt"), (128, 8, 0, "ntt"),
    (128, 8, 1, "qm1"), (128, 8, 1, "ntt"),
    (128, 8, 2, "qm1"), (128, 8, 2, "ntt"),          # k_hrot: 15 rotations accumulated in 128 bits
    (128, 1, 2, "qm1"), (128, 1, 2, "alt"),          # k_hrot: 127 rotations, its 64-rotation folds
    (4096, 1, 0, "qm1"), (4096, 1, 0, "alt"),        # s = 4096: the 12-step ladder
    (1024, 1024, 0, "ntt"), (1024, 1024, 0, "qm1"),  # p = 1024: the tensor's 512-part folds
])
def test_worst_case_residues_scan(env, O, d, p, order, pattern):
    torch, B = env
    q0, q1, P = O.primes()
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    n_rot = O.n_rot_for(d, p)
    osk, opk, orlk, ogk = O.keygen(LOGN, 1, n_rot)
    if order == 2:
        B.bm_evk_add_hoisted(prm, 1, evk)
        ogk = O.keygen_hoisted(LOGN, 1, d // p)
    evk_dev = B.bm_evk_to_device(prm, evk)
    n_sets, nq = (2, 2) if p <= 8 else (1, 1)
    db = pattern_ct(pattern, n_sets * p, (q0, q1)).reshape(n_sets, p, 2, 2, N)
    qc = pattern_ct(pattern, nq * p, (q0, q1)).reshape(nq, p, 2, 2, N)
    if pattern == "alt":          # break the symmetry between the DB and the query side
        qc = qc[:, :, ::-1].copy()
    d_db, d_q = to_dev(torch, B, prm, db, 2), to_dev(torch, B, prm, qc, 2)
    out = torch.empty((nq, n_sets, 2, N), dtype=torch.int64, device="cuda")
    ws = torch.empty(B.bm_match_ws_bytes(prm, n_sets, nq, order), dtype=torch.uint8, device="cuda")
    B.bm_match(prm, evk_dev, d_db, n_sets, d_q, nq, out, ws, order)
    B.bm_sync()
    got = out.cpu().numpy().view(np.uint64)
    ref, pairs = O.match(LOGN, d, p, order, orlk, ogk, db, qc, n_threads=NTH)
    for k, (j, t) in enumerate(pairs):
        assert np.array_equal(got[j, t], ref[k].reshape(2, N)), (j, t)


@pytest.mark.parametrize("pattern", ["qm1", "alt", "ntt"])
def test_worst_case_residues_expand(env, O, pattern):
    """f3 (bm_expand, Algorithm 1) on extreme level-2 inputs == or_expand."""
    torch, B = env
    d, p = 128, 8
    q0, q1, P = O.primes()
    q2 = O.q2()
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    xk = B.bm_xk_keygen(prm, 1)
    _, ogk1 = O.keygen_exp(LOGN, 1, d, p)
    masks = O.expand_masks(LOGN, d, p)
    xk_dev = B.bm_xk_to_device(prm, pk, xk, masks, None, enroll=False)
    ct = pattern_ct(pattern, 2, (q0, q1, q2))
    d_in = to_dev(torch, B, prm, ct, 3)
    out = torch.empty((2, p, 2, 2, N), dtype=torch.int64, device="cuda")
    ws = torch.empty(B.bm_expand_ws_bytes(prm, 2), dtype=torch.uint8, device="cuda")
    B.bm_expand(prm, xk_dev, d_in, 2, out, ws)
    c = torch.empty_like(out)
    B.bm_ct_to_coeff(prm, out, 2, c)
    B.bm_sync()
    got = c.cpu().numpy().view(np.uint64)
    assert np.array_equal(got, O.expand(LOGN, d, p, masks, ogk1, ct))


@pytest.mark.parametrize("pattern", ["qm1", "ntt"])
def test_worst_case_residues_compressed(env, O, pattern):
    """f1 (bm_match_cmp: tensor over three limbs, 3-digit relin + Res q2, level-1 ladder, compression)
    on extreme level-2 inputs == or_match_cmp."""
    torch, B = env
    d, p = 128, 8
    q0, q1, P = O.primes()
    q2 = O.q2()
    prm = B.bm_params_init(d, p)
    ck = B.bm_ck_keygen(prm, 1)
    orlk2, ogkl, ogkc = O.keygen_cmp(LOGN, 1, d, p)
    mask = O.cmp_mask(LOGN, d, p)
    ck_dev = B.bm_ck_to_device(prm, ck, mask)
    n_sets, nq = 3, 1
    db = pattern_ct(pattern, n_sets * p, (q0, q1, q2)).reshape(n_sets, p, 2, 3, N)
    qc = pattern_ct(pattern, nq * p, (q0, q1, q2)).reshape(nq, p, 2, 3, N)
    d_db, d_q = to_dev(torch, B, prm, db, 3), to_dev(torch, B, prm, qc, 3)
    G = -(-n_sets // prm.s)
    out = torch.empty((nq, G, 2, N), dtype=torch.int64, device="cuda")
    ws = torch.empty(B.bm_match_cmp_ws_bytes(prm, n_sets, nq), dtype=torch.uint8, device="cuda")
    B.bm_match_cmp(prm, ck_dev, d_db, n_sets, d_q, nq, out, ws)
    B.bm_sync()
    exp = O.match_cmp(LOGN, d, p, orlk2, ogkl, ogkc, mask, db, qc, n_threads=NTH)
    assert np.array_equal(out.cpu().numpy().view(np.uint64).reshape(exp.shape), exp)


@pytest.mark.slow
def test_full_grid_parity_at_bench_launch(env, O):
    """Every one of the 9,216 (query, set) pairs of the configs[1] bench step (384 genuine queries x
    24 sets, p = 8, one bm_match launch of the bench's shape: one 9,216-pair chunk, 62 full ladder
    waves + a cluster tail) equals the oracle bit for bit.  Both sides encrypt the oracle-encoded
    plaintexts with the same seeds (~2 min of oracle time on 16 host threads)."""
    torch, B = env
    d, p = 128, 8
    T = I.templates(2)
    Q, _ = I.queries(2)
    prm = B.bm_params_init(d, p)
    S, s, Bk = O.layout(LOGN, d, p)
    n_sets, nq = -(-T.shape[0] // Bk), Q.shape[0]
    sk, pk, evk = B.bm_keygen(prm, 1)
    pk_dev, evk_dev = B.bm_pk_to_device(prm, pk), B.bm_evk_to_device(prm, evk)
    osk, opk, orlk, ogk = O.keygen(LOGN, 1, O.n_rot_for(d, p))
    db_pt = O.encode(O.pack_db(T, LOGN, d, p, 0, n_sets).reshape(-1, S), LOGN)
    q_pt = O.encode(O.pack_query(Q, LOGN, d, p).reshape(-1, S), LOGN)
    d_db = torch.empty((n_sets, p, 2, 2, N), dtype=torch.int64, device="cuda")
    d_q = torch.empty((nq, p, 2, 2, N), dtype=torch.int64, device="cuda")
    B.bm_encrypt(prm, pk_dev, torch.from_numpy(db_pt).cuda(), 0, 2, d_db)
    B.bm_encrypt(prm, pk_dev, torch.from_numpy(q_pt).cuda(), 0, 3, d_q)
    out = torch.empty((nq, n_sets, 2, N), dtype=torch.int64, device="cuda")
    ws = torch.empty(B.bm_match_ws_bytes(prm, n_sets, nq), dtype=torch.uint8, device="cuda")
    B.bm_match(prm, evk_dev, d_db, n_sets, d_q, nq, out, ws)
    B.bm_sync()
    got = out.cpu().numpy().view(np.uint64)
    odb = O.encrypt(LOGN, opk, db_pt, 0, 2).reshape(n_sets, p, 2, 2, N)
    oq = O.encrypt(LOGN, opk, q_pt, 0, 3).reshape(nq, p, 2, 2, N)
    ref, pairs = O.match(LOGN, d, p, 0, orlk, ogk, odb, oq, n_threads=NTH)
    ref = ref.reshape(nq, n_sets, 2, N)
    bad = np.nonzero([not np.array_equal(got[j, t], ref[j, t]) for j, t in pairs])[0]
    assert bad.size == 0, f"{bad.size} of {len(pairs)} pairs differ, first {pairs[bad[0]]}"
