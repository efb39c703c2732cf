"""GPU parity of f1: output compression with
HE-C^3 one level up on the chain extended by q2 (reading R28).  bm_match_cmp (through the
C ABI) against the oracle's or_match_cmp, bit-exact on every residue of the packed level-0 outputs,
given identical keys (tests/test_abi.py pins the host key generator), identical level-2 inputs
(oracle-encrypted) and the oracle-encoded score mask."""
import os

import numpy as np
import pytest

from paper_2408_06167_b200 import inputs as I

pytestmark = pytest.mark.gpu

LOGN = 13
NTH = max(1, min(16, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the GPU tests need a B200 (there is no CPU fallback)")
    from paper_2408_06167_b200 import build
    build.build(verbose=False)
    from paper_2408_06167_b200 import bm
    return torch, bm


class CSetup:
    def __init__(self, env, O, d, p, T, Q, key_seed=1):
        torch, B = env
        self.torch, self.B, self.O, self.d, self.p = torch, B, O, d, p
        self.prm = B.bm_params_init(d, p)
        S, s, Bk = O.layout(LOGN, d, p)
        self.n_sets = -(-T.shape[0] // Bk)
        self.nq = Q.shape[0]
        self.sk, self.pk, self.evk = B.bm_keygen(self.prm, key_seed)
        self.ck = B.bm_ck_keygen(self.prm, key_seed)
        self.osk, self.opk, _, _ = O.keygen(LOGN, key_seed, 0)
        self.opk_q2, _ = O.keygen_exp(LOGN, key_seed, d, p)
        self.orlk2, self.ogkl, self.ogkc = O.keygen_cmp(LOGN, key_seed, d, p)
        self.mask = O.cmp_mask(LOGN, d, p)
        self.ck_dev = B.bm_ck_to_device(self.prm, self.ck, self.mask)
        zdb = O.pack_db(T, LOGN, d, p, 0, self.n_sets)
        self.odb = O.encrypt_l2(LOGN, self.opk, self.opk_q2, O.encode(zdb.reshape(-1, S), LOGN), 0, 2).reshape(
            self.n_sets, p, 2, 3, -1)
        zq = O.pack_query(Q, LOGN, d, p)
        self.oq = O.encrypt_l2(LOGN, self.opk, self.opk_q2, O.encode(zq.reshape(-1, S), LOGN), 0, 3).reshape(
            self.nq, p, 2, 3, -1)
        self.d_db = self.from_coeff(self.odb)
        self.d_q = self.from_coeff(self.oq)

    def from_coeff(self, ct):
        t = self.torch.from_numpy(np.ascontiguousarray(ct).view(np.int64)).cuda()
        out = self.torch.empty_like(t)
        self.B.bm_ct_from_coeff(self.prm, t, 3, out)
        return out

    def gpu(self):
        torch, B = self.torch, self.B
        G = -(-self.n_sets // self.prm.s)
        out = torch.empty((self.nq, G, 2, 8192), dtype=torch.int64, device="cuda")
        ws = torch.empty(B.bm_match_cmp_ws_bytes(self.prm, self.n_sets, self.nq), dtype=torch.uint8, device="cuda")
        B.bm_match_cmp(self.prm, self.ck_dev, self.d_db, self.n_sets, self.d_q, self.nq, out, ws)
        B.bm_sync()
        return out.cpu().numpy().view(np.uint64)

    def oracle(self):
        return self.O.match_cmp(LOGN, self.d, self.p, self.orlk2, self.ogkl, self.ogkc, self.mask, self.odb, self.oq,
                                n_threads=NTH)


@pytest.mark.parametrize("d,p,n_tmpl,nq", [(16, 4, 5500, 2), (128, 8, 4300, 1), (32, 32, 40, 1)])
def test_compressed_scan_parity(env, O, d, p, n_tmpl, nq):
    """bm_match_cmp == or_match_cmp bit for bit: s = 4 with 6 sets (two packed groups, the second
    partial), s = 16 with 17 sets, and s = 1 (no ladder, no rotation: mask + Res only)."""
    T = I.random_unit(n_tmpl, d, 31)
    Q = I.random_unit(nq, d, 32)
    st = CSetup(env, O, d, p, T, Q)
    got = st.gpu()
    exp = st.oracle()
    assert np.array_equal(got.reshape(exp.shape), exp)


def test_compressed_scan_chunked_and_scores(env, O):
    """Chunks that split the sets of a packed group (option cmp_chunk = 5) give the same residues; the
    packed slots decrypt to the plaintext cosines (1e-6) with the genuine template on top."""
    torch, B = env
    d, p = 16, 4
    T = I.random_unit(5000, d, 33)
    Q = T[4321:4322] + 0.05 * np.random.default_rng(9).standard_normal((1, d))
    Q /= np.linalg.norm(Q)
    st = CSetup(env, O, d, p, T, Q)
    whole = st.gpu()
    with B.options(cmp_chunk=5):
        parts = st.gpu()
    assert np.array_equal(whole, parts)
    S, s, Bk = O.layout(LOGN, d, p)
    slots = B.bm_decrypt_packed(st.prm, st.sk, whole.reshape(-1, 2, 1, 8192))
    sc = np.zeros(st.n_sets * Bk)
    for g in range(slots.shape[0]):
        for u in range(s):
            t = g * s + u
            if t < st.n_sets:
                sc[t * Bk:(t + 1) * Bk] = slots[g, u::s]
    cos = T @ Q[0]
    assert np.abs(sc[:len(T)] - cos).max() < 1e-6
    assert np.abs(sc[len(T):]).max() < 1e-6
    assert B.bm_top1(sc[:len(T)])[0] == 4321
