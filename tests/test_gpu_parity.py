"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle, bit-exact on every
RNS residue of the coefficient-domain outputs, given identical seeded keys, plaintexts
(encoded by the oracle) and encryption randomness (north_star)."""
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


class Setup:
    """Keys + oracle-encoded plaintexts, encrypted by BOTH sides with the same seeds."""

    def __init__(self, env, O, d, p, T, Q, key_seed=1, db_seed=2, q_seed=3, n_rot=None, hoisted=False):
        torch, B = env
        self.torch, self.B, self.O = torch, B, O
        self.d, self.p = d, p
        self.prm = B.bm_params_init(d, p)
        S, s, Bk = O.layout(LOGN, d, p)
        self.n_sets = -(-T.shape[0] // Bk)
        self.nq = Q.shape[0]
        self.sk, self.pk, self.evk = B.bm_keygen(self.prm, key_seed)
        self.osk, self.opk, self.orlk, self.ogk = O.keygen(LOGN, key_seed, O.n_rot_for(d, p))
        if hoisted:   # f2: Galois keys of every rotation 1..s-1 on both sides
            B.bm_evk_add_hoisted(self.prm, key_seed, self.evk)
            self.ohgk = O.keygen_hoisted(LOGN, key_seed, s)
        self.pk_dev = B.bm_pk_to_device(self.prm, self.pk)
        self.evk_dev = B.bm_evk_to_device(self.prm, self.evk)
        self.db_pt = O.encode(O.pack_db(T, LOGN, d, p, 0, self.n_sets).reshape(-1, S), LOGN)
        self.q_pt = O.encode(O.pack_query(Q, LOGN, d, p).reshape(-1, S), LOGN)
        self.db_seed, self.q_seed = db_seed, q_seed
        dev = torch.device("cuda")
        self.d_db = torch.empty((self.n_sets, p, 2, 2, 8192), dtype=torch.int64, device=dev)
        self.d_q = torch.empty((self.nq, p, 2, 2, 8192), dtype=torch.int64, device=dev)
        B.bm_encrypt(self.prm, self.pk_dev, torch.from_numpy(self.db_pt).to(dev), 0, db_seed, self.d_db)
        B.bm_encrypt(self.prm, self.pk_dev, torch.from_numpy(self.q_pt).to(dev), 0, q_seed, self.d_q)
        B.bm_sync()

    def oracle_db(self, sets):
        O, p = self.O, self.p
        out = np.zeros((len(sets), p, 2, 2, 8192), np.uint64)
        for k, t in enumerate(sets):
            out[k] = O.encrypt(LOGN, self.opk, self.db_pt[t * p:(t + 1) * p], t * p, self.db_seed).reshape(p, 2, 2, -1)
        return out

    def oracle_q(self, qs):
        O, p = self.O, self.p
        out = np.zeros((len(qs), p, 2, 2, 8192), np.uint64)
        for k, j in enumerate(qs):
            out[k] = O.encrypt(LOGN, self.opk, self.q_pt[j * p:(j + 1) * p], j * p, self.q_seed).reshape(p, 2, 2, -1)
        return out

    def gpu_match(self, order=0):
        torch, B = self.torch, self.B
        out = torch.empty((self.nq, self.n_sets, B.n_components(order), 8192), dtype=torch.int64, device="cuda")
        ws = torch.empty(max(1, B.bm_match_ws_bytes(self.prm, self.n_sets, self.nq, order)), dtype=torch.uint8,
                         device="cuda")
        evk = None if order == B.ORDER_DEG2 else self.evk_dev      # the degree-2 output needs no keys
        B.bm_match(self.prm, evk, self.d_db, self.n_sets, self.d_q, self.nq, out, ws, order)
        B.bm_sync()
        return out.cpu().numpy().view(np.uint64)

    def oracle_pairs(self, pairs, order=0):
        qs = sorted({j for j, _ in pairs})
        ts = sorted({t for _, t in pairs})
        qi = {j: k for k, j in enumerate(qs)}
        ti = {t: k for k, t in enumerate(ts)}
        local = np.array([(qi[j], ti[t]) for j, t in pairs], np.int64).reshape(-1, 2)
        if order == 3:
            out, _ = self.O.match_deg2(LOGN, self.d, self.p, self.oracle_db(ts), self.oracle_q(qs), pairs=local,
                                       n_threads=NTH)
            return out.reshape(-1, 3, 8192)
        gk = self.ohgk if order in (2, 4) else self.ogk
        out, _ = self.O.match(LOGN, self.d, self.p, order, self.orlk, gk, self.oracle_db(ts), self.oracle_q(qs),
                              pairs=local, n_threads=NTH)
        return out.reshape(-1, 2, 8192)


def test_encrypt_parity(env, O):
    """GPU pk-encryption (NTT domain) converted to coefficients == oracle encryption."""
    torch, B = env
    T = I.templates(2, 700)
    st = Setup(env, O, 128, 4, T, I.queries(2, 2)[0])
    coeff = torch.empty_like(st.d_db)
    B.bm_ct_to_coeff(st.prm, st.d_db, 2, coeff)
    got = coeff.cpu().numpy().view(np.uint64)
    exp = st.oracle_db(list(range(st.n_sets)))
    assert np.array_equal(got, exp)
    # from_coeff o to_coeff = identity
    back = torch.empty_like(coeff)
    B.bm_ct_from_coeff(st.prm, coeff, 2, back)
    B.bm_sync()
    assert torch.equal(back, st.d_db)


@pytest.mark.parametrize("order", [0, 1])
def test_config1_parity_and_scores(env, O, order):
    torch, B = env
    T = I.templates(1)
    Q, exp = I.queries(1)
    st = Setup(env, O, 16, 1, T, Q)
    got = st.gpu_match(order)
    ref = st.oracle_pairs([(0, 0)], order)
    assert np.array_equal(got[0, 0], ref[0])
    sc = B.bm_decrypt(st.prm, st.sk, got.reshape(-1, 2, 1, 8192))[0][:256]
    cos = T @ Q[0]
    assert np.abs(sc - cos).max() < 1e-6
    assert B.bm_top1(sc)[0] == exp[0] == int(np.argmax(cos))


@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_config2_sampled_parity(env, O, p):
    """BASELINE.json configs[1] (d = 128, 6,144 templates) at each p of the sweep, 3 genuine
    queries against every set on the GPU; bit-exact parity on sampled pairs incl. the last set."""
    torch, B = env
    T = I.templates(2)
    Q, expq = I.queries(2, 3)
    st = Setup(env, O, 128, p, T, Q)
    got = st.gpu_match(0)
    rng = np.random.default_rng(p)
    pairs = [(0, 0), (2, st.n_sets - 1), (1, int(rng.integers(st.n_sets)))]
    ref = st.oracle_pairs(pairs)
    for k, (j, t) in enumerate(pairs):
        assert np.array_equal(got[j, t], ref[k]), (j, t)
    # decrypted scores of every template vs float64 cosine; top-1 identity
    sc = B.bm_decrypt(st.prm, st.sk, got.reshape(-1, 2, 1, 8192)).reshape(3, -1)[:, :T.shape[0]]
    cos = Q @ T.T
    assert np.abs(sc - cos).max() < 1e-6
    assert np.array_equal(sc.argmax(1), cos.argmax(1))
    assert np.array_equal(sc.argmax(1), expq)


def test_paper_order_parity(env, O):
    T = I.templates(2, 512)
    Q, _ = I.queries(2, 2)
    st = Setup(env, O, 128, 4, T, Q)
    got = st.gpu_match(1)
    ref = st.oracle_pairs([(1, 3), (0, 1)], 1)
    assert np.array_equal(got[1, 3], ref[0]) and np.array_equal(got[0, 1], ref[1])
    hoisted = st.gpu_match(0)
    assert not np.array_equal(hoisted[1, 3], got[1, 3])  # reading R8: orders differ in residues


@pytest.mark.parametrize("chunk", [7, 1])
def test_chunking_ragged(env, O, chunk):
    """Pairs processed in small chunks (option chunk_pairs): 5 queries x 2 sets; chunk 7 gives query
    blocks of 3 + 2 (ragged 2x2 tensor tiles), chunk 1 splits the set range too."""
    torch, B = env
    T = I.random_unit(300, 32, 5)
    Q = I.random_unit(5, 32, 6)
    st = Setup(env, O, 32, 2, T, Q)       # s = 16, B = 256 -> 2 sets; last set ragged (44 templates)
    with B.options(chunk_pairs=chunk):
        got = st.gpu_match(0)
    pairs = [(4, 1), (3, 0), (0, 1)]
    ref = st.oracle_pairs(pairs)
    for k, (j, t) in enumerate(pairs):
        assert np.array_equal(got[j, t], ref[k])
    again = st.gpu_match(0)
    assert np.array_equal(got, again)


@pytest.mark.parametrize("d,p", [(16, 16), (4096, 8), (1024, 1024)])
def test_layout_extremes(env, O, d, p):
    """s = 1 (no ladder, output INTT kernel), the largest d (s = 512, B = 8, 9 rotations) and
    p = 1024 parts (the tensor's 128-bit / FP64 sums are folded mod q every 512 parts)."""
    T = I.random_unit(20, d, d)
    Q = I.random_unit(1, d, d + 1)
    st = Setup(env, O, d, p, T, Q)
    got = st.gpu_match(0)
    ref = st.oracle_pairs([(0, st.n_sets - 1)])
    assert np.array_equal(got[0, st.n_sets - 1], ref[0])
    sc = st.B.bm_decrypt(st.prm, st.sk, got.reshape(-1, 2, 1, 8192)).reshape(-1)[:20]
    assert np.abs(sc - T @ Q[0]).max() < 1e-6


def test_edge_cases_and_errors(env, O):
    torch, B = env
    prm = B.bm_params_init(128, 8)
    sk, pk, evk = B.bm_keygen(prm, 9)
    evk_dev = B.bm_evk_to_device(prm, evk)
    dummy = torch.zeros(8 * 4 * 8192, dtype=torch.int64, device="cuda")   # one set / query / result of any p <= 8
    # empty scans are no-ops
    B.bm_match(prm, evk_dev, dummy, 0, dummy, 3, dummy, None)
    B.bm_match(prm, evk_dev, dummy, 5, dummy, 0, dummy, None)
    # a key set generated for s = 16 lacks the rotations s = 32 needs
    prm4 = B.bm_params_init(128, 4)
    with pytest.raises(B.BMError) as e:
        B.bm_match(prm4, evk_dev, dummy, 1, dummy, 1, dummy, dummy)
    assert e.value.name == "BM_ERR_MISSING_ROTATION_KEY"
    tiny = torch.zeros(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(B.BMError) as e:
        B.bm_match(prm, evk_dev, dummy, 1, dummy, 1, dummy, tiny)
    assert e.value.name == "BM_ERR_WORKSPACE"
    with pytest.raises(B.BMError) as e:
        B.bm_match(prm, evk_dev, dummy, 1, dummy, 1, dummy, dummy, order=7)
    assert e.value.name == "BM_ERR_INVALID_ARG"


@pytest.mark.parametrize("groups", [3, 8])
def test_match_host_pipelined_equals_device(env, O, groups):
    """bm_match_host (host buffers, grouped + overlapped copies) == bm_match on device buffers;
    bm_match_host_ring with a 3-row host ring holds the last 3 queries' rows (query j at row j mod 3)."""
    torch, B = env
    T = I.templates(2, 700)
    Q, _ = I.queries(2, 7)
    st = Setup(env, O, 128, 8, T, Q)
    dev_out = st.gpu_match(0)
    h_q = st.d_q.cpu().pin_memory()
    h_out = torch.empty((st.nq, st.n_sets, 2, 8192), dtype=torch.int64).pin_memory()
    with B.options(host_groups=groups):
        ws = torch.empty(B.bm_match_host_ws_bytes(st.prm, st.n_sets, st.nq), dtype=torch.uint8, device="cuda")
        B.bm_match_host(st.prm, st.evk_dev, st.d_db, st.n_sets, h_q, st.nq, h_out, ws)
        assert np.array_equal(h_out.numpy().view(np.uint64), dev_out)
        ring = torch.zeros((3, st.n_sets, 2, 8192), dtype=torch.int64).pin_memory()
        B.bm_match_host_ring(st.prm, st.evk_dev, st.d_db, st.n_sets, h_q, st.nq, ring, 3, ws)
        for j in range(st.nq - 3, st.nq):
            assert np.array_equal(ring[j % 3].numpy().view(np.uint64), dev_out[j]), j


@pytest.mark.parametrize("nq", [1, 2, 3, 5])
def test_match_host_few_queries(env, O, nq):
    """bm_match_host with fewer queries than its default 4 groups (one query per group; regression: the
    first group used to take all nq < 4 queries into a one-query slot -> BM_ERR_WORKSPACE)."""
    torch, B = env
    T = I.templates(2, 700)
    Q, _ = I.queries(2, nq)
    st = Setup(env, O, 128, 8, T, Q)
    dev_out = st.gpu_match(0)
    h_q = st.d_q.cpu().pin_memory()
    h_out = torch.empty((st.nq, st.n_sets, 2, 8192), dtype=torch.int64).pin_memory()
    ws = torch.empty(B.bm_match_host_ws_bytes(st.prm, st.n_sets, st.nq), dtype=torch.uint8, device="cuda")
    B.bm_match_host(st.prm, st.evk_dev, st.d_db, st.n_sets, h_q, st.nq, h_out, ws)
    assert np.array_equal(h_out.numpy().view(np.uint64), dev_out)


def test_scan_pipelined_streams_equal_device(env, O):
    """bench.py's N > 1 step structure (dist.scan_pipelined: per-group scans on a compute stream,
    collectives on a comm stream) at world size 1 on the GPU == one bm_match over all queries."""
    torch, B = env
    from paper_2408_06167_b200 import dist as pdist
    T = I.templates(2, 700)
    Q, _ = I.queries(2, 8)
    st = Setup(env, O, 128, 8, T, Q)
    ref = st.gpu_match(0)
    G = 4
    gq = st.nq // G
    out = torch.zeros((st.nq, st.n_sets, 2, 8192), dtype=torch.int64, device="cuda")
    ws = torch.empty(B.bm_match_ws_bytes(st.prm, st.n_sets, gq), dtype=torch.uint8, device="cuda")

    def match(g, q_g, out_g):
        B.bm_match(st.prm, st.evk_dev, st.d_db, st.n_sets, q_g, q_g.shape[0], out_g, ws)

    pdist.scan_pipelined(match, st.d_q, out, None, G, torch.cuda.Stream(), torch.cuda.Stream())
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint64), ref)


def test_config2_full_size_bench_launch(env, O):
    """BASELINE.json configs[1] at full size in bench.py's launch configuration: 6,144 templates,
    384 genuine queries, p = 8, all 9,216 (query, set) pairs in one bm_match launch (one chunk).
    Bit-exact parity on sampled pairs (incl. the last query and set), and on sampled queries the
    decrypted scores of every template vs float64 cosine and the top-1 identity."""
    torch, B = env
    T = I.templates(2)
    Q, expq = I.queries(2, 384)
    st = Setup(env, O, 128, 8, T, Q)
    assert st.n_sets * st.nq == 9216
    got = st.gpu_match(0)
    rng = np.random.default_rng(2024)
    pairs = [(383, st.n_sets - 1), (0, 0), (int(rng.integers(384)), int(rng.integers(st.n_sets)))]
    ref = st.oracle_pairs(pairs)
    for k, (j, t) in enumerate(pairs):
        assert np.array_equal(got[j, t], ref[k]), (j, t)
    qs = np.sort(rng.choice(384, 6, replace=False))
    sc = B.bm_decrypt(st.prm, st.sk, got[qs].reshape(-1, 2, 1, 8192)).reshape(len(qs), -1)[:, :T.shape[0]]
    cos = Q[qs] @ T.T
    assert np.abs(sc - cos).max() < 1e-6
    assert np.array_equal(sc.argmax(1), expq[qs])


# ----------------------------------------------------------------------------- f2: hoisted rotation sum
@pytest.mark.parametrize("order", [2, 4])
@pytest.mark.parametrize("d,p,nt", [(16, 1, 256), (128, 8, 6144), (128, 1, 700), (4096, 8, 20), (64, 32, 300),
                                    (64, 16, 300)])
def test_hoisted_rotation_order_parity(env, O, d, p, nt, order):
    """BM_ORDER_HOISTED_ROT / BM_ORDER_BSGS (f2; not the paper's ladder): bit-exact
    vs the oracle's hoisted_rot_sum / bsgs_rot_sum on sampled pairs, scores vs float64 cosine, and the
    same top-1 as the ladder.  s = 16, 16, 128, 512 (the 128-bit sums are folded every 64 rotations),
    2 (BSGS: b = 2, g = 1, one pass) and 4 (b = g = 2)."""
    torch, B = env
    T = I.templates(1) if d == 16 else (I.templates(2, nt) if d == 128 else I.random_unit(nt, d, 3))
    Q = I.queries(1)[0] if d == 16 else (I.queries(2, 3)[0] if d == 128 else I.random_unit(1, d, 4))
    st = Setup(env, O, d, p, T, Q, hoisted=True)
    got = st.gpu_match(order)
    pairs = [(0, st.n_sets - 1)] + ([(Q.shape[0] - 1, 0)] if st.n_sets > 1 or Q.shape[0] > 1 else [])
    ref = st.oracle_pairs(pairs, order)
    for k, (j, t) in enumerate(pairs):
        assert np.array_equal(got[j, t], ref[k]), (j, t)
    sc = B.bm_decrypt(st.prm, st.sk, got.reshape(-1, 2, 1, 8192)).reshape(Q.shape[0], -1)[:, :T.shape[0]]
    cos = Q @ T.T
    assert np.abs(sc - cos).max() < 1e-6
    assert np.array_equal(sc.argmax(1), cos.argmax(1))
    if d == 128 and p == 8:   # residues differ from the ladder's (own parity), decrypted values agree
        lad = st.gpu_match(0)
        assert not np.array_equal(lad[0, 0], got[0, 0])


def test_hoisted_rotation_needs_its_keys(env, O):
    torch, B = env
    prm = B.bm_params_init(128, 8)
    sk, pk, evk = B.bm_keygen(prm, 9)
    evk_dev = B.bm_evk_to_device(prm, evk)
    dummy = torch.zeros(8 * 4 * 8192, dtype=torch.int64, device="cuda")
    with pytest.raises(B.BMError) as e:
        B.bm_match(prm, evk_dev, dummy, 1, dummy, 1, dummy, dummy, order=2)
    assert e.value.name == "BM_ERR_MISSING_ROTATION_KEY"


@pytest.mark.parametrize("d,nt,nq,chunk", [(16, 9000, 3, None), (16, 9000, 3, 4), (128, 300, 2, None),
                                            (1024, 20, 1, None)])
def test_degree2_output_parity(env, O, d, nt, nq, chunk):
    """f2's relin-free degree-2 output (BM_ORDER_DEG2, p = d; R32): every
    (query, set) result (d0, d1, d2) equals the oracle's match_deg2 bit for bit (3 sets with a ragged
    last one at d = 16; chunked into 4-pair rectangles), decrypts with (1, s, s^2) to the float64 cosines
    within 1e-5 (tests/test_oracle_ckks.py::test_deg2_scan_decrypts_with_s_squared derives it), with the
    same top-1; the host-buffer pipeline returns the same rows."""
    torch, B = env
    with B.options(chunk_pairs=chunk or B.bm_get_option("chunk_pairs")):
        _degree2_case(env, O, d, nt, nq)


def _degree2_case(env, O, d, nt, nq):
    torch, B = env
    T = I.random_unit(nt, d, 81)
    Q = T[[5, nt // 2, nt - 1][:nq]] + 0.01 * np.random.default_rng(82).standard_normal((nq, d))
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    st = Setup(env, O, d, d, T, Q)
    got = st.gpu_match(B.ORDER_DEG2)
    pairs = [(j, t) for j in range(st.nq) for t in range(st.n_sets)]
    if len(pairs) > 6:
        pairs = [pairs[0], pairs[len(pairs) // 2], pairs[-1]]
    ref = st.oracle_pairs(pairs, 3)
    for k, (j, t) in enumerate(pairs):
        assert np.array_equal(got[j, t], ref[k]), (j, t)
    sc = B.bm_decrypt_deg2(st.prm, st.sk, got).reshape(st.nq, -1)[:, :nt]
    cos = Q @ T.T
    assert np.abs(sc - cos).max() < 1e-5
    assert np.array_equal(sc.argmax(1), cos.argmax(1))
    h_q = st.d_q.cpu().numpy().view(np.uint64)
    h_out = np.zeros((st.nq, st.n_sets, 3, 8192), np.uint64)
    ws = torch.empty(B.bm_match_host_ws_bytes(st.prm, st.n_sets, st.nq, 3), dtype=torch.uint8, device="cuda")
    B.bm_match_host(st.prm, None, st.d_db, st.n_sets, h_q, st.nq, h_out, ws, order=3)
    assert np.array_equal(h_out, got)


def test_degree2_output_needs_p_equal_d(env, O):
    torch, B = env
    prm = B.bm_params_init(128, 8)
    dummy = torch.zeros(8 * 4 * 8192, dtype=torch.int64, device="cuda")
    with pytest.raises(B.BMError) as e:
        B.bm_match(prm, None, dummy, 1, dummy, 1, dummy, dummy, order=3)
    assert e.value.name == "BM_ERR_INVALID_LAYOUT"
    with pytest.raises(B.BMError) as e:          # the other orders still need their keys
        B.bm_match(prm, None, dummy, 1, dummy, 1, dummy, dummy, order=0)
    assert e.value.name == "BM_ERR_INVALID_ARG"


@pytest.mark.parametrize("order,chunk", [(0, None), (0, 5), (2, None), (4, None), (1, None)])
def test_match_rows_fused_gather(env, O, order, chunk):
    """bm_match_rows (a8 fused into the output kernels, the multi-GPU gather path of dist.P2PGather):
    results land in caller-given rows at global set numbers.  Rows in reversed order inside a wider
    row buffer (n_sets + 3 global sets, this 'rank' at set offset 2) must hold exactly bm_match's
    results, bit for bit, for every op order (ladder, paper order, f2's hoisted rotations; the
    ladder, k_hrot and k_out_intt all store through the same row map), also when chunked; nothing
    outside this rank's set range is touched."""
    torch, B = env
    if chunk:
        B.bm_set_option("chunk_pairs", chunk)
    T = I.random_unit(700, 64, 21)
    Q = I.random_unit(3, 64, 22)
    st = Setup(env, O, 64, 4, T, Q, hoisted=(order in (2, 4)))   # s = 16, B = 256 -> 3 sets
    ref = st.gpu_match(order)
    n_glob, off = st.n_sets + 3, 2
    res = torch.full((st.nq, n_glob, 2, 8192), -1, dtype=torch.int64, device="cuda")
    base, row_bytes = res.data_ptr(), n_glob * 2 * 8192 * 8
    rows = torch.tensor([base + (st.nq - 1 - j) * row_bytes for j in range(st.nq)], dtype=torch.int64,
                        device="cuda")
    ws = torch.empty(max(1, B.bm_match_ws_bytes(st.prm, st.n_sets, st.nq, order)), dtype=torch.uint8, device="cuda")
    B.bm_match_rows(st.prm, st.evk_dev, st.d_db, st.n_sets, st.d_q, st.nq, rows, off, ws, order)
    B.bm_sync()
    got = res.cpu().numpy()
    for j in range(st.nq):
        row = got[st.nq - 1 - j]
        assert np.array_equal(row[off:off + st.n_sets].view(np.uint64), ref[j])
        assert (row[:off] == -1).all() and (row[off + st.n_sets:] == -1).all()
    # the IPC handle of the row buffer (what P2PGather exchanges) and its offset inside the allocation
    h, o = B.bm_ipc_handle(res)
    assert len(h) == 64 and 0 <= o < 1 << 40
    with pytest.raises(ValueError):
        B.bm_match_rows(st.prm, st.evk_dev, st.d_db, st.n_sets, st.d_q, st.nq, rows, -1, ws, order)
    B.bm_set_option("chunk_pairs", 16384)


def test_small_query_batches_swapped_tensor_tiles(env, O):
    """Fewer queries than the tensor tile's query side (cq < 8) with >= 8 sets run k_tensor with the
    roles swapped (sets on the wide side; the Karatsuba products are symmetric): every query's
    results equal those of the same query inside a full batch of 8 bit for bit, for batches of
    1, 3 and 5 (ragged tiles on both sides), and one pair equals the oracle."""
    torch, B = env
    T = I.random_unit(5000, 16, 31)
    Q = I.random_unit(8, 16, 32)
    st = Setup(env, O, 16, 2, T, Q)          # s = 8, B = 512 -> 10 sets
    assert st.n_sets >= 8
    full = st.gpu_match(0)
    for nq in (1, 3, 5):
        for j0 in (0, 8 - nq):
            out = torch.empty((nq, st.n_sets, 2, 8192), dtype=torch.int64, device="cuda")
            ws = torch.empty(B.bm_match_ws_bytes(st.prm, st.n_sets, nq, 0), dtype=torch.uint8, device="cuda")
            B.bm_match(st.prm, st.evk_dev, st.d_db, st.n_sets, st.d_q[j0:j0 + nq], nq, out, ws, 0)
            B.bm_sync()
            assert np.array_equal(out.cpu().numpy().view(np.uint64), full[j0:j0 + nq]), (nq, j0)
    ref = st.oracle_pairs([(7, 9)])
    assert np.array_equal(full[7, 9], ref[0])


@pytest.mark.parametrize("order,c3", [(0, False), (1, False), (0, True), (1, True)])
def test_latency_mode_cluster_ladder(env, O, order, c3):
    """Launches with fewer pairs than half the SMs run the ladder on 2-CTA clusters (k_ladder_t<true>:
    rank c owns component c, c1 copied over DSMEM each step): bit-identical to the one-CTA ladder
    (option ladder_c2 = 0) and to the oracle, for the hoisted and the paper order, s = 16 (4 steps)
    and s = 2 (the last step is the first); likewise the 3-rank pipelined ladder (k_ladder_c3,
    the default at <= n_SM / 3 pairs: the c1 chain in two domains, sigma applied to coefficients)."""
    torch, B = env
    for d, p, n in ((64, 4, 600), (16, 8, 900)):
        T = I.random_unit(n, d, 41)
        Q = I.random_unit(2, d, 42)
        st = Setup(env, O, d, p, T, Q)
        assert 2 * st.nq * st.n_sets <= 148
        # the 3-rank pipelined ladder (k_ladder_c3) is the default at <= n_SM / 3 pairs
        with B.options(ladder_c3=int(c3)):
            got = st.gpu_match(order)
        with B.options(ladder_c2=0):
            ref_gpu = st.gpu_match(order)
        assert np.array_equal(got, ref_gpu), (d, p)
        ref = st.oracle_pairs([(1, st.n_sets - 1)], order)
        assert np.array_equal(got[1, st.n_sets - 1], ref[0]), (d, p)


@pytest.mark.parametrize("extra", [12, 60])
def test_ladder_tail_wave_on_clusters(env, O, extra):
    """A launch of more than n_SM pairs whose last wave is at most half full runs that wave on the
    cluster ladder (floor(np / n_SM) full waves on k_ladder_t<false>, the rest from pair offset
    MatchK::pair0 on k_ladder_c3 when tail <= n_SM / 3, else on k_ladder_t<true>): n_SM + extra pairs
    (extra = 12: the 3-CTA tail; extra = 60: n_SM / 3 < tail <= n_SM / 2, the 2-CTA tail) equal the
    one-kernel launch (option ladder_tail = 0) bit for bit, and a tail pair equals the oracle.  The
    pair count comes from the device's SM count."""
    torch, B = env
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    np_ = n_sm + extra
    assert 0 < extra and 2 * extra <= n_sm and (extra > n_sm // 3) == (extra == 60)
    nq = 1
    n_sets = np_                              # 1 query x n_SM + extra sets of B = 2048 templates
    T = I.random_unit(n_sets * 2048 - 100, 16, 51)
    Q = I.random_unit(nq, 16, 52)
    st = Setup(env, O, 16, 8, T, Q)          # s = 2
    assert st.n_sets * st.nq == np_
    got = st.gpu_match(0)
    with B.options(ladder_tail=0):
        ref_gpu = st.gpu_match(0)
    assert np.array_equal(got, ref_gpu)
    ref = st.oracle_pairs([(0, np_ - 1), (0, np_ - extra)])
    assert np.array_equal(got[0, np_ - 1], ref[0]) and np.array_equal(got[0, np_ - extra], ref[1])


def test_decrypt_dev_equals_host_decrypt(env, O):
    """bm_decrypt_dev (client-side decryption on the device: c0 + c1 s by NTT, FP64 FFT decode) gives
    the scores of the host bm_decrypt (the direct O(N) cosine sum of PAPER.md:347-349's decode) to
    1e-9, and both the float64 cosines to 1e-6; the launch counter sees the kernel."""
    torch, B = env
    T = I.templates(2, 700)
    Q, _ = I.queries(2, 3)
    st = Setup(env, O, 128, 8, T, Q)
    got = st.gpu_match(0)
    host = B.bm_decrypt(st.prm, st.sk, got.reshape(-1, 2, 1, 8192))
    sk_dev = B.bm_sk_to_device(st.prm, st.sk)
    n0 = B.bm_launch_count()
    dev = B.bm_decrypt_dev(st.prm, sk_dev, torch.from_numpy(got.view(np.int64)).cuda())
    B.bm_sync()
    assert B.bm_launch_count() == n0 + 1
    dev = dev.cpu().numpy()
    assert dev.shape == host.shape
    assert np.abs(dev - host).max() < 1e-9
    sc = dev.reshape(st.nq, -1)[:, :T.shape[0]]
    assert np.abs(sc - Q @ T.T).max() < 1e-6
    # the layout (d, p) only selects the score slots: the same ciphertexts decode to S / s scores each
    prm2 = B.bm_params_init(64, 4)
    assert B.bm_decrypt_dev(prm2, sk_dev, torch.from_numpy(got.view(np.int64)).cuda()).shape[1] == prm2.B


def test_binding_validates_sizes(env, O):
    """The binding refuses tensors too small for the scan it describes (the C ABI trusts sizes)."""
    torch, B = env
    prm = B.bm_params_init(128, 8)
    sk, pk, evk = B.bm_keygen(prm, 9)
    evk_dev = B.bm_evk_to_device(prm, evk)
    db = torch.zeros((2, 8, 2, 2, 8192), dtype=torch.int64, device="cuda")
    q = torch.zeros((3, 8, 2, 2, 8192), dtype=torch.int64, device="cuda")
    out = torch.zeros((3, 2, 2, 8192), dtype=torch.int64, device="cuda")
    ws = torch.empty(B.bm_match_ws_bytes(prm, 2, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        B.bm_match(prm, evk_dev, db, 3, q, 3, out, ws)            # 3 sets, 2 present
    with pytest.raises(ValueError):
        B.bm_match(prm, evk_dev, db, 2, q, 4, out, ws)            # 4 queries, 3 present
    with pytest.raises(ValueError):
        B.bm_match(prm, evk_dev, db, 2, q, 3, out[:2], ws)        # output too small
    with pytest.raises(ValueError):
        B.bm_match(prm, evk_dev, db.float(), 2, q, 3, out, ws)    # wrong dtype


def test_rng_os_mode_fresh_encryption_randomness(env, O):
    """BM_RNG_OS: two encryptions of the same plaintext with the same seed and object numbers differ
    (a fresh 160-bit key extension per call) yet both decrypt to it; BM_RNG_SEEDED repeats exactly."""
    torch, B = env
    prm = B.bm_params_init(16, 1)
    sk, pk, evk = B.bm_keygen(prm, 1)
    pk_dev = B.bm_pk_to_device(prm, pk)
    pt = torch.from_numpy(O.encode(O.pack_query(I.random_unit(1, 16, 3), 13, 16, 1).reshape(-1, 4096), 13)).cuda()
    outs = []
    try:
        for mode in (B.RNG_OS, B.RNG_OS, B.RNG_SEEDED, B.RNG_SEEDED):
            B.bm_rng_mode(mode)
            o = torch.empty((1, 2, 2, 8192), dtype=torch.int64, device="cuda")
            B.bm_encrypt(prm, pk_dev, pt, 0, 3, o)
            B.bm_sync()
            outs.append(o)
    finally:
        B.bm_rng_mode(B.RNG_SEEDED)
    assert not torch.equal(outs[0], outs[1]) and torch.equal(outs[2], outs[3])
    for o in (outs[0], outs[1]):
        c = torch.empty_like(o)
        B.bm_ct_to_coeff(prm, o, 2, c)
        B.bm_sync()
        m = O.decrypt(13, B.bm_sk_export(sk), c.cpu().numpy().view(np.uint64)[0], 2)[0]
        err = O.centred_i64(m, prm.q[0]) - pt.cpu().numpy()[0]
        assert np.abs(err).max() < 2 ** 20                 # the encryption noise only


def test_bench_ring_wraparound_equals_bm_match(env, O):
    """bench.py's bounded outputs: query groups written round-robin into R = 2 ring slots on two
    alternating streams (each slot reused every R groups) leave in every slot exactly bm_match's
    results of the last group that used it, bit for bit; sampled pairs equal the oracle."""
    torch, B = env
    T = I.templates(2, 3 * 256 + 40)          # p = 8: B = 256 -> 4 sets (the last ragged)
    Q, _ = I.queries(2, 7)
    st = Setup(env, O, 128, 8, T, Q)
    full = st.gpu_match(0)
    gq, R = 2, 2                              # groups {0,1}, {2,3}, {4,5}, {6}: slot 0 <- groups 0, 2; slot 1 <- 1, 3
    ring = [torch.full((gq, st.n_sets, 2, 8192), -1, dtype=torch.int64, device="cuda") for _ in range(R)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ws = [torch.empty(B.bm_match_ws_bytes(st.prm, st.n_sets, gq), dtype=torch.uint8, device="cuda") for _ in range(2)]
    last = {}
    main = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(main)
    for g in range(-(-st.nq // gq)):
        q0, n = g * gq, min(gq, st.nq - g * gq)
        B.bm_match(st.prm, st.evk_dev, st.d_db, st.n_sets, st.d_q[q0:q0 + n], n, ring[g % R][:n], ws[g % 2], 0,
                   stream=streams[g % 2])
        last[g % R] = (q0, n)
    for s in streams:
        main.wait_stream(s)
    torch.cuda.synchronize()
    for slot, (q0, n) in last.items():
        got = ring[slot][:n].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, full[q0:q0 + n]), slot
    ref = st.oracle_pairs([(6, st.n_sets - 1), (5, 0)])
    assert np.array_equal(full[6, st.n_sets - 1], ref[0]) and np.array_equal(full[5, 0], ref[1])


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_random_layouts_fuzz(env, O, seed):
    """Seeded random layouts (d a power of two in [4, 2048], p | d), template counts (ragged last
    sets) and batch sizes, both op orders: two random pairs per case equal the oracle bit for bit and
    the decrypted scores match the float64 cosines."""
    torch, B = env
    rng = np.random.default_rng(1000 + seed)
    d = int(2 ** rng.integers(2, 12))
    p = int(2 ** rng.integers(0, int(np.log2(d)) + 1))
    Bk = 4096 * p // d
    n_tmpl = int(rng.integers(1, 3 * Bk + 1))
    nq = int(rng.integers(1, 6))
    order = int(rng.integers(0, 2))
    T = I.random_unit(n_tmpl, d, 70 + seed)
    Q = I.random_unit(nq, d, 80 + seed)
    st = Setup(env, O, d, p, T, Q)
    got = st.gpu_match(order)
    pairs = sorted({(int(rng.integers(nq)), int(rng.integers(st.n_sets))) for _ in range(2)})
    ref = st.oracle_pairs(pairs, order)
    for k, (j, t) in enumerate(pairs):
        assert np.array_equal(got[j, t], ref[k]), (d, p, n_tmpl, nq, order, j, t)
    sc = B.bm_decrypt(st.prm, st.sk, got.reshape(-1, 2, 1, 8192)).reshape(nq, -1)[:, :n_tmpl]
    assert np.abs(sc - Q @ T.T).max() < 1e-6, (d, p)
