"""K1 on the tensor cores (k_tensor_mma: tcgen05.mma kind::i8, k_tensor_mma.cuh) against the CUDA-core
K1 (k_tensor) and the CPU oracle.

The byte-split contraction must give the same canonical residues d0, d1, d2 as the 128-bit
multiply-accumulate, so bm_match's outputs for a DB registered in the tensor-core layout
(bm_db_tc_register) are compared bit for bit with the option tensor_mma on and off (the library's
launch counter shows which K1 ran: the tensor-core K1 is two launches, the
query-operand expansion and the MMA kernel), on uniform residues and on the extreme q - 1 everywhere
(the largest byte sums the s32 accumulators see), over ragged set and query tiles, chunking, p = 4 and
8, and then against the oracle on a shape the MMA path takes."""
import numpy as np
import pytest

from paper_2408_06167_b200 import inputs as I

pytestmark = pytest.mark.gpu

LOGN = 13
N = 1 << LOGN


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: the GPU tests need a B200 (there is no CPU fallback)")
    from paper_2408_06167_b200 import build
    build.build(verbose=False)
    from paper_2408_06167_b200 import bm
    return torch, bm


def residues(O, shape, seed, pattern):
    """[..., 2 comps, 2 limbs, N] canonical NTT-domain residues (uniform, or q - 1 everywhere)."""
    q0, q1, _ = O.primes()
    rng = np.random.default_rng(seed)
    out = np.empty(shape + (2, 2, N), np.uint64)
    for li, q in enumerate((q0, q1)):
        if pattern == "qm1":
            out[..., li, :] = np.uint64(q - 1)
        else:
            out[..., li, :] = rng.integers(0, q, size=shape + (2, N), dtype=np.uint64)
    return out


def run(torch, B, prm, evk_dev, d_db, n_sets, d_q, nq, mma):
    B.bm_set_option("tensor_mma", 1 if mma else 0)
    out = torch.empty((nq, n_sets, 2, N), dtype=torch.int64, device="cuda")
    ws = torch.empty(B.bm_match_ws_bytes(prm, n_sets, nq, 0), dtype=torch.uint8, device="cuda")
    B.bm_sync()
    n0 = B.bm_launch_count()
    B.bm_match(prm, evk_dev, d_db, n_sets, d_q, nq, out, ws, 0)
    B.bm_sync()
    n = B.bm_launch_count() - n0
    B.bm_set_option("tensor_mma", 1)
    return out.cpu().numpy(), n


@pytest.mark.parametrize("d,p,n_sets,nq,chunk,pattern,n_mma", [
    (128, 8, 300, 8, None, "uni", 1),     # 3 set tiles, the last one ragged (44 of 128)
    (128, 8, 130, 13, None, "uni", 1),    # 2 query tiles (the second holds 5 queries), 2 set tiles
    (128, 8, 256, 8, None, "qm1", 1),     # the largest byte sums (s32 accumulators, the 2^40 fold)
    (64, 4, 200, 6, None, "uni", 1),      # p = 4: one K = 32 MMA per component product
    (64, 4, 128, 8, None, "qm1", 1),
    (128, 8, 300, 16, 2048, "uni", 2),    # chunks of 8 x 256 sets (MMA) and 8 x 44 sets (CUDA-core K1), twice
    (128, 8, 300, 8, 1040, "uni", 1),     # chunks of 130 sets: only the first starts on a 128-set tile
])
def test_tensor_mma_equals_cuda_core(env, O, d, p, n_sets, nq, chunk, pattern, n_mma):
    torch, B = env
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    evk_dev = B.bm_evk_to_device(prm, evk)
    d_db = torch.from_numpy(residues(O, (n_sets, p), 11, pattern).view(np.int64)).cuda()
    d_q = torch.from_numpy(residues(O, (nq, p), 12, pattern).view(np.int64)).cuda()
    packed = torch.empty(B.bm_db_tc_bytes(prm, n_sets), dtype=torch.uint8, device="cuda")
    B.bm_db_tc_register(prm, d_db, n_sets, packed)
    if chunk:
        B.bm_set_option("chunk_pairs", chunk)
    try:
        ref, n_ref = run(torch, B, prm, evk_dev, d_db, n_sets, d_q, nq, False)
        got, n_got = run(torch, B, prm, evk_dev, d_db, n_sets, d_q, nq, True)
    finally:
        B.bm_set_option("chunk_pairs", 16384)
        B.bm_db_tc_unregister(d_db)
    assert n_got == n_ref + n_mma, (n_got, n_ref)   # one more K1 launch per chunk that took the MMA path
    assert np.array_equal(got, ref)


def test_tensor_mma_oracle_parity(env, O):
    """A shape the MMA path takes (64 sets of 256 templates, 8 queries, d = 128, p = 8) against the
    CPU oracle: sampled pairs bit-exact, every score within 1e-6 of the cosine."""
    import test_gpu_parity as G
    torch, B = env
    T = I.random_unit(64 * 256, 128, 31)
    Q = I.random_unit(8, 128, 32)
    st = G.Setup(env, O, 128, 8, T, Q)
    assert st.n_sets == 64
    packed = torch.empty(B.bm_db_tc_bytes(st.prm, st.n_sets), dtype=torch.uint8, device="cuda")
    B.bm_db_tc_register(st.prm, st.d_db, st.n_sets, packed)
    counts = []
    for mma in (0, 1):
        B.bm_set_option("tensor_mma", mma)
        n0 = B.bm_launch_count()
        got = st.gpu_match(0)
        counts.append(B.bm_launch_count() - n0)
    assert counts[1] == counts[0] + 1            # the tensor-core K1 (query expansion + MMA kernel) ran
    B.bm_db_tc_unregister(st.d_db)
    pairs = [(0, 0), (7, 63), (3, 17), (5, 40)]
    ref = st.oracle_pairs(pairs)
    for k, (j, t) in enumerate(pairs):
        assert np.array_equal(got[j, t], ref[k])
    sc = B.bm_decrypt(st.prm, st.sk, got.reshape(-1, 2, 1, N))
    sc = np.asarray(sc).reshape(8, 64, -1)[:, :, :256].reshape(8, -1)
    cos = Q @ T.T
    assert np.abs(sc - cos).max() < 1e-6


def test_tensor_mma_registration(env, O):
    """An unregistered DB takes the CUDA-core K1; register / unregister validate their arguments."""
    torch, B = env
    prm = B.bm_params_init(128, 8)
    sk, pk, evk = B.bm_keygen(prm, 1)
    evk_dev = B.bm_evk_to_device(prm, evk)
    d_db = torch.from_numpy(residues(O, (130, 8), 41, "uni").view(np.int64)).cuda()
    d_q = torch.from_numpy(residues(O, (8, 8), 42, "uni").view(np.int64)).cuda()
    ref, n_off = run(torch, B, prm, evk_dev, d_db, 130, d_q, 8, True)       # not registered
    packed = torch.empty(B.bm_db_tc_bytes(prm, 130), dtype=torch.uint8, device="cuda")
    assert B.bm_db_tc_bytes(prm, 130) == 2 * 8192 * 128 * 16 * 8 * 2      # two 128-set tiles
    B.bm_db_tc_register(prm, d_db, 130, packed)
    B.bm_db_tc_register(prm, d_db, 130, packed)                            # again: replaces the entry
    got, n_on = run(torch, B, prm, evk_dev, d_db, 130, d_q, 8, True)
    assert n_on == n_off + 1 and np.array_equal(got, ref)
    B.bm_db_tc_unregister(d_db)
    with pytest.raises(B.BMError):
        B.bm_db_tc_unregister(d_db)
    with pytest.raises(ValueError):
        B.bm_db_tc_register(prm, d_db, 130, packed[:1000])
    assert B.bm_db_tc_bytes(B.bm_params_init(128, 2), 130) == 0           # p = 2: no tensor-core layout
