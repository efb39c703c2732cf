"""CPU-side checks of the C-ABI library: it loads, exports every symbol include/blindmatch.h
declares, and its host (client-side) functions -- key generation, packing/encoding,
decryption -- agree with the oracle.  No kernel is launched here."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2408_06167_b200 import inputs as I

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "blindmatch.h")


@pytest.fixture(scope="module")
def B():
    from paper_2408_06167_b200 import build
    build.build(verbose=False)
    from paper_2408_06167_b200 import bm
    return bm


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bm_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(B):
    lib = ctypes.CDLL(B.LIB_PATH)
    names = _declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    # the Python binding wraps every declared function under the same name
    assert set(names) == set(B.EXPORTED)


def test_params_and_errors(B):
    prm = B.bm_params_init(128, 8)
    assert (prm.N, prm.slots, prm.s, prm.B, prm.log_s) == (8192, 4096, 16, 256, 4)
    assert list(prm.q) == [2 ** 58 - 835583, 2 ** 40 - 147455, 2 ** 60 - 16383]
    assert prm.scale == 2.0 ** 40 and prm.out_scale == 2.0 ** 80 / prm.q[1]
    for d, p in ((3, 1), (16, 32), (8192, 1), (16, 0)):
        with pytest.raises(B.BMError) as e:
            B.bm_params_init(d, p)
        assert e.value.name == "BM_ERR_INVALID_LAYOUT"


@pytest.mark.parametrize("d,p", [(16, 1), (128, 4)])
def test_keygen_matches_oracle(B, O, d, p):
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 12345)
    osk, opk, orlk, ogk = O.keygen(13, 12345, O.n_rot_for(d, p))
    assert np.array_equal(B.bm_sk_export(sk), osk)
    assert np.array_equal(B.bm_pk_export(pk), opk)
    rlk, gk = B.bm_evk_export(evk)
    assert np.array_equal(rlk, orlk)
    assert gk.shape[0] == prm.log_s and np.array_equal(gk, ogk)


def test_encoder_within_one_of_oracle(B, O):
    """Product FFT encoder vs the oracle's encoder: identical up to the FP rounding of
    half-way cases (reading R15): |diff| <= 1 and almost all coefficients equal."""
    prm = B.bm_params_init(128, 4)
    T = I.templates(2, 300)
    pt = B.bm_encode_db(prm, T, 0, 3)
    z = O.pack_db(T, 13, 128, 4, 0, 3).reshape(-1, 4096)
    opt = O.encode(z, 13).reshape(pt.shape)
    diff = np.abs(pt - opt)
    assert diff.max() <= 1 and (diff != 0).mean() < 1e-3
    Q, _ = I.queries(2, 5)
    pq = B.bm_encode_query(prm, Q)
    oq = O.encode(O.pack_query(Q, 13, 128, 4).reshape(-1, 4096), 13).reshape(pq.shape)
    dq = np.abs(pq - oq)
    assert dq.max() <= 1 and (dq != 0).mean() < 1e-3


def test_encode_errors(B):
    prm = B.bm_params_init(16, 1)
    with pytest.raises(B.BMError) as e:
        B.bm_encode_query(prm, np.zeros((1, 16)))
    assert e.value.name == "BM_ERR_ZERO_VECTOR"
    bad = np.ones((1, 16))
    bad[0, 3] = np.nan
    with pytest.raises(B.BMError) as e:
        B.bm_encode_query(prm, bad)
    assert e.value.name == "BM_ERR_MAGNITUDE"


def test_decrypt_matches_oracle(B, O):
    """Client-side decryption of an oracle-made level-0 scan result."""
    d, p = 16, 1
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    osk, opk, orlk, ogk = O.keygen(13, 1, O.n_rot_for(d, p))
    T = I.templates(1)
    Q, _ = I.queries(1)
    zdb = O.pack_db(T, 13, d, p, 0, 1)
    db = O.encrypt(13, opk, O.encode(zdb.reshape(-1, 4096), 13), 0, 2).reshape(1, p, 2, 2, -1)
    qc = O.encrypt(13, opk, O.encode(O.pack_query(Q, 13, d, p).reshape(-1, 4096), 13), 0, 3).reshape(1, p, 2, 2, -1)
    out, _ = O.match(13, d, p, 0, orlk, ogk, db, qc)
    m = B.bm_decrypt_raw(prm, sk, out)
    q0 = prm.q[0]
    om = O.decrypt(13, osk, out[0], 1)[0]
    assert np.array_equal(m[0], O.centred_i64(om, q0))
    sc = B.bm_decrypt(prm, sk, out)[0]
    osc = O.scores_from_output(13, d, p, osk, out[0], q0)
    assert np.abs(sc - osc).max() < 1e-9
    assert B.bm_top1(sc)[0] == 17
    assert B.bm_top1(np.array([0.5, 0.7, 0.7, 0.1]))[0] == 1   # lowest index wins ties


def test_decrypt_deg2_matches_oracle(B, O):
    """Client-side decryption (1, s, s^2) of an oracle-made degree-2 result (f2 BM_ORDER_DEG2, p = d)."""
    d = p = 16
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    osk, opk, orlk, ogk = O.keygen(13, 1, 0)
    T = I.random_unit(200, d, 5)
    Q = I.random_unit(1, d, 6)
    db = O.encrypt(13, opk, O.encode(O.pack_db(T, 13, d, p, 0, 1).reshape(-1, 4096), 13), 0, 2).reshape(1, p, 2, 2, -1)
    qc = O.encrypt(13, opk, O.encode(O.pack_query(Q, 13, d, p).reshape(-1, 4096), 13), 0, 3).reshape(1, p, 2, 2, -1)
    out, _ = O.match_deg2(13, d, p, db, qc)
    sc = B.bm_decrypt_deg2(prm, sk, out.reshape(1, 3, -1))[0]
    q0 = prm.q[0]
    om = O.decrypt_deg2(13, osk, out[0].reshape(3, -1))
    osc = O.decode_slots(O.centred_i64(om, q0), 13, prm.out_scale)
    assert np.abs(sc - osc[:prm.B]).max() < 1e-9
    assert np.abs(sc[:200] - T @ Q[0]).max() < 1e-5
    with pytest.raises(B.BMError):                     # residues must be canonical
        B.bm_decrypt_deg2(prm, sk, np.full((1, 3, 8192), q0, np.uint64))


def test_key_import_roundtrip(B):
    prm = B.bm_params_init(32, 2)
    sk, pk, evk = B.bm_keygen(prm, 77)
    rlk, gk = B.bm_evk_export(evk)
    evk2 = B.bm_evk_import(prm, rlk, gk)
    r2, g2 = B.bm_evk_export(evk2)
    assert np.array_equal(r2, rlk) and np.array_equal(g2, gk)
    pk2 = B.bm_pk_import(prm, B.bm_pk_export(pk))
    assert np.array_equal(B.bm_pk_export(pk2), B.bm_pk_export(pk))
    bad = rlk.copy()
    bad[0, 0, 0, 0] = prm.q[0]
    with pytest.raises(B.BMError):
        B.bm_evk_import(prm, bad, gk)


def test_device_calls_fail_loudly_without_gpu(B):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    prm = B.bm_params_init(16, 1)
    sk, pk, evk = B.bm_keygen(prm, 1)
    with pytest.raises(B.BMError) as e:
        B.bm_evk_to_device(prm, evk)
    assert e.value.name == "BM_ERR_CUDA"


def test_fused_gather_entry_points_validate_arguments(B):
    """bm_match_rows / bm_ipc_*: argument errors are reported before any device work (callable
    without a GPU), and the IPC calls fail with BM_ERR_CUDA, not a crash, when there is no device."""
    import ctypes
    import torch
    lib = B._lib
    prm = B.bm_params_init(16, 1)
    P = ctypes.byref(prm)
    one = ctypes.c_void_p(8)   # never dereferenced: the argument checks come first
    # NULL evk, NULL row table (checked before the key digest is read)
    assert lib.bm_match_rows(P, None, one, 1, one, 1, one, 0, one, 1, 0, None) == -1
    assert lib.bm_match_rows(P, one, one, 1, one, 1, None, 0, one, 1, 0, None) == -1
    h = (ctypes.c_uint8 * 64)()
    off = ctypes.c_uint64(0)
    assert lib.bm_ipc_handle(None, h, ctypes.byref(off)) == -1
    assert lib.bm_ipc_open(None, ctypes.byref(ctypes.c_void_p())) == -1
    assert lib.bm_ipc_close(None) == -1
    if not torch.cuda.is_available():
        assert lib.bm_ipc_handle(one, h, ctypes.byref(off)) == -5          # BM_ERR_CUDA
        assert lib.bm_ipc_open(h, ctypes.byref(ctypes.c_void_p())) == -5


# ----------------------------------------------------------------------------- f3 host side
@pytest.mark.parametrize("d,p", [(128, 8), (16, 1)])
def test_expansion_keys_match_oracle(B, O, d, p):
    """f3: the product's expansion keys (pk limb q2, level-1 Galois keys of strides s 2^t) equal
    the oracle's bit for bit (independent implementations of reading R26)."""
    prm = B.bm_params_init(d, p)
    assert prm.q2 == O.q2()
    xk = B.bm_xk_keygen(prm, 4242)
    pk_q2, gk1 = B.bm_xk_export(xk)
    opk_q2, ogk1 = O.keygen_exp(13, 4242, d, p, n_rot=O.n_rot_enroll(13, d, p))   # log2 B strides (f3 + f4)
    assert np.array_equal(pk_q2, opk_q2)
    assert gk1.shape == ogk1.shape and np.array_equal(gk1, ogk1)
    xk2 = B.bm_xk_import(prm, pk_q2, gk1)
    a, b = B.bm_xk_export(xk2)
    assert np.array_equal(a, pk_q2) and np.array_equal(b, gk1)
    bad = pk_q2.copy()
    bad[0, 0] = prm.q2
    with pytest.raises(B.BMError):
        B.bm_xk_import(prm, bad, gk1)


def test_expansion_encoders_within_one_of_oracle(B, O):
    """f3 client encoders: the tiled query (scale 2^40) and the masks X_i (scale q2) agree with the
    oracle's encoder up to half-way FP roundings (reading R15)."""
    prm = B.bm_params_init(128, 8)
    Q, _ = I.queries(2, 6)
    pq = B.bm_encode_query_tiled(prm, Q)
    oq = O.encode(O.tile_query(Q, 13, 128), 13)
    assert np.abs(pq - oq).max() <= 1 and (pq != oq).mean() < 1e-3
    pm = B.bm_encode_masks(prm)
    om = O.expand_masks(13, 128, 8)
    assert np.abs(pm - om).max() <= 1 and (pm != om).mean() < 1e-3
    pe = B.bm_encode_masks(prm, B.MASK_ENROLL)
    oe = O.enroll_masks(13, 128, 8)
    assert np.abs(pe - oe).max() <= 1 and (pe != oe).mean() < 1e-3
    T = I.templates(2, 7)
    pv = B.bm_encode_enroll(prm, T)
    ov = O.encode(O.enroll_vector(T / np.linalg.norm(T, axis=1, keepdims=True), 13, 128), 13)
    assert np.abs(pv - ov).max() <= 1 and (pv != ov).mean() < 1e-3



# ----------------------------------------------------------------------------- f1 host side
@pytest.mark.parametrize("d,p", [(16, 4), (128, 8)])
def test_compression_keys_match_oracle(B, O, d, p):
    """f1: the product's rlk2 / level-1 ladder keys / level-0 right-rotation keys equal the oracle's."""
    prm = B.bm_params_init(d, p)
    ck = B.bm_ck_keygen(prm, 99)
    rlk2, gkl, gkc = B.bm_ck_export(prm, ck)
    orlk2, ogkl, ogkc = O.keygen_cmp(13, 99, d, p)
    assert np.array_equal(rlk2, orlk2)
    assert gkl.shape == ogkl.shape and np.array_equal(gkl, ogkl)
    assert gkc.shape == ogkc.shape and np.array_equal(gkc, ogkc)
    m = B.bm_encode_cmp_mask(prm)
    om = O.cmp_mask(13, d, p)
    assert np.abs(m - om).max() <= 1 and (m != om).mean() < 1e-3



# ----------------------------------------------------------------------------- serialisation
def test_ciphertext_frame_roundtrip_and_errors(B, O):
    """bm_ct_export / bm_ct_import: oracle ciphertexts of levels 0, 1, 2 survive the
    frame bit for bit with level and scale; other params, a bad magic, a short buffer and a
    non-canonical residue are rejected."""
    prm = B.bm_params_init(16, 1)
    sk, pk, rlk, gk = O.keygen(13, 1, 0)
    pk_q2, _ = O.keygen_exp(13, 1, 16, 1)
    pt = O.encode(np.random.default_rng(3).uniform(-1, 1, (2, 4096)), 13)
    c1 = O.encrypt(13, pk, pt, 0, 9)
    c2 = O.encrypt_l2(13, pk, pk_q2, pt, 0, 9)
    c0 = np.ascontiguousarray(c1[:, :, :1, :])
    for ct, lev, sc in ((c0, 0, 2.0 ** 80 / prm.q[1]), (c1, 1, 2.0 ** 40), (c2, 2, 2.0 ** 40)):
        data = B.bm_ct_export(prm, ct, lev, sc)
        assert len(data) == 64 + ct.size * 8 and data[:4] == b"BMCT"
        back, lev2, sc2 = B.bm_ct_import(prm, data)
        assert lev2 == lev and sc2 == sc and np.array_equal(back, ct)
    data = B.bm_ct_export(prm, c1, 1, 2.0 ** 40)
    other = bytearray(data)
    other[8] ^= 1                                      # a frame made under another parameter digest
    with pytest.raises(B.BMError) as e:
        B.bm_ct_import(prm, bytes(other))
    assert e.value.name == "BM_ERR_KEY_MISMATCH"
    with pytest.raises(B.BMError):
        B.bm_ct_import(prm, b"XXXX" + data[4:])
    with pytest.raises(B.BMError):
        B.bm_ct_import(prm, data[:-8])
    bad = c1.copy()
    bad[0, 1, 1, 5] = prm.q[1]
    with pytest.raises(B.BMError):
        B.bm_ct_export(prm, bad, 1, 2.0 ** 40)


def test_rng_modes(B):
    """BM_RNG_OS (the library default): the keygen family draws a 160-bit process key from getrandom()
    -- the same seed gives the same secret within the process (so bm_xk_keygen / bm_ck_keygen /
    bm_evk_add_hoisted stay consistent with bm_keygen) but not the seeded-mode (oracle) secret;
    BM_RNG_SEEDED restores the deterministic streams.  Unknown modes are refused; the options and the
    launch counter are process-wide and validated."""
    prm = B.bm_params_init(16, 1)
    assert B.bm_get_rng_mode() == B.RNG_SEEDED          # conftest selects the test mode
    seeded = B.bm_sk_export(B.bm_keygen(prm, 7)[0])
    try:
        B.bm_rng_mode(B.RNG_OS)
        a = B.bm_sk_export(B.bm_keygen(prm, 7)[0])
        b = B.bm_sk_export(B.bm_keygen(prm, 7)[0])
        assert np.array_equal(a, b)                      # one process key
        assert not np.array_equal(a, seeded)             # 224-bit key, not the 64-bit seed alone
        assert set(np.unique(a)) <= {-1, 0, 1}
    finally:
        B.bm_rng_mode(B.RNG_SEEDED)
    assert np.array_equal(B.bm_sk_export(B.bm_keygen(prm, 7)[0]), seeded)
    with pytest.raises(B.BMError):
        B.bm_rng_mode(5)
    with pytest.raises(B.BMError):
        B.bm_set_option("chunk_pairs", 0)
    with pytest.raises(B.BMError):
        B.bm_set_option("ladder_c2", 2)
    with B.options(chunk_pairs=33):
        assert B.bm_get_option("chunk_pairs") == 33
    assert B.bm_get_option("chunk_pairs") == 16384
    assert B.bm_launch_count() >= 0
    # the tensor-core K1's switch and the packed DB's size (host-only calls)
    assert B.bm_get_option("tensor_mma") == 1
    with pytest.raises(B.BMError):
        B.bm_set_option("tensor_mma", 2)
    with B.options(tensor_mma=0):
        assert B.bm_get_option("tensor_mma") == 0
    assert B.bm_get_option("tensor_mma") == 1
    for d, p, n_sets, tiles in [(128, 8, 1, 1), (128, 8, 128, 1), (128, 8, 129, 2), (64, 4, 4096, 32)]:
        assert B.bm_db_tc_bytes(B.bm_params_init(d, p), n_sets) == tiles * 2 * 8192 * 128 * 16 * p
    assert B.bm_db_tc_bytes(B.bm_params_init(128, 1), 100) == 0        # p not 4 or 8: no tensor-core layout
    assert B.bm_db_tc_bytes(B.bm_params_init(128, 16), 100) == 0
    assert B.bm_db_tc_bytes(B.bm_params_init(128, 8), 0) == 0
