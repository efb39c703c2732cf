"""Thin ctypes binding of libblindmatch (include/blindmatch.h).  Argument marshalling only:
every step of the scan runs in the library's sm_100a kernels.  PyTorch supplies device
memory (tensor.data_ptr()) and streams (torch.cuda.current_stream().cuda_stream).

Importing this module fails loudly if libblindmatch.so is missing: there is no CPU fallback.
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BM_LIB_PATH") or os.path.join(_PKG, "libblindmatch.so")   # override: A/B builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2408_06167_b200.build` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

N = 8192
SLOTS = 4096
ORDER_HOISTED = 0
ORDER_PAPER = 1
ORDER_HOISTED_ROT = 2   # f2: hoisted rotation sum, not the paper's ladder
ORDER_DEG2 = 3          # f2: relin-free degree-2 output (p = d), [nq][n_sets][3][N]; bm_decrypt_deg2
ORDER_BSGS = 4          # f2: baby-step giant-step rotation sum (hoisted keys), not the paper's ladder

BM_OK = 0
ERRORS = {
    -1: "BM_ERR_INVALID_ARG", -2: "BM_ERR_INVALID_LAYOUT", -3: "BM_ERR_INSECURE_PARAMS", -4: "BM_ERR_INVALID_PRIME",
    -5: "BM_ERR_CUDA", -6: "BM_ERR_OOM", -7: "BM_ERR_ZERO_VECTOR", -8: "BM_ERR_MAGNITUDE", -9: "BM_ERR_CAPACITY",
    -10: "BM_ERR_LEVEL", -11: "BM_ERR_MISSING_ROTATION_KEY", -12: "BM_ERR_KEY_MISMATCH", -13: "BM_ERR_WORKSPACE",
}


class BMError(RuntimeError):
    def __init__(self, code, fn):
        self.code = code
        self.name = ERRORS.get(code, str(code))
        super().__init__(f"{fn}: {self.name} ({_lib.bm_strerror(code).decode()})")


class bm_params(ctypes.Structure):
    _fields_ = [("logN", ctypes.c_int32), ("N", ctypes.c_int32), ("slots", ctypes.c_int32),
                ("d", ctypes.c_int32), ("p", ctypes.c_int32), ("s", ctypes.c_int32), ("B", ctypes.c_int32),
                ("log_s", ctypes.c_int32), ("q", ctypes.c_uint64 * 3), ("scale", ctypes.c_double),
                ("out_scale", ctypes.c_double), ("digest", ctypes.c_uint8 * 32), ("q2", ctypes.c_uint64)]


_vp = ctypes.c_void_p
_i32, _i64, _u64, _sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
_P = ctypes.POINTER(bm_params)
_pp = ctypes.POINTER(ctypes.c_void_p)

_SIGS = {
    "bm_params_init": (_i32, [_P, _i32, _i32]),
    "bm_rng_mode": (_i32, [_i32]), "bm_get_rng_mode": (_i32, []),
    "bm_keygen": (_i32, [_P, _u64, _pp, _pp, _pp]),
    "bm_evk_add_hoisted": (_i32, [_P, _u64, _vp]),
    "bm_sk_free": (None, [_vp]), "bm_pk_free": (None, [_vp]), "bm_evk_free": (None, [_vp]),
    "bm_sk_export": (_i32, [_vp, _vp]), "bm_pk_export": (_i32, [_vp, _vp]),
    "bm_evk_export": (_i32, [_vp, _vp, _vp, ctypes.POINTER(_i32)]),
    "bm_sk_import": (_i32, [_P, _vp, _pp]), "bm_pk_import": (_i32, [_P, _vp, _pp]),
    "bm_evk_import": (_i32, [_P, _vp, _vp, _i32, _pp]),
    "bm_pk_to_device": (_i32, [_P, _vp, _pp]), "bm_evk_to_device": (_i32, [_P, _vp, _pp]),
    "bm_pk_dev_free": (None, [_vp]), "bm_evk_dev_free": (None, [_vp]),
    "bm_encode_db": (_i32, [_P, _vp, _i64, _i64, _i64, _vp]),
    "bm_encode_query": (_i32, [_P, _vp, _i64, _vp]),
    "bm_encrypt": (_i32, [_P, _vp, _vp, _i64, _u64, _u64, _vp, _vp]),
    "bm_encrypt_db": (_i32, [_P, _vp, _vp, _i64, _i64, _i64, _u64, _vp, _vp]),
    "bm_encrypt_query": (_i32, [_P, _vp, _vp, _i64, _i64, _u64, _vp, _vp]),
    "bm_ct_to_coeff": (_i32, [_P, _vp, _i64, _i32, _vp, _vp]),
    "bm_ct_from_coeff": (_i32, [_P, _vp, _i64, _i32, _vp, _vp]),
    "bm_match_ws_bytes": (_sz, [_P, _i64, _i32, _i32]),
    "bm_db_tc_bytes": (_sz, [_P, _i64]),
    "bm_db_tc_register": (_i32, [_P, _vp, _i64, _vp, _sz, _vp]),
    "bm_db_tc_unregister": (_i32, [_vp]),
    "bm_match": (_i32, [_P, _vp, _vp, _i64, _vp, _i32, _vp, _vp, _sz, _i32, _vp]),
    "bm_match_rows": (_i32, [_P, _vp, _vp, _i64, _vp, _i32, _vp, _i64, _vp, _sz, _i32, _vp]),
    "bm_ipc_handle": (_i32, [_vp, _vp, ctypes.POINTER(_u64)]),
    "bm_ipc_open": (_i32, [_vp, _pp]), "bm_ipc_close": (_i32, [_vp]),
    "bm_match_host_ws_bytes": (_sz, [_P, _i64, _i32, _i32]),
    "bm_match_host": (_i32, [_P, _vp, _vp, _i64, _vp, _i32, _vp, _vp, _sz, _i32, _vp]),
    "bm_set_profiling": (None, [_i32]), "bm_profile_reset": (None, []),
    "bm_profile_read": (_i32, [_vp, _vp, _vp]),
    "bm_decrypt": (_i32, [_P, _vp, _vp, _i64, _vp]),
    "bm_decrypt_raw": (_i32, [_P, _vp, _vp, _i64, _vp]),
    "bm_decrypt_deg2": (_i32, [_P, _vp, _vp, _i64, _vp]),
    "bm_ct_export": (_i32, [_P, _vp, _i64, _i32, ctypes.c_double, _vp, ctypes.POINTER(_sz)]),
    "bm_ct_import": (_i32, [_P, _vp, _sz, _vp, ctypes.POINTER(_i64), ctypes.POINTER(_i32),
                            ctypes.POINTER(ctypes.c_double)]),
    "bm_top1": (_i32, [_vp, _i64, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_double)]),
    # f3: server-side query expansion (Algorithm 1) on the chain extended by q2
    "bm_xk_keygen": (_i32, [_P, _u64, _pp]), "bm_xk_free": (None, [_vp]),
    "bm_xk_export": (_i32, [_vp, _vp, _vp, ctypes.POINTER(_i32)]),
    "bm_xk_import": (_i32, [_P, _vp, _vp, _i32, _pp]),
    "bm_xk_to_device": (_i32, [_P, _vp, _vp, _vp, _vp, _pp]), "bm_xk_dev_free": (None, [_vp]),
    "bm_encode_query_tiled": (_i32, [_P, _vp, _i64, _vp]),
    "bm_encode_enroll": (_i32, [_P, _vp, _i64, _vp]),
    "bm_encode_masks": (_i32, [_P, _i32, _vp]),
    "bm_enroll_ws_bytes": (_sz, [_P, _i64]),
    "bm_enroll": (_i32, [_P, _vp, _vp, _i64, _i64, _vp, _i64, _vp, _sz, _vp]),
    "bm_encrypt_l2": (_i32, [_P, _vp, _vp, _i64, _u64, _u64, _vp, _vp]),
    "bm_expand_ws_bytes": (_sz, [_P, _i32]),
    "bm_expand": (_i32, [_P, _vp, _vp, _i32, _vp, _vp, _sz, _vp]),
    # f1: output compression (HE-C^3 one level up)
    "bm_ck_keygen": (_i32, [_P, _u64, _pp]), "bm_ck_free": (None, [_vp]),
    "bm_ck_export": (_i32, [_vp, _vp, _vp, _vp]),
    "bm_encode_cmp_mask": (_i32, [_P, _vp]),
    "bm_ck_to_device": (_i32, [_P, _vp, _vp, _pp]), "bm_ck_dev_free": (None, [_vp]),
    "bm_match_cmp_ws_bytes": (_sz, [_P, _i64, _i32]),
    "bm_match_cmp": (_i32, [_P, _vp, _vp, _i64, _vp, _i32, _vp, _vp, _sz, _vp]),
    "bm_decrypt_packed": (_i32, [_P, _vp, _vp, _i64, _vp]),
    "bm_sk_to_device": (_i32, [_P, _vp, _pp]), "bm_sk_dev_free": (None, [_vp]),
    "bm_decrypt_dev": (_i32, [_P, _vp, _vp, _i64, _vp, _vp]),
    "bm_match_host_ring": (_i32, [_P, _vp, _vp, _i64, _vp, _i32, _vp, _i32, _vp, _sz, _i32, _vp]),
    "bm_set_option": (_i32, [_i32, _i64]), "bm_get_option": (_i64, [_i32]),
    "bm_launch_count": (_i64, []), "bm_launch_count_reset": (None, []),
    "bm_sync": (_i32, [_vp]),
    "bm_strerror": (ctypes.c_char_p, [_i32]),
    "bm_build_info": (ctypes.c_char_p, []),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = sorted(_SIGS)


def _chk(rc, fn):
    if rc != BM_OK:
        raise BMError(rc, fn)


def _np_ptr(a):
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("expected a C-contiguous numpy array")
    return ctypes.c_void_p(a.ctypes.data)


def _dptr(t):
    """device pointer of a contiguous CUDA tensor"""
    if not (t.is_cuda and t.is_contiguous()):
        raise ValueError("expected a contiguous CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _need(t, n_u64, name):
    """a CUDA tensor of 8-byte integers holding at least n_u64 elements (the C ABI trusts the sizes)."""
    import torch
    if t is None:
        raise ValueError(f"{name}: missing")
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous CUDA tensor")
    if t.dtype not in (torch.int64, torch.uint64):
        raise ValueError(f"{name}: expected int64 / uint64, got {t.dtype}")
    if t.numel() < n_u64:
        raise ValueError(f"{name}: {t.numel()} elements, the call needs {n_u64}")


def _stream(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


# --------------------------------------------------------------------------- handles
class _Handle:
    _free = None

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr and self._free is not None and _lib is not None:   # not at interpreter exit
            getattr(_lib, self._free)(self.ptr)
            self.ptr = None


class SecretKey(_Handle):
    _free = "bm_sk_free"


class PublicKey(_Handle):
    _free = "bm_pk_free"


class EvalKey(_Handle):
    _free = "bm_evk_free"


class PublicKeyDev(_Handle):
    _free = "bm_pk_dev_free"


class EvalKeyDev(_Handle):
    _free = "bm_evk_dev_free"


class CompressKey(_Handle):
    _free = "bm_ck_free"


class CompressKeyDev(_Handle):
    _free = "bm_ck_dev_free"


class ExpandKey(_Handle):
    _free = "bm_xk_free"


class ExpandKeyDev(_Handle):
    _free = "bm_xk_dev_free"


# --------------------------------------------------------------------------- API (same names as the C ABI)
RNG_SEEDED, RNG_OS = 0, 1


def bm_rng_mode(mode):
    """RNG_OS (the library default): getrandom()-keyed streams (224-bit keys, fresh per encryption);
    RNG_SEEDED: deterministic in the seed (tests, benchmarks, oracle parity)."""
    _chk(_lib.bm_rng_mode(mode), "bm_rng_mode")


def bm_get_rng_mode():
    return int(_lib.bm_get_rng_mode())


def bm_params_init(d, p):
    prm = bm_params()
    _chk(_lib.bm_params_init(ctypes.byref(prm), d, p), "bm_params_init")
    return prm


def bm_keygen(prm, seed):
    sk, pk, evk = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _chk(_lib.bm_keygen(ctypes.byref(prm), seed, ctypes.byref(sk), ctypes.byref(pk), ctypes.byref(evk)), "bm_keygen")
    return SecretKey(sk), PublicKey(pk), EvalKey(evk)


def bm_evk_add_hoisted(prm, seed, evk):
    """f2: add the Galois keys of every rotation 1..s-1 (same seed as bm_keygen) to evk."""
    _chk(_lib.bm_evk_add_hoisted(ctypes.byref(prm), seed, evk.ptr), "bm_evk_add_hoisted")
    return evk


def bm_sk_export(sk):
    out = np.zeros(N, np.int8)
    _chk(_lib.bm_sk_export(sk.ptr, _np_ptr(out)), "bm_sk_export")
    return out


def bm_pk_export(pk):
    out = np.zeros((2, 2, N), np.uint64)
    _chk(_lib.bm_pk_export(pk.ptr, _np_ptr(out)), "bm_pk_export")
    return out


def bm_evk_export(evk):
    n = _i32()
    _chk(_lib.bm_evk_export(evk.ptr, None, None, ctypes.byref(n)), "bm_evk_export")
    rlk = np.zeros((2, 2, 3, N), np.uint64)
    gk = np.zeros((max(n.value, 1), 2, 2, N), np.uint64)
    _chk(_lib.bm_evk_export(evk.ptr, _np_ptr(rlk), _np_ptr(gk), ctypes.byref(n)), "bm_evk_export")
    return rlk, gk[:n.value]


def bm_sk_import(prm, s):
    out = ctypes.c_void_p()
    s = np.ascontiguousarray(s, np.int8)
    _chk(_lib.bm_sk_import(ctypes.byref(prm), _np_ptr(s), ctypes.byref(out)), "bm_sk_import")
    return SecretKey(out)


def bm_pk_import(prm, v):
    out = ctypes.c_void_p()
    v = np.ascontiguousarray(v, np.uint64)
    _chk(_lib.bm_pk_import(ctypes.byref(prm), _np_ptr(v), ctypes.byref(out)), "bm_pk_import")
    return PublicKey(out)


def bm_evk_import(prm, rlk, gk):
    out = ctypes.c_void_p()
    rlk = np.ascontiguousarray(rlk, np.uint64)
    gk = np.ascontiguousarray(gk, np.uint64)
    n = gk.shape[0] if gk.ndim == 4 else 0
    _chk(_lib.bm_evk_import(ctypes.byref(prm), _np_ptr(rlk), _np_ptr(gk) if n else None, n, ctypes.byref(out)),
         "bm_evk_import")
    return EvalKey(out)


def bm_pk_to_device(prm, pk):
    out = ctypes.c_void_p()
    _chk(_lib.bm_pk_to_device(ctypes.byref(prm), pk.ptr, ctypes.byref(out)), "bm_pk_to_device")
    return PublicKeyDev(out)


def bm_evk_to_device(prm, evk):
    out = ctypes.c_void_p()
    _chk(_lib.bm_evk_to_device(ctypes.byref(prm), evk.ptr, ctypes.byref(out)), "bm_evk_to_device")
    return EvalKeyDev(out)


def bm_encode_db(prm, tmpl, first_set, n_sets):
    tmpl = np.ascontiguousarray(tmpl, np.float64)
    out = np.zeros((n_sets, prm.p, N), np.int64)
    _chk(_lib.bm_encode_db(ctypes.byref(prm), _np_ptr(tmpl), tmpl.shape[0], first_set, n_sets, _np_ptr(out)),
         "bm_encode_db")
    return out


def bm_encode_query(prm, q):
    q = np.ascontiguousarray(q, np.float64)
    out = np.zeros((q.shape[0], prm.p, N), np.int64)
    _chk(_lib.bm_encode_query(ctypes.byref(prm), _np_ptr(q), q.shape[0], _np_ptr(out)), "bm_encode_query")
    return out


def bm_encrypt(prm, pk_dev, d_pt, first_obj, seed, d_out, stream=None):
    """d_pt: CUDA int64 [n][N]; d_out: CUDA uint64/int64 [n][2][2][N] (NTT domain)."""
    n = d_pt.shape[0]
    _chk(_lib.bm_encrypt(ctypes.byref(prm), pk_dev.ptr, _dptr(d_pt), n, first_obj, seed, _dptr(d_out),
                         _stream(stream)), "bm_encrypt")


def bm_encrypt_db(prm, pk_dev, tmpl, first_set, n_sets, seed, d_out, stream=None):
    tmpl = np.ascontiguousarray(tmpl, np.float64)
    _chk(_lib.bm_encrypt_db(ctypes.byref(prm), pk_dev.ptr, _np_ptr(tmpl), tmpl.shape[0], first_set, n_sets, seed,
                            _dptr(d_out), _stream(stream)), "bm_encrypt_db")


def bm_encrypt_query(prm, pk_dev, q, first_query, seed, d_out, stream=None):
    q = np.ascontiguousarray(q, np.float64)
    _chk(_lib.bm_encrypt_query(ctypes.byref(prm), pk_dev.ptr, _np_ptr(q), q.shape[0], first_query, seed,
                               _dptr(d_out), _stream(stream)), "bm_encrypt_query")


def bm_ct_to_coeff(prm, d_in, n_limbs, d_out, stream=None):
    _chk(_lib.bm_ct_to_coeff(ctypes.byref(prm), _dptr(d_in), d_in.numel() // (2 * n_limbs * N), n_limbs, _dptr(d_out),
                             _stream(stream)), "bm_ct_to_coeff")


def bm_ct_from_coeff(prm, d_in, n_limbs, d_out, stream=None):
    _chk(_lib.bm_ct_from_coeff(ctypes.byref(prm), _dptr(d_in), d_in.numel() // (2 * n_limbs * N), n_limbs,
                               _dptr(d_out), _stream(stream)), "bm_ct_from_coeff")


def bm_match_ws_bytes(prm, n_sets, nq, order=ORDER_HOISTED):
    return int(_lib.bm_match_ws_bytes(ctypes.byref(prm), n_sets, nq, order))


def bm_db_tc_bytes(prm, n_sets):
    return int(_lib.bm_db_tc_bytes(ctypes.byref(prm), n_sets))


_TC_KEEP = {}   # d_db pointer -> (d_db, d_packed): the registered buffers stay alive until unregistered


def bm_db_tc_register(prm, d_db, n_sets, d_packed, stream=None):
    """Pack the DB into the tensor-core layout (d_packed: a CUDA uint8 tensor of >= bm_db_tc_bytes bytes)
    and register it: bm_match then runs K1 on the tensor cores for d_db.  The binding holds references
    to both tensors until bm_db_tc_unregister (d_db must not change meanwhile)."""
    if d_packed.numel() * d_packed.element_size() < bm_db_tc_bytes(prm, n_sets):
        raise ValueError("d_packed: smaller than bm_db_tc_bytes")
    _need(d_db, n_sets * prm.p * 4 * N, "d_db")
    _chk(_lib.bm_db_tc_register(ctypes.byref(prm), _dptr(d_db), n_sets, _dptr(d_packed),
                                d_packed.numel() * d_packed.element_size(), _stream(stream)), "bm_db_tc_register")
    _TC_KEEP[d_db.data_ptr()] = (d_db, d_packed)


def bm_db_tc_unregister(d_db):
    _chk(_lib.bm_db_tc_unregister(_dptr(d_db)), "bm_db_tc_unregister")
    _TC_KEEP.pop(d_db.data_ptr(), None)


def _check_scan(prm, d_db, n_sets, d_q, nq, n_limbs=2):
    if n_sets < 0 or nq < 0:
        raise ValueError("n_sets and nq must be >= 0")
    if n_sets and nq:
        _need(d_db, n_sets * prm.p * 2 * n_limbs * N, "d_db")
        _need(d_q, nq * prm.p * 2 * n_limbs * N, "d_q")


def n_components(order):
    """Result polynomials per (query, set): 3 for the degree-2 output, else 2."""
    return 3 if order == ORDER_DEG2 else 2


def bm_match(prm, evk_dev, d_db, n_sets, d_q, nq, d_out, d_ws, order=ORDER_HOISTED, stream=None):
    """evk_dev may be None for ORDER_DEG2 (no key switch)."""
    _check_scan(prm, d_db, n_sets, d_q, nq)
    if n_sets and nq:
        _need(d_out, nq * n_sets * n_components(order) * N, "d_out")
    ws_bytes = d_ws.numel() * d_ws.element_size() if d_ws is not None else 0
    _chk(_lib.bm_match(ctypes.byref(prm), evk_dev.ptr if evk_dev is not None else None, _dptr(d_db) if n_sets else None, n_sets,
                       _dptr(d_q) if nq else None, nq, _dptr(d_out) if nq * n_sets else None,
                       _dptr(d_ws) if ws_bytes else None, ws_bytes, order, _stream(stream)), "bm_match")


def bm_match_rows(prm, evk_dev, d_db, n_sets, d_q, nq, d_rows, set_offset, d_ws, order=ORDER_HOISTED, stream=None):
    """The scan with the gather fused into its output kernels: d_rows is a CUDA int64 tensor of nq
    device addresses (local or peer, see bm_ipc_open); (query j, local set t) lands at row j, global
    set set_offset + t (include/blindmatch.h)."""
    _check_scan(prm, d_db, n_sets, d_q, nq)
    _need(d_rows, nq, "d_rows")
    if set_offset < 0:
        raise ValueError("set_offset must be >= 0")
    ws_bytes = d_ws.numel() * d_ws.element_size()
    _chk(_lib.bm_match_rows(ctypes.byref(prm), evk_dev.ptr if evk_dev is not None else None, _dptr(d_db) if n_sets else None, n_sets,
                            _dptr(d_q) if nq else None, nq, _dptr(d_rows), set_offset,
                            _dptr(d_ws) if ws_bytes else None, ws_bytes, order, _stream(stream)), "bm_match_rows")


def bm_ipc_handle(d_tensor):
    """(64-byte CUDA IPC handle of the allocation holding d_tensor, byte offset of d_tensor in it)."""
    h = (ctypes.c_uint8 * 64)()
    off = _u64(0)
    _chk(_lib.bm_ipc_handle(ctypes.c_void_p(d_tensor.data_ptr()), h, ctypes.byref(off)), "bm_ipc_handle")
    return bytes(h), int(off.value)


def bm_ipc_open(handle):
    """Map a peer process's allocation: returns its base address in this process."""
    h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    p = ctypes.c_void_p()
    _chk(_lib.bm_ipc_open(h, ctypes.byref(p)), "bm_ipc_open")
    return int(p.value)


def bm_ipc_close(base):
    _chk(_lib.bm_ipc_close(ctypes.c_void_p(base)), "bm_ipc_close")


def bm_match_host_ws_bytes(prm, n_sets, nq, order=ORDER_HOISTED):
    return int(_lib.bm_match_host_ws_bytes(ctypes.byref(prm), n_sets, nq, order))


def _hp(x, n_u64, name):
    """host pointer of a contiguous CPU tensor / numpy array of at least n_u64 8-byte elements"""
    if isinstance(x, np.ndarray):
        if x.itemsize != 8 or x.size < n_u64:
            raise ValueError(f"{name}: expected >= {n_u64} 8-byte elements")
        return _np_ptr(x)
    if x.is_cuda or not x.is_contiguous() or x.element_size() != 8 or x.numel() < n_u64:
        raise ValueError(f"{name}: expected a contiguous CPU tensor of >= {n_u64} 8-byte elements")
    return ctypes.c_void_p(x.data_ptr())


def bm_match_host(prm, evk_dev, d_db, n_sets, h_q, nq, h_out, d_ws, order=ORDER_HOISTED, stream=None):
    """h_q / h_out: (pinned) CPU tensors or numpy arrays."""
    _need(d_db, n_sets * prm.p * 4 * N, "d_db")
    ws_bytes = d_ws.numel() * d_ws.element_size()
    _chk(_lib.bm_match_host(ctypes.byref(prm), evk_dev.ptr if evk_dev is not None else None, _dptr(d_db), n_sets, _hp(h_q, nq * prm.p * 4 * N, "h_q"),
                            nq, _hp(h_out, nq * n_sets * n_components(order) * N, "h_out"), _dptr(d_ws), ws_bytes, order,
                            _stream(stream)), "bm_match_host")


def bm_match_host_ring(prm, evk_dev, d_db, n_sets, h_q, nq, h_ring, ring_rows, d_ws, order=ORDER_HOISTED,
                       stream=None):
    """bm_match_host with query j's results written to host row j mod ring_rows of h_ring
    [ring_rows][n_sets][2][N] (bounded host memory for very large result sets)."""
    _need(d_db, n_sets * prm.p * 4 * N, "d_db")
    ws_bytes = d_ws.numel() * d_ws.element_size()
    _chk(_lib.bm_match_host_ring(ctypes.byref(prm), evk_dev.ptr if evk_dev is not None else None, _dptr(d_db), n_sets,
                                 _hp(h_q, nq * prm.p * 4 * N, "h_q"), nq,
                                 _hp(h_ring, ring_rows * n_sets * n_components(order) * N, "h_ring"), ring_rows, _dptr(d_ws), ws_bytes,
                                 order, _stream(stream)), "bm_match_host_ring")


# --------------------------------------------------------------------------- options / counters
OPTIONS = {"chunk_pairs": 0, "expand_chunk": 1, "host_groups": 2, "ladder_c2": 3, "ladder_c3": 4,
           "ladder_tail": 5, "cmp_chunk": 6, "tensor_mma": 7}


def bm_set_option(name, value):
    _chk(_lib.bm_set_option(OPTIONS[name], int(value)), "bm_set_option")


def bm_get_option(name):
    return int(_lib.bm_get_option(OPTIONS[name]))


class options:
    """with bm.options(chunk_pairs=7, ladder_c3=0): ...  -- library options set for the block and
    restored afterwards (tests and tuning runs; the defaults are the product)."""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = bm_get_option(k)
            bm_set_option(k, v)
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            bm_set_option(k, v)


def bm_launch_count():
    return int(_lib.bm_launch_count())


def bm_launch_count_reset():
    _lib.bm_launch_count_reset()


# --------------------------------------------------------------------------- device-side client decryption
class SecretKeyDev(_Handle):
    _free = "bm_sk_dev_free"


def bm_sk_to_device(prm, sk):
    out = ctypes.c_void_p()
    _chk(_lib.bm_sk_to_device(ctypes.byref(prm), sk.ptr, ctypes.byref(out)), "bm_sk_to_device")
    return SecretKeyDev(out)


def bm_decrypt_dev(prm, sk_dev, d_ct, d_scores=None, stream=None):
    """d_ct: CUDA int64 [n][2][N] level-0 coefficient-domain results (bm_match's d_out, any leading
    shape) -> d_scores CUDA float64 [n][B] (allocated if None)."""
    import torch
    n = d_ct.numel() // (2 * N)
    _need(d_ct, n * 2 * N, "d_ct")
    if d_scores is None:
        d_scores = torch.empty((n, prm.B), dtype=torch.float64, device=d_ct.device)
    if d_scores.dtype != torch.float64 or d_scores.numel() < n * prm.B or not d_scores.is_contiguous():
        raise ValueError("d_scores: expected a contiguous float64 CUDA tensor of n x B")
    _chk(_lib.bm_decrypt_dev(ctypes.byref(prm), sk_dev.ptr, _dptr(d_ct), n, _dptr(d_scores), _stream(stream)),
         "bm_decrypt_dev")
    return d_scores


def bm_set_profiling(on):
    _lib.bm_set_profiling(1 if on else 0)


def bm_profile_reset():
    _lib.bm_profile_reset()


def bm_profile_read():
    ms = np.zeros(7, np.float64)
    la = np.zeros(7, np.int64)
    un = np.zeros(7, np.int64)
    _chk(_lib.bm_profile_read(_np_ptr(ms), _np_ptr(la), _np_ptr(un)), "bm_profile_read")
    return ms, la, un


PROFILE_CLASSES = ["tensor", "digits", "relin", "unused3", "ladder", "hrot", "out_intt"]


def bm_decrypt(prm, sk, h_ct):
    """h_ct: uint64 [n][2][1][N] canonical -> scores float64 [n][B]."""
    h_ct = np.ascontiguousarray(h_ct, np.uint64)
    n = h_ct.size // (2 * N)
    out = np.zeros((n, prm.B), np.float64)
    _chk(_lib.bm_decrypt(ctypes.byref(prm), sk.ptr, _np_ptr(h_ct), n, _np_ptr(out)), "bm_decrypt")
    return out


def bm_decrypt_raw(prm, sk, h_ct):
    h_ct = np.ascontiguousarray(h_ct, np.uint64)
    n = h_ct.size // (2 * N)
    out = np.zeros((n, N), np.int64)
    _chk(_lib.bm_decrypt_raw(ctypes.byref(prm), sk.ptr, _np_ptr(h_ct), n, _np_ptr(out)), "bm_decrypt_raw")
    return out


def bm_decrypt_deg2(prm, sk, h_ct):
    """f2 degree-2 results: h_ct uint64 [n][3][N] canonical (BM_ORDER_DEG2) -> scores float64 [n][B]."""
    h_ct = np.ascontiguousarray(h_ct, np.uint64)
    n = h_ct.size // (3 * N)
    out = np.zeros((n, prm.B), np.float64)
    _chk(_lib.bm_decrypt_deg2(ctypes.byref(prm), sk.ptr, _np_ptr(h_ct), n, _np_ptr(out)), "bm_decrypt_deg2")
    return out


def bm_top1(scores):
    s = np.ascontiguousarray(scores, np.float64)
    idx = _i64()
    best = ctypes.c_double()
    _chk(_lib.bm_top1(_np_ptr(s), s.size, ctypes.byref(idx), ctypes.byref(best)), "bm_top1")
    return idx.value, best.value


def bm_sync(stream=None):
    _chk(_lib.bm_sync(_stream(stream)), "bm_sync")


def bm_strerror(code):
    return _lib.bm_strerror(code).decode()


def bm_build_info():
    return _lib.bm_build_info().decode()


# --------------------------------------------------------------------------- f3: query expansion
def bm_xk_keygen(prm, seed):
    """f3 expansion keys (pk limb q2 + level-1 Galois keys) of bm_keygen(prm, seed)'s secret."""
    out = ctypes.c_void_p()
    _chk(_lib.bm_xk_keygen(ctypes.byref(prm), seed, ctypes.byref(out)), "bm_xk_keygen")
    return ExpandKey(out)


def bm_xk_export(xk):
    n = _i32()
    _chk(_lib.bm_xk_export(xk.ptr, None, None, ctypes.byref(n)), "bm_xk_export")
    pk_q2 = np.zeros((2, N), np.uint64)
    gk1 = np.zeros((max(n.value, 1), 2, 2, 3, N), np.uint64)
    _chk(_lib.bm_xk_export(xk.ptr, _np_ptr(pk_q2), _np_ptr(gk1), ctypes.byref(n)), "bm_xk_export")
    return pk_q2, gk1[:n.value]


def bm_xk_import(prm, pk_q2, gk1):
    out = ctypes.c_void_p()
    pk_q2 = np.ascontiguousarray(pk_q2, np.uint64)
    gk1 = np.ascontiguousarray(gk1, np.uint64)
    n = gk1.shape[0] if gk1.ndim == 5 else 0
    _chk(_lib.bm_xk_import(ctypes.byref(prm), _np_ptr(pk_q2), _np_ptr(gk1) if n else None, n, ctypes.byref(out)),
         "bm_xk_import")
    return ExpandKey(out)


def bm_encode_query_tiled(prm, q):
    q = np.ascontiguousarray(q, np.float64)
    out = np.zeros((q.shape[0], N), np.int64)
    _chk(_lib.bm_encode_query_tiled(ctypes.byref(prm), _np_ptr(q), q.shape[0], _np_ptr(out)), "bm_encode_query_tiled")
    return out


MASK_EXPAND, MASK_ENROLL = 0, 1


def bm_encode_masks(prm, kind=MASK_EXPAND):
    out = np.zeros((prm.p, N), np.int64)
    _chk(_lib.bm_encode_masks(ctypes.byref(prm), kind, _np_ptr(out)), "bm_encode_masks")
    return out


def bm_encode_enroll(prm, v):
    v = np.ascontiguousarray(v, np.float64)
    out = np.zeros((v.shape[0], N), np.int64)
    _chk(_lib.bm_encode_enroll(ctypes.byref(prm), _np_ptr(v), v.shape[0], _np_ptr(out)), "bm_encode_enroll")
    return out


def bm_xk_to_device(prm, pk, xk, masks=None, emasks=None, enroll=True):
    """masks / emasks: int64 [p][N] expansion / enrollment plaintexts (defaults: bm_encode_masks;
    enroll=False skips the enrollment masks)."""
    m = np.ascontiguousarray(bm_encode_masks(prm) if masks is None else masks, np.int64)
    e = None
    if enroll or emasks is not None:
        e = np.ascontiguousarray(bm_encode_masks(prm, MASK_ENROLL) if emasks is None else emasks, np.int64)
    out = ctypes.c_void_p()
    _chk(_lib.bm_xk_to_device(ctypes.byref(prm), pk.ptr, xk.ptr, _np_ptr(m), _np_ptr(e) if e is not None else None,
                              ctypes.byref(out)), "bm_xk_to_device")
    return ExpandKeyDev(out)


def bm_encrypt_l2(prm, xk_dev, d_pt, first_obj, seed, d_out, stream=None):
    """d_pt: CUDA int64 [n][N]; d_out: CUDA [n][2][3][N] (level 2, NTT domain)."""
    _chk(_lib.bm_encrypt_l2(ctypes.byref(prm), xk_dev.ptr, _dptr(d_pt), d_pt.shape[0], first_obj, seed, _dptr(d_out),
                            _stream(stream)), "bm_encrypt_l2")


def bm_expand_ws_bytes(prm, nq):
    return int(_lib.bm_expand_ws_bytes(ctypes.byref(prm), nq))


def bm_expand(prm, xk_dev, d_in, nq, d_out, d_ws, stream=None):
    """Algorithm 1: d_in [nq][2][3][N] level 2 -> d_out [nq][p][2][2][N] level 1 (NTT domain)."""
    ws_bytes = d_ws.numel() * d_ws.element_size() if d_ws is not None else 0
    _chk(_lib.bm_expand(ctypes.byref(prm), xk_dev.ptr, _dptr(d_in) if nq else None, nq, _dptr(d_out) if nq else None,
                        _dptr(d_ws) if ws_bytes else None, ws_bytes, _stream(stream)), "bm_expand")


def bm_enroll_ws_bytes(prm, n):
    return int(_lib.bm_enroll_ws_bytes(ctypes.byref(prm), n))


def bm_enroll(prm, xk_dev, d_in, first_template, d_db, d_ws, stream=None):
    """f4: accumulate the level-2 template cts d_in [n][2][3][N] into d_db [n_sets][p][2][2][N]."""
    n = d_in.shape[0]
    ws_bytes = d_ws.numel() * d_ws.element_size() if d_ws is not None else 0
    _chk(_lib.bm_enroll(ctypes.byref(prm), xk_dev.ptr, _dptr(d_in) if n else None, n, first_template, _dptr(d_db),
                        d_db.shape[0], _dptr(d_ws) if ws_bytes else None, ws_bytes, _stream(stream)), "bm_enroll")


# --------------------------------------------------------------------------- f1: output compression
def bm_ck_keygen(prm, seed):
    out = ctypes.c_void_p()
    _chk(_lib.bm_ck_keygen(ctypes.byref(prm), seed, ctypes.byref(out)), "bm_ck_keygen")
    return CompressKey(out)


def bm_ck_export(prm, ck):
    rlk2 = np.zeros((3, 2, 4, N), np.uint64)
    gkl = np.zeros((max(prm.log_s, 1), 2, 2, 3, N), np.uint64)
    gkc = np.zeros((max(prm.s - 1, 1), 2, 2, N), np.uint64)
    _chk(_lib.bm_ck_export(ck.ptr, _np_ptr(rlk2), _np_ptr(gkl), _np_ptr(gkc)), "bm_ck_export")
    return rlk2, gkl[:prm.log_s], gkc[:prm.s - 1]


def bm_encode_cmp_mask(prm):
    out = np.zeros(N, np.int64)
    _chk(_lib.bm_encode_cmp_mask(ctypes.byref(prm), _np_ptr(out)), "bm_encode_cmp_mask")
    return out


def bm_ck_to_device(prm, ck, mask=None):
    m = np.ascontiguousarray(bm_encode_cmp_mask(prm) if mask is None else mask, np.int64)
    out = ctypes.c_void_p()
    _chk(_lib.bm_ck_to_device(ctypes.byref(prm), ck.ptr, _np_ptr(m), ctypes.byref(out)), "bm_ck_to_device")
    return CompressKeyDev(out)


def bm_match_cmp_ws_bytes(prm, n_sets, nq):
    return int(_lib.bm_match_cmp_ws_bytes(ctypes.byref(prm), n_sets, nq))


def bm_match_cmp(prm, ck_dev, d_db, n_sets, d_q, nq, d_out, d_ws, stream=None):
    """f1: level-2 DB / query parts -> packed level-0 results d_out [nq][ceil(n_sets/s)][2][N]."""
    ws_bytes = d_ws.numel() * d_ws.element_size() if d_ws is not None else 0
    _chk(_lib.bm_match_cmp(ctypes.byref(prm), ck_dev.ptr, _dptr(d_db) if n_sets else None, n_sets,
                           _dptr(d_q) if nq else None, nq, _dptr(d_out) if nq * n_sets else None,
                           _dptr(d_ws) if ws_bytes else None, ws_bytes, _stream(stream)), "bm_match_cmp")


def bm_decrypt_packed(prm, sk, h_ct):
    """h_ct: uint64 [n][2][1][N] packed results -> all S slots float64 [n][S]."""
    h_ct = np.ascontiguousarray(h_ct, np.uint64)
    n = h_ct.size // (2 * N)
    out = np.zeros((n, SLOTS), np.float64)
    _chk(_lib.bm_decrypt_packed(ctypes.byref(prm), sk.ptr, _np_ptr(h_ct), n, _np_ptr(out)), "bm_decrypt_packed")
    return out


# --------------------------------------------------------------------------- serialisation
def bm_ct_export(prm, ct, level, scale):
    """ct: uint64 [n][2][level+1][N] coefficient domain (host) -> framed bytes."""
    ct = np.ascontiguousarray(ct, np.uint64)
    n = ct.size // (2 * (level + 1) * N)
    ln = _sz()
    _chk(_lib.bm_ct_export(ctypes.byref(prm), _np_ptr(ct), n, level, scale, None, ctypes.byref(ln)), "bm_ct_export")
    buf = np.zeros(ln.value, np.uint8)
    _chk(_lib.bm_ct_export(ctypes.byref(prm), _np_ptr(ct), n, level, scale, _np_ptr(buf), ctypes.byref(ln)),
         "bm_ct_export")
    return buf.tobytes()


def bm_ct_import(prm, data):
    """framed bytes -> (ct uint64 [n][2][level+1][N], level, scale)."""
    buf = np.frombuffer(data, np.uint8).copy()
    n, lev, sc = _i64(), _i32(), ctypes.c_double()
    _chk(_lib.bm_ct_import(ctypes.byref(prm), _np_ptr(buf), buf.size, None, ctypes.byref(n), ctypes.byref(lev),
                           ctypes.byref(sc)), "bm_ct_import")
    ct = np.zeros((n.value, 2, lev.value + 1, N), np.uint64)
    _chk(_lib.bm_ct_import(ctypes.byref(prm), _np_ptr(buf), buf.size, _np_ptr(ct) if n.value else None,
                           ctypes.byref(n), ctypes.byref(lev), ctypes.byref(sc)), "bm_ct_import")
    return ct, lev.value, sc.value
