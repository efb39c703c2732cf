"""Small launches of every kernel family for compute-sanitizer (SURVEY.md sec. 5 "Race detection /
sanitizers"; diagnostic, not a test).  Usage on the GPU box:

    compute-sanitizer --tool memcheck  python tools/sanitize.py all
    compute-sanitizer --tool racecheck python tools/sanitize.py small
    compute-sanitizer --tool synccheck python tools/sanitize.py small

Legs: configs[0] (1 pair: the 3-CTA pipelined latency ladder k_ladder_c3 + swapped tensor tiles),
the 2-CTA latency ladder (k_ladder_t<true>), a launch of n_SM + 12 pairs (full waves on
k_ladder_t<false> + the cluster tail from MatchK::pair0), f2's k_hrot (hoisted and BSGS), f2's
degree-2 output (k_rescale_deg2), the paper order (k_relin
accumulating), s = 1 (k_out_intt), f3 bm_expand, f4 bm_enroll, f1 bm_match_cmp, device decryption.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_06167_b200 import bm as B  # noqa: E402
from paper_2408_06167_b200 import inputs as I  # noqa: E402

N = 8192
dev = torch.device("cuda")


def scan(d, p, n_tmpl, nq, order=0, **opts):
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    if order in (2, 4):
        B.bm_evk_add_hoisted(prm, 1, evk)
    pk_dev, evk_dev = B.bm_pk_to_device(prm, pk), B.bm_evk_to_device(prm, evk)
    n_sets = -(-n_tmpl // prm.B)
    T = I.random_unit(n_tmpl, d, 3)
    Q = I.random_unit(nq, d, 4)
    d_db = torch.empty((n_sets, p, 2, 2, N), dtype=torch.int64, device=dev)
    d_q = torch.empty((nq, p, 2, 2, N), dtype=torch.int64, device=dev)
    B.bm_encrypt_db(prm, pk_dev, T, 0, n_sets, 2, d_db)
    B.bm_encrypt_query(prm, pk_dev, Q, 0, 3, d_q)
    out = torch.empty((nq, n_sets, 2, N), dtype=torch.int64, device=dev)
    with B.options(**opts):
        ws = torch.empty(max(1, B.bm_match_ws_bytes(prm, n_sets, nq, order)), dtype=torch.uint8, device=dev)
        B.bm_match(prm, evk_dev, d_db, n_sets, d_q, nq, out, ws, order)
    B.bm_sync()
    sc = B.bm_decrypt_dev(prm, B.bm_sk_to_device(prm, sk), out)
    B.bm_sync()
    err = float((sc.view(nq, -1)[:, :n_tmpl].cpu() - torch.from_numpy(Q @ T.T)).abs().max())
    print(f"scan d={d} p={p} pairs={n_sets * nq} order={order} {opts}: max err {err:.2e}", flush=True)
    return prm, sk, pk, evk_dev


def deg2():
    d = p = 32
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    pk_dev = B.bm_pk_to_device(prm, pk)
    T = I.random_unit(5000, d, 8)
    Q = I.random_unit(2, d, 9)
    d_db = torch.empty((2, p, 2, 2, N), dtype=torch.int64, device=dev)
    d_q = torch.empty((2, p, 2, 2, N), dtype=torch.int64, device=dev)
    B.bm_encrypt_db(prm, pk_dev, T, 0, 2, 2, d_db)
    B.bm_encrypt_query(prm, pk_dev, Q, 0, 3, d_q)
    out = torch.empty((2, 2, 3, N), dtype=torch.int64, device=dev)
    ws = torch.empty(B.bm_match_ws_bytes(prm, 2, 2, B.ORDER_DEG2), dtype=torch.uint8, device=dev)
    B.bm_match(prm, None, d_db, 2, d_q, 2, out, ws, B.ORDER_DEG2)
    B.bm_sync()
    sc = B.bm_decrypt_deg2(prm, sk, out.cpu().numpy().view(np.uint64)).reshape(2, -1)[:, :5000]
    print(f"f2 degree-2 output: max err {np.abs(sc - Q @ T.T).max():.2e}", flush=True)


def next_rows():
    d, p = 64, 8
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    xk = B.bm_xk_keygen(prm, 1)
    xk_dev = B.bm_xk_to_device(prm, pk, xk)
    Q = I.random_unit(2, d, 5)
    pt = torch.from_numpy(B.bm_encode_query_tiled(prm, Q)).to(dev)
    l2 = torch.empty((2, 2, 3, N), dtype=torch.int64, device=dev)
    B.bm_encrypt_l2(prm, xk_dev, pt, 0, 3, l2)
    qx = torch.empty((2, p, 2, 2, N), dtype=torch.int64, device=dev)
    ws = torch.empty(B.bm_expand_ws_bytes(prm, 2), dtype=torch.uint8, device=dev)
    B.bm_expand(prm, xk_dev, l2, 2, qx, ws)
    B.bm_sync()
    print("f3 bm_expand ok", flush=True)
    T = I.random_unit(40, d, 6)
    tp = torch.from_numpy(B.bm_encode_enroll(prm, T)).to(dev)
    tl2 = torch.empty((40, 2, 3, N), dtype=torch.int64, device=dev)
    B.bm_encrypt_l2(prm, xk_dev, tp, 0, 5, tl2)
    db = torch.zeros((1, p, 2, 2, N), dtype=torch.int64, device=dev)
    ws = torch.empty(B.bm_enroll_ws_bytes(prm, 40), dtype=torch.uint8, device=dev)
    B.bm_enroll(prm, xk_dev, tl2, 0, db, ws)
    B.bm_sync()
    print("f4 bm_enroll ok", flush=True)
    ck_dev = B.bm_ck_to_device(prm, B.bm_ck_keygen(prm, 1))
    n_sets = 3
    dbl2 = torch.empty((n_sets, p, 2, 3, N), dtype=torch.int64, device=dev)
    T2 = I.random_unit(n_sets * prm.B, d, 7)
    B.bm_encrypt_l2(prm, xk_dev, torch.from_numpy(B.bm_encode_db(prm, T2, 0, n_sets).reshape(-1, N)).to(dev), 0, 2,
                    dbl2)
    ql2 = torch.empty((1, p, 2, 3, N), dtype=torch.int64, device=dev)
    B.bm_encrypt_l2(prm, xk_dev, torch.from_numpy(B.bm_encode_query(prm, Q[:1]).reshape(-1, N)).to(dev), 0, 3, ql2)
    out = torch.empty((1, -(-n_sets // prm.s), 2, N), dtype=torch.int64, device=dev)
    ws = torch.empty(B.bm_match_cmp_ws_bytes(prm, n_sets, 1), dtype=torch.uint8, device=dev)
    B.bm_match_cmp(prm, ck_dev, dbl2, n_sets, ql2, 1, out, ws)
    B.bm_sync()
    print("f1 bm_match_cmp ok", flush=True)


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "all"
    torch.cuda.set_device(0)
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    scan(16, 1, 256, 1)                                  # k_ladder_c3 (1 pair)
    scan(64, 4, 600, 2, ladder_c3=0)                     # k_ladder_t<true> (6 pairs)
    if mode == "small":
        return
    scan(16, 8, (n_sm + 12) * 2048 - 100, 1)             # one-CTA waves + the cluster tail
    scan(128, 8, 700, 3, order=2)                        # k_hrot
    scan(128, 8, 700, 3, order=4)                        # k_hrot<true> + k_hrot<false> (BSGS)
    deg2()                                               # k_rescale_deg2
    scan(128, 8, 700, 3, order=1)                        # paper order (k_relin accumulates)
    scan(16, 16, 300, 2)                                 # s = 1: k_out_intt
    next_rows()


if __name__ == "__main__":
    main()
