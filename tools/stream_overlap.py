"""Diagnostic: do bm_match calls on two streams overlap (filling each other's kernel tails)?"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2408_06167_b200 import bm as B, inputs as I
prm = B.bm_params_init(128, 8)
sk, pk, evk = B.bm_keygen(prm, 1)
pk_dev, evk_dev = B.bm_pk_to_device(prm, pk), B.bm_evk_to_device(prm, evk)
T = I.templates(2); n_sets = 24; nq = 384
db = torch.empty((n_sets, 8, 2, 2, 8192), dtype=torch.int64, device="cuda")
B.bm_encrypt_db(prm, pk_dev, T, 0, n_sets, 2, db)
Q, _ = I.queries(2, nq)
q = torch.empty((nq, 8, 2, 2, 8192), dtype=torch.int64, device="cuda")
B.bm_encrypt_query(prm, pk_dev, Q, 0, 3, q)
out = torch.empty((nq, n_sets, 2, 8192), dtype=torch.int64, device="cuda")
for G in (1, 4, 8, 16):
    gq = nq // G
    wss = [torch.empty(B.bm_match_ws_bytes(prm, n_sets, gq), dtype=torch.uint8, device="cuda") for _ in range(2)]
    for nstreams in (1, 2):
        streams = [torch.cuda.Stream() for _ in range(nstreams)]
        def run():
            for g in range(G):
                s = streams[g % nstreams]
                B.bm_match(prm, evk_dev, db, n_sets, q[g * gq:(g + 1) * gq], gq, out[g * gq:(g + 1) * gq], wss[g % nstreams], 0, s)
        run(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3): run()
        torch.cuda.synchronize()
        print(f"groups {G:2d} streams {nstreams}: {(time.perf_counter() - t0) / 3 * 1e3:.2f} ms", flush=True)
