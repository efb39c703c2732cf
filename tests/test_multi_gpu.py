"""Multi-GPU path on real GPUs: skipped unless two or more GPUs
are visible.  Two ranks over NCCL (one process per GPU) shard a database by contiguous sets, rank 0
encrypts the queries and broadcasts them (a3), every rank scans its own sets, and the results reach
their roots (a8) both ways bench.py can gather them:
  * fused: bm_match_rows storing straight into the roots' rows through CUDA IPC peer pointers
    (dist.P2PGather / dist.scan_p2p, with a bounded root ring), and
  * NCCL: dist.scan_pipelined's per-group all_to_all.
Each root then compares, bit for bit, every row it received with a single-GPU scan of the WHOLE
database that it computes itself (the sharded encryption is a bit-exact partition).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

D, P_PARTS, N_TMPL, NQ, G = 64, 4, 9 * 256 + 77, 8, 2   # s = 16, B = 256: 10 sets (last ragged)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    from paper_2408_06167_b200 import bm as B
    from paper_2408_06167_b200 import dist as pdist
    from paper_2408_06167_b200 import inputs as I
    B.bm_rng_mode(B.RNG_SEEDED)
    N = B.N
    prm = B.bm_params_init(D, P_PARTS)
    sk, pk, evk = B.bm_keygen(prm, 1)
    pk_dev, evk_dev = B.bm_pk_to_device(prm, pk), B.bm_evk_to_device(prm, evk)
    T = I.random_unit(N_TMPL, D, 61)
    Q = I.random_unit(NQ, D, 62)
    n_sets = -(-N_TMPL // prm.B)
    lo, cnt = pdist.shard_sets(n_sets, world, rank)
    d_db = torch.empty((cnt, P_PARTS, 2, 2, N), dtype=torch.int64, device=dev)
    B.bm_encrypt_db(prm, pk_dev, T, lo, cnt, 2, d_db)      # global set numbers: a slice of the full DB
    d_q = torch.zeros((NQ, P_PARTS, 2, 2, N), dtype=torch.int64, device=dev)
    if rank == 0:
        B.bm_encrypt_query(prm, pk_dev, Q, 0, 3, d_q)
    torch.cuda.synchronize()
    gq = NQ // G
    ws = torch.empty(B.bm_match_ws_bytes(prm, cnt, gq), dtype=torch.uint8, device=dev)
    comm, comp = torch.cuda.Stream(), [torch.cuda.Stream(), torch.cuda.Stream()]
    # ---- fused gather into root rings (2 slots = every group keeps its rows here)
    per = gq // world
    res = torch.full((G * per, n_sets, 2, N), -1, dtype=torch.int64, device=dev)
    gat = pdist.P2PGather(B, res, NQ, G, n_sets, ring=G)
    flag = torch.zeros(1, dtype=torch.float64, device=dev)

    def match_rows(g, q_g, rows_g):
        B.bm_match_rows(prm, evk_dev, d_db, cnt, q_g, q_g.shape[0], rows_g, lo, ws, stream=torch.cuda.current_stream())
    pdist.scan_p2p(match_rows, d_q, gat, G, comm, comp, flag)
    torch.cuda.synchronize()
    dist.barrier()
    # ---- NCCL all_to_all gather (ring of G slots)
    outs = [torch.empty((gq, cnt, 2, N), dtype=torch.int64, device=dev) for _ in range(G)]
    recv = [torch.empty((world, per, cnt, 2, N), dtype=torch.int64, device=dev) for _ in range(G)]

    def match(g, q_g, out_g):
        B.bm_match(prm, evk_dev, d_db, cnt, q_g, q_g.shape[0], out_g, ws, stream=torch.cuda.current_stream())
    pdist.scan_pipelined(match, d_q, outs, recv, G, comm, comp[0])
    torch.cuda.synchronize()
    dist.barrier()
    # ---- reference: this root scans the whole database alone
    full = torch.empty((n_sets, P_PARTS, 2, 2, N), dtype=torch.int64, device=dev)
    B.bm_encrypt_db(prm, pk_dev, T, 0, n_sets, 2, full)
    ref = torch.empty((NQ, n_sets, 2, N), dtype=torch.int64, device=dev)
    wsr = torch.empty(B.bm_match_ws_bytes(prm, n_sets, NQ), dtype=torch.uint8, device=dev)
    B.bm_match(prm, evk_dev, full, n_sets, d_q, NQ, ref, wsr)
    torch.cuda.synchronize()
    ok_p2p = ok_nccl = 0
    checked = 0
    for j, (root, row) in enumerate(pdist.p2p_row_map(NQ, G, world, ring=G)):
        if root != rank:
            continue
        checked += 1
        ok_p2p += int(torch.equal(res[row], ref[j]))
        g, i = divmod(j, gq)
        k, m = divmod(i, per)
        assert k == rank
        got = torch.cat([recv[g][src, m, :pdist.shard_sets(n_sets, world, src)[1]] for src in range(world)])
        ok_nccl += int(torch.equal(got, ref[j]))
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array([checked, ok_p2p, ok_nccl]))
    gat.close()
    dist.barrier()
    dist.destroy_process_group()


def test_two_gpu_fused_and_nccl_gather_equal_single_gpu(tmp_path):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (the multi-GPU path; CPU coverage: test_dist_gloo.py)")
    from paper_2408_06167_b200 import build
    build.build(verbose=False)
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        checked, ok_p2p, ok_nccl = np.load(tmp_path / f"r{r}.npy")
        assert checked == NQ // 2 and ok_p2p == checked and ok_nccl == checked
