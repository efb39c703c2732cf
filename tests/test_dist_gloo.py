"""Multi-rank path of the scan on CPU (world size 2, gloo): DB sharded by sets, query broadcast
from rank 0, local scan, all_to_all gather to the query-block roots (dist.py).
The local scan is the oracle (this container has no GPU); the collective plumbing is the same
code bench.py runs over NCCL.  The gathered result must equal the single-process scan of the
whole DB bit for bit, and the sharded encryption must be a partition of the unsharded one."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

LOGN, D, P_PARTS = 6, 8, 2   # N = 64, S = 32, s = 4, B = 8 -> small, fast oracle
N_TMPL, NQ, WORLD = 37, 4, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup():
    from oracle import oracle as O
    from paper_2408_06167_b200 import inputs as I
    S, s, B = O.layout(LOGN, D, P_PARTS)
    T = I.random_unit(N_TMPL, D, 11)
    Q = I.random_unit(NQ, D, 12)
    n_sets = -(-N_TMPL // B)
    sk, pk, rlk, gk = O.keygen(LOGN, 1, O.n_rot_for(D, P_PARTS))
    return O, T, Q, n_sets, (sk, pk, rlk, gk)


def _encrypt_sets(O, T, pk, first_set, n_sets):
    S, s, B = O.layout(LOGN, D, P_PARTS)
    z = O.pack_db(T, LOGN, D, P_PARTS, first_set, n_sets).reshape(-1, S)
    ct = O.encrypt(LOGN, pk, O.encode(z, LOGN), first_set * P_PARTS, 2)
    return ct.reshape(n_sets, P_PARTS, 2, 2, -1)


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_06167_b200 import dist as pdist
    O, T, Q, n_sets, (sk, pk, rlk, gk) = _setup()
    lo, cnt = pdist.shard_sets(n_sets, world, rank)
    local_db = _encrypt_sets(O, T, pk, lo, cnt)
    # a3: rank 0 (the client-facing main server) encrypts the query; everyone receives it
    N = 1 << LOGN
    q = torch.zeros((NQ, P_PARTS, 2, 2, N), dtype=torch.int64)
    if rank == 0:
        S = N // 2
        qc = O.encrypt(LOGN, pk, O.encode(O.pack_query(Q, LOGN, D, P_PARTS).reshape(-1, S), LOGN), 0, 3)
        q.copy_(torch.from_numpy(qc.reshape(q.shape).view(np.int64)))
    pdist.broadcast_queries(q)
    # local scan over this rank's sets (ragged: the last rank may hold fewer sets)
    per = -(-n_sets // world)
    out = torch.zeros((NQ, per, 2, N), dtype=torch.int64)
    if cnt:
        res, pairs = O.match(LOGN, D, P_PARTS, 0, rlk, gk, local_db, q.numpy().view(np.uint64))
        for i, (j, t) in enumerate(pairs):
            out[j, t] = torch.from_numpy(res[i].reshape(2, N).view(np.int64))
    recv = pdist.gather_results(out)
    q0, nq_local = pdist.query_block(NQ, world, rank)
    np.save(os.path.join(out_dir, f"recv{rank}.npy"), recv.numpy())
    np.save(os.path.join(out_dir, f"db{rank}.npy"), local_db)
    t = pdist.max_over_ranks(float(rank + 1), torch.device("cpu"))
    assert t == float(world)
    dist.destroy_process_group()


def test_two_rank_scan_matches_single_process(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(WORLD, port, str(tmp_path)), nprocs=WORLD, join=True)
    from paper_2408_06167_b200 import dist as pdist
    O, T, Q, n_sets, (sk, pk, rlk, gk) = _setup()
    N = 1 << LOGN
    full_db = _encrypt_sets(O, T, pk, 0, n_sets)
    # sharded encryption is a bit-exact partition of the unsharded DB
    parts = [np.load(tmp_path / f"db{r}.npy") for r in range(WORLD)]
    assert np.array_equal(np.concatenate(parts), full_db)
    S = N // 2
    qc = O.encrypt(LOGN, pk, O.encode(O.pack_query(Q, LOGN, D, P_PARTS).reshape(-1, S), LOGN), 0, 3)
    ref, pairs = O.match(LOGN, D, P_PARTS, 0, rlk, gk, full_db, qc.reshape(NQ, P_PARTS, 2, 2, N))
    ref = ref.reshape(NQ, n_sets, 2, N)
    per = -(-n_sets // WORLD)
    for r in range(WORLD):
        recv = np.load(tmp_path / f"recv{r}.npy").view(np.uint64)  # [src rank][nq/W][per][2][N]
        q0, nql = pdist.query_block(NQ, WORLD, r)
        for src in range(WORLD):
            lo, cnt = pdist.shard_sets(n_sets, WORLD, src)
            assert np.array_equal(recv[src, :, :cnt], ref[q0:q0 + nql, lo:lo + cnt])


def test_shard_ranges_cover_and_balance():
    from paper_2408_06167_b200 import dist as pdist
    for T in (1, 7, 24, 4096, 131072):
        for W in (1, 2, 4, 8):
            got = [pdist.shard_sets(T, W, r) for r in range(W)]
            covered = [t for lo, cnt in got for t in range(lo, lo + cnt)]
            assert covered == list(range(T))
            assert max(c for _, c in got) - min(c for _, c in got) <= -(-T // W)
    assert pdist.query_block(384, 8, 3) == (144, 48)
    with pytest.raises(AssertionError):
        pdist.query_block(10, 4, 0)


def _worker_pipelined(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_06167_b200 import dist as pdist
    O, T, Q, n_sets, (sk, pk, rlk, gk) = _setup()
    lo, cnt = pdist.shard_sets(n_sets, world, rank)
    local_db = _encrypt_sets(O, T, pk, lo, cnt)
    N = 1 << LOGN
    q = torch.zeros((NQ, P_PARTS, 2, 2, N), dtype=torch.int64)
    if rank == 0:
        S = N // 2
        qc = O.encrypt(LOGN, pk, O.encode(O.pack_query(Q, LOGN, D, P_PARTS).reshape(-1, S), LOGN), 0, 3)
        q.copy_(torch.from_numpy(qc.reshape(q.shape).view(np.int64)))
    per = -(-n_sets // world)
    out = torch.zeros((NQ, per, 2, N), dtype=torch.int64)
    G = 2
    recv = torch.zeros((G, world, NQ // (G * world), per, 2, N), dtype=torch.int64)

    def match(g, q_g, out_g):   # the local scan of one query group (the oracle stands in for bm_match)
        if cnt:
            res, pairs = O.match(LOGN, D, P_PARTS, 0, rlk, gk, local_db, q_g.numpy().view(np.uint64))
            for i, (j, t) in enumerate(pairs):
                out_g[j, t] = torch.from_numpy(res[i].reshape(2, N).view(np.int64))

    pdist.scan_pipelined(match, q, out, recv, G)
    np.save(os.path.join(out_dir, f"precv{rank}.npy"), recv.numpy())
    dist.destroy_process_group()


def test_two_rank_pipelined_scan_matches_single_process(tmp_path):
    """bench.py's N > 1 step: broadcast, scan and all_to_all per query group (dist.scan_pipelined);
    query j of group g lands on rank group_query_block(...) with the results of every rank's sets."""
    port = _free_port()
    mp.spawn(_worker_pipelined, args=(WORLD, port, str(tmp_path)), nprocs=WORLD, join=True)
    from paper_2408_06167_b200 import dist as pdist
    O, T, Q, n_sets, (sk, pk, rlk, gk) = _setup()
    N = 1 << LOGN
    full_db = _encrypt_sets(O, T, pk, 0, n_sets)
    S = N // 2
    qc = O.encrypt(LOGN, pk, O.encode(O.pack_query(Q, LOGN, D, P_PARTS).reshape(-1, S), LOGN), 0, 3)
    ref, pairs = O.match(LOGN, D, P_PARTS, 0, rlk, gk, full_db, qc.reshape(NQ, P_PARTS, 2, 2, N))
    ref = ref.reshape(NQ, n_sets, 2, N)
    G = 2
    for r in range(WORLD):
        recv = np.load(tmp_path / f"precv{r}.npy").view(np.uint64)  # [G][src rank][nq/(G W)][per][2][N]
        for g in range(G):
            q0, nql = pdist.group_query_block(NQ, G, WORLD, r, g)
            for src in range(WORLD):
                lo, cnt = pdist.shard_sets(n_sets, WORLD, src)
                assert np.array_equal(recv[g, src, :, :cnt], ref[q0:q0 + nql, lo:lo + cnt])


def _worker_p2p(rank, world, port, out_dir):
    """The fused gather's data movement with the oracle as the local scan: every rank 'stores' each
    local result at the address the output kernels use (row of p2p_row_map, global set lo + t,
    component c: flat offset ((lo + t) * 2 + c) * N of the root's row), the stores travel to the
    roots by all_gather_object (standing in for NVLink), and each root's buffer is saved."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_06167_b200 import dist as pdist
    O, T, Q, n_sets, (sk, pk, rlk, gk) = _setup()
    lo, cnt = pdist.shard_sets(n_sets, world, rank)
    local_db = _encrypt_sets(O, T, pk, lo, cnt)
    N = 1 << LOGN
    q = torch.zeros((NQ, P_PARTS, 2, 2, N), dtype=torch.int64)
    if rank == 0:
        S = N // 2
        qc = O.encrypt(LOGN, pk, O.encode(O.pack_query(Q, LOGN, D, P_PARTS).reshape(-1, S), LOGN), 0, 3)
        q.copy_(torch.from_numpy(qc.reshape(q.shape).view(np.int64)))
    pdist.broadcast_queries(q)
    groups = 2
    rmap = pdist.p2p_row_map(NQ, groups, world)
    stores = []   # (root, row, flat offset in the row, values)
    if cnt:
        res, pairs = O.match(LOGN, D, P_PARTS, 0, rlk, gk, local_db, q.numpy().view(np.uint64))
        for i, (j, t) in enumerate(pairs):
            root, row = rmap[j]
            for c in range(2):
                stores.append((root, row, ((lo + t) * 2 + c) * N, res[i].reshape(2, N)[c].copy()))
    allst = [None] * world
    dist.all_gather_object(allst, stores)
    mine = np.zeros((NQ // world, n_sets * 2 * N), np.uint64)
    for st in allst:
        for root, row, off, v in st:
            if root == rank:
                mine[row, off:off + N] = v
    np.save(os.path.join(out_dir, f"p2p{rank}.npy"), mine)
    dist.destroy_process_group()


def test_two_rank_fused_gather_rows_match_single_process(tmp_path):
    port = _free_port()
    mp.spawn(_worker_p2p, args=(WORLD, port, str(tmp_path)), nprocs=WORLD, join=True)
    from paper_2408_06167_b200 import dist as pdist
    O, T, Q, n_sets, (sk, pk, rlk, gk) = _setup()
    N = 1 << LOGN
    full_db = _encrypt_sets(O, T, pk, 0, n_sets)
    S = N // 2
    qc = O.encrypt(LOGN, pk, O.encode(O.pack_query(Q, LOGN, D, P_PARTS).reshape(-1, S), LOGN), 0, 3)
    ref, _ = O.match(LOGN, D, P_PARTS, 0, rlk, gk, full_db, qc.reshape(NQ, P_PARTS, 2, 2, N))
    ref = ref.reshape(NQ, n_sets * 2 * N)
    rmap = pdist.p2p_row_map(NQ, 2, WORLD)
    bufs = [np.load(tmp_path / f"p2p{r}.npy") for r in range(WORLD)]
    for j, (root, row) in enumerate(rmap):
        assert np.array_equal(bufs[root][row], ref[j])
    # the roots are the pipelined all_to_all's: group g's block k lands on rank k
    for g in range(2):
        for k in range(WORLD):
            q0, cnt = pdist.group_query_block(NQ, 2, WORLD, k, g)
            assert all(rmap[j][0] == k for j in range(q0, q0 + cnt))
    assert sorted(rmap) == sorted((k, i) for k in range(WORLD) for i in range(NQ // WORLD))


class _FakeIPC:
    """Stands in for the CUDA IPC calls of the binding (no GPU here): handles name the rank's
    buffer, opening maps rank k's buffer to a fake base 1000 (k + 1); `fail` makes one call raise."""

    def __init__(self, rank, fail=None):
        self.rank, self.fail, self.closed = rank, fail, []

    def bm_ipc_handle(self, res):
        if self.fail == ("handle", self.rank):
            raise RuntimeError("no handle")
        return bytes([self.rank]) * 64, 8 * self.rank

    def bm_ipc_open(self, h):
        if self.fail == ("open", self.rank):
            raise RuntimeError("no open")
        return 1000 * (h[0] + 1)

    def bm_ipc_close(self, b):
        self.closed.append(b)


def _worker_ipc(rank, world, port, out_dir, fail):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2408_06167_b200 import dist as pdist
    fake = _FakeIPC(rank, fail)
    res = torch.zeros(4, dtype=torch.int64)
    opened = []
    try:
        bases = pdist.exchange_ipc_bases(fake, res, opened)
        out = ("ok", [b - (res.data_ptr() if k == rank else 0) for k, b in enumerate(bases)])
    except RuntimeError as ex:
        out = ("raised", str(ex), fake.closed)
    np.save(os.path.join(out_dir, f"ipc{rank}.npy"), np.array([repr(out)]))
    dist.destroy_process_group()


@pytest.mark.parametrize("fail", [None, ("handle", 1), ("open", 0)])
def test_ipc_exchange_agrees_across_ranks(tmp_path, fail):
    """dist.exchange_ipc_bases: the peer bases are the opened handles plus each rank's offset, and a
    failure on ANY rank (handle or open) makes EVERY rank raise (bench.py then falls back to the
    NCCL gather on all ranks together) with the mappings already opened closed again."""
    port = _free_port()
    mp.spawn(_worker_ipc, args=(WORLD, port, str(tmp_path), fail), nprocs=WORLD, join=True)
    outs = [eval(str(np.load(tmp_path / f"ipc{r}.npy")[0])) for r in range(WORLD)]
    if fail is None:
        for r, o in enumerate(outs):
            assert o[0] == "ok"
            assert o[1] == [0 if k == r else 1000 * (k + 1) + 8 * k for k in range(WORLD)]
    else:
        assert all(o[0] == "raised" for o in outs)
        if fail[0] == "open":   # rank 1 had opened rank 0's buffer before rank 0 failed: closed again
            assert outs[1][2] == [1000]
