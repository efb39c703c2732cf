"""Multi-GPU plumbing of the scan ("Cluster Architecture"): the template DB is
sharded by sets over ranks (one process per GPU), the encrypted query is broadcast from the main
rank, each rank scans its own sets with bm_match, and the result ciphertexts are gathered.
No reduction exists on this path: sets are independent.

Gather: query j's results go to a root rank; roots are assigned in contiguous query blocks
(rank k owns queries [k nq/W, (k+1) nq/W)), so every rank is the root of the same number of
queries and the exchange is one all_to_all over the [nq][local sets][2][N] result buffers.
Collectives go through torch.distributed (NCCL on GPUs; gloo in the CPU tests).

Fused gather (P2PGather / scan_p2p): the output kernels of the scan store every result directly
into its root's buffer through CUDA IPC peer pointers (bm_match_rows over NVLink), so a8 overlaps
the scan pair by pair and no result collective runs; one 8-byte all-reduce orders the roots' reads
after every writer's scan.
"""
import torch
import torch.distributed as dist


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


def shard_sets(n_sets, world_size, rank):
    """Contiguous set range of `rank`: [r ceil(T/W), min(T, (r+1) ceil(T/W)))."""
    per = -(-n_sets // world_size)
    lo = min(n_sets, rank * per)
    hi = min(n_sets, lo + per)
    return lo, hi - lo


def query_block(nq, world_size, rank):
    """Queries whose gathered results land on `rank` (requires nq % world_size == 0)."""
    assert nq % world_size == 0, "nq must be a multiple of the world size"
    per = nq // world_size
    return rank * per, per


def broadcast_queries(d_q, src=0, group=None):
    """a3: replicate the query ciphertexts [nq][p][2][2][N] on every rank."""
    w, _ = world()
    if w > 1:
        dist.broadcast(d_q, src=src, group=group)
    return d_q


def gather_results(d_out, recv=None, group=None):
    """a8: d_out [nq][n_local][2][N] (this rank's sets) -> recv [W][nq/W][n_local][2][N]:
    recv[r] holds rank r's sets for the queries this rank is root of."""
    w, _ = world()
    if w == 1:
        return d_out.unsqueeze(0)
    nq = d_out.shape[0]
    assert nq % w == 0
    if recv is None:
        recv = torch.empty((w, nq // w) + tuple(d_out.shape[1:]), dtype=d_out.dtype, device=d_out.device)
    dist.all_to_all_single(recv.view(-1), d_out.contiguous().view(-1), group=group)
    return recv


def group_query_block(nq, groups, world_size, rank, g):
    """Pipelined gather: queries [g nq/G, (g+1) nq/G) of group g are split into W equal blocks and
    block k lands on rank k; returns (first query, count) of the block `rank` is root of."""
    assert nq % (groups * world_size) == 0, "nq must be a multiple of groups x world size"
    gq = nq // groups
    per = gq // world_size
    return g * gq + rank * per, per


def scan_pipelined(match, d_q, d_out, recv, groups, comm_stream=None, compute_stream=None):
    """a3 + scan + a8 for one query batch, overlapped over `groups` query groups.

    match(g, q_slice, out_slice) runs the local scan of group g (on the current stream).
    d_q [nq][p][2][2][N] (filled on rank 0), d_out [nq][n_local][2][N], recv
    [G][W][nq/(G W)][n_local][2][N].  Group g's broadcast and result all_to_all run on
    `comm_stream` while other groups are scanned on `compute_stream`: the collectives are issued in
    the same order on every rank (b0, b1, then a_g, b_{g+2}, ...), broadcasts two groups ahead.
    With one rank, or without CUDA streams (gloo), the same sequence runs in order.

    Bounded outputs (result sets larger than memory, BASELINE.json configs[3]): d_out and recv may
    instead be LISTS of R slots ([nq/G][n_local][2][N] and [W][nq/(G W)][n_local][2][N]); group g
    uses slot g mod R, overwriting group g - R's results (a slot is rewritten only after its
    previous all_to_all has completed)."""
    w, _ = world()
    nq = d_q.shape[0]
    G = groups
    assert nq % G == 0
    gq = nq // G
    qs = [d_q[g * gq:(g + 1) * gq] for g in range(G)]
    ring = isinstance(d_out, (list, tuple))
    if ring:
        outs = [d_out[g % len(d_out)] for g in range(G)]
        recv = [recv[g % len(recv)] for g in range(G)] if recv is not None else None
    else:
        outs = [d_out[g * gq:(g + 1) * gq] for g in range(G)]
    cuda = comm_stream is not None and compute_stream is not None
    if not cuda:
        for g in range(G):
            broadcast_queries(qs[g])
            match(g, qs[g], outs[g])
            if w > 1:
                gather_results(outs[g], recv[g])
        return recv
    bw = [None] * G
    done = [None] * G
    sent = [None] * G
    R = len(d_out) if ring else G

    def bcast(g):
        if w > 1:
            with torch.cuda.stream(comm_stream):
                bw[g] = dist.broadcast(qs[g], src=0, async_op=True)

    def a2a(g):
        if w > 1:
            with torch.cuda.stream(comm_stream):
                comm_stream.wait_event(done[g])
                dist.all_to_all_single(recv[g].view(-1), outs[g].view(-1), async_op=True).wait()
                sent[g] = torch.cuda.Event()
                sent[g].record(comm_stream)

    compute_stream.wait_stream(torch.cuda.current_stream())
    comm_stream.wait_stream(torch.cuda.current_stream())
    for g in range(min(2, G)):
        bcast(g)
    for g in range(G):
        with torch.cuda.stream(compute_stream):
            if bw[g] is not None:
                bw[g].wait()
            if g >= R and sent[g - R] is not None:   # the slot's previous results have left
                compute_stream.wait_event(sent[g - R])
            match(g, qs[g], outs[g])
            done[g] = torch.cuda.Event()
            done[g].record(compute_stream)
        if g >= 1:
            a2a(g - 1)
        if g + 2 < G:
            bcast(g + 2)
    a2a(G - 1)
    cur = torch.cuda.current_stream()
    cur.wait_stream(compute_stream)
    cur.wait_stream(comm_stream)
    return recv


def p2p_row_map(nq, groups, world_size, ring=None):
    """[(root rank, row in the root's buffer)] for every query of a batch, with the roots of the
    pipelined all_to_all (group g's queries split into W equal blocks, block k -> rank k): the root
    holds its G nq/(G W) rows in (group, block position) order.  With ring = R the root holds only R
    groups' rows: group g's rows are slot g mod R (bounded outputs; later groups overwrite)."""
    assert nq % (groups * world_size) == 0, "nq must be a multiple of groups x world size"
    gq = nq // groups
    per = gq // world_size
    out = []
    for j in range(nq):
        g, i = divmod(j, gq)
        k, m = divmod(i, per)
        out.append((k, (g if ring is None else g % ring) * per + m))
    return out


def exchange_ipc_bases(B, res, opened):
    """CUDA IPC exchange of the ranks' root buffers: [base address of rank k's buffer in this
    process] (this rank: res itself).  Opened peer mappings are appended to `opened`.  Every step is
    collective and agreed on: a rank that fails still takes part, so all ranks raise together (and
    bench.py falls back to the NCCL gather) instead of hanging in a collective."""
    w, r = world()
    try:
        mine = B.bm_ipc_handle(res)
    except Exception as ex:  # noqa: BLE001
        mine = repr(ex)
    allh = [None] * w
    dist.all_gather_object(allh, mine)
    bad = [x for x in allh if not isinstance(x, tuple)]
    if bad:
        raise RuntimeError(f"CUDA IPC handle unavailable: {bad[0]}")
    bases, err = [], None
    for k, (hk, ok) in enumerate(allh):
        if k == r:
            bases.append(res.data_ptr())
            continue
        try:
            b = B.bm_ipc_open(hk)
            opened.append(b)
            bases.append(b + ok)
        except Exception as ex:  # noqa: BLE001
            err = repr(ex)
            break
    errs = [None] * w
    dist.all_gather_object(errs, err)
    if any(e is not None for e in errs):
        for b in opened:
            B.bm_ipc_close(b)
        opened.clear()
        raise RuntimeError(f"CUDA IPC open failed: {next(e for e in errs if e is not None)}")
    return bases


class P2PGather:
    """a8 fused into the scan (bm_match_rows): `res` is this rank's root buffer
    [nq/W][n_sets_global][2][N] (int64, CUDA, the rows of p2p_row_map); the ranks exchange CUDA IPC
    handles of their buffers (all_gather_object) and open their peers', so `rows` holds, for every
    query of the batch, the device address of its row on its root GPU (nq int64 on this device)."""

    def __init__(self, B, res, nq, groups, n_sets_global, ring=None):
        w, r = world()
        self.B = B
        self.res = res
        self.ring = ring
        row_bytes = n_sets_global * 2 * B.N * 8
        if not (res.is_cuda and res.dtype == torch.int64 and res.is_contiguous()):
            raise ValueError("P2PGather: res must be a contiguous int64 CUDA tensor")
        n_rows = nq // w if ring is None else ring * (nq // groups // w)
        if res.numel() * 8 < n_rows * row_bytes:
            raise ValueError(f"P2PGather: res holds {res.numel() * 8} bytes, the rows need {n_rows * row_bytes}")
        self.opened = []
        if w == 1:
            bases = [res.data_ptr()]
        else:
            bases = exchange_ipc_bases(B, res, self.opened)
        addrs = [bases[k] + row * row_bytes for k, row in p2p_row_map(nq, groups, w, ring)]
        self.rows = torch.tensor(addrs, dtype=torch.int64, device=res.device)
        self.gq = nq // groups

    def rows_of(self, g):
        return self.rows[g * self.gq:(g + 1) * self.gq]

    def close(self):
        for b in self.opened:
            self.B.bm_ipc_close(b)
        self.opened = []


def scan_p2p(match_rows, d_q, gather, groups, comm_stream, compute_stream, flag):
    """a3 + scan + fused a8: group g's broadcast runs on `comm_stream` two groups ahead while the
    scans run on `compute_stream` (or, given a list of streams, group g on stream g mod len: one
    group's kernels fill the tails of the previous group's); match_rows(g, q_slice, rows_slice)
    writes every result straight to its root (gather.rows_of(g)).  `flag` (one float64 on this
    device) is all-reduced after the last scan of every stream: NCCL completes it only when every
    rank has passed its scans, so each root's buffer is complete once the call's work on the current
    stream is."""
    w, _ = world()
    nq = d_q.shape[0]
    G = groups
    gq = nq // G
    qs = [d_q[g * gq:(g + 1) * gq] for g in range(G)]
    bw = [None] * G
    cs = list(compute_stream) if isinstance(compute_stream, (list, tuple)) else [compute_stream]

    def bcast(g):
        if w > 1:
            with torch.cuda.stream(comm_stream):
                bw[g] = dist.broadcast(qs[g], src=0, async_op=True)

    for s in cs:
        s.wait_stream(torch.cuda.current_stream())
    comm_stream.wait_stream(torch.cuda.current_stream())
    for g in range(min(2, G)):
        bcast(g)
    for g in range(G):
        s = cs[g % len(cs)]
        with torch.cuda.stream(s):
            if bw[g] is not None:
                bw[g].wait()
            match_rows(g, qs[g], gather.rows_of(g))
        if g + 2 < G:
            bcast(g + 2)
    for s in cs[1:]:
        cs[0].wait_stream(s)
    with torch.cuda.stream(cs[0]):
        if w > 1:
            dist.all_reduce(flag)
    cur = torch.cuda.current_stream()
    cur.wait_stream(cs[0])
    cur.wait_stream(comm_stream)


def max_over_ranks(x, device):
    """max of a float over ranks (timing rule: the job time is the slowest rank)."""
    w, _ = world()
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    if w > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
