#!/usr/bin/env python
"""Benchmark of the encrypted 1:N cosine scan (HE-C^3) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C] [--p P]

Workloads (--config C = SURVEY.md sec. 8d C1..C5 = BASELINE.json configs[C-1]; default C = 4):
  C4 (the metric's own configuration, BASELINE.json "d=128, N=8192 at 1/2/4/8 B200"): 1,048,576
     unit-norm Gaussian templates (stand-ins for IJB-C ArcFace embeddings), d = 128,
     p = 8 (the best of the C2 sweep), 256 queries (128 genuine + 128 impostor), the database
     STRONG-scaled over the N GPUs (rank r owns the contiguous sets dist.shard_sets(4096, N, r),
     encrypted with their global object numbers and one shared seed: a bit-exact partition of the
     1-GPU database).  Results (128 KiB per (query, set) pair, 128 GiB per batch) stream through a
     bounded device ring (--ring-gib, overwritten), the paper's cluster setting.
  C2: 6,144 templates, 384 genuine queries, p in {1,2,4,8};  C3: d = 32, 65,536 clustered templates,
  64 queries, p in {1,2,4};  C5: d = 512, 4,194,304 templates, 1,024 queries, p in {4,8,16} (at N < 8
  --shard-of 8 runs rank 0's shard of the 8-GPU split: a labelled 1-GPU prefix);  C1: d = 16, one set.
One step = the whole hot path for the whole query batch: bm_match of every (query, set) pair of
this rank (tensor + part sum, relinearise, rescale, log2(s) rotate-and-add steps, coefficient-
domain output) in query groups of ~16K pairs alternating two streams, plus for N > 1 the query
broadcast (a3) and the result gather (a8, fused into the output kernels as NVLink peer stores).
Metric: encrypted templates matched per second = templates x queries / s, all ranks (BASELINE.json).

After the timed region the same step runs once more, untimed, with every result decrypted on the
device (bm_decrypt_dev) and checked: max |score - float64 cosine|, top-1 agreement with the
plaintext argmax, and a sample of >= 32 pairs (spread over query groups, sets and the last set)
compared bit for bit with the CPU oracle (oracle/, which also re-encrypts those sets and queries).

--impl reference runs the CPU oracle (oracle/, plain C) on the host cores on a bounded sample of
the same workload (this tier has no reference implementation).
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_RING = 8192
BFLY = (N_RING // 2) * 13          # butterflies (= modmuls) per 8192-point transform
IMAD_PER_CLK_SM = 64               # FMA-heavy pipe, 16 lanes/clk/SMSP (B300_MICROARCH.md "Pipe rates")
# FMA-pipe issue slots (in IMAD units) of the cheapest 64-bit Shoup modmul a w mod q: 4 IMAD (low
# words) + 3 IMAD.WIDE + 2 IMAD.HI, the wide / high forms at half the IMAD rate (measured 25-29 vs
# 63 lanes/clk/SM, tools/pipe_bench.cu, profiles/r01_pipe_bench.txt): 4 + 2 x 5 = 14
IMAD_SLOTS_PER_MODMUL = 14
METRIC = "encrypted templates matched/sec (d=128, N=8192)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5],
                    help="SURVEY.md sec. 8d C1..C5 = BASELINE.json configs[0..4]")
    ap.add_argument("--p", type=int, default=None, help="parts (default: the config's)")
    ap.add_argument("--nq", type=int, default=None, help="queries per batch (default: the config's)")
    ap.add_argument("--order", type=int, default=0, choices=[0, 1, 2, 4],
                    help="0 hoisted (product), 1 paper order, 2 f2 hoisted rotations, 4 f2 baby-step giant-step")
    ap.add_argument("--shard-of", type=int, default=None,
                    help="run rank r's shard of an S-way split (C5 default at N < 8: 8, a labelled prefix)")
    ap.add_argument("--ring-gib", type=float, default=4.0, help="device result ring (bounded outputs)")
    ap.add_argument("--chunk", type=int, default=16384, help="pairs per query group / bm_match chunk")
    ap.add_argument("--streams", type=int, default=2, choices=[1, 2])
    ap.add_argument("--group-queries", type=int, default=None,
                    help="queries per bm_match call (default: ~--chunk pairs, at least 8 when the batch has them)")
    ap.add_argument("--gather", choices=["p2p", "nccl"], default="p2p",
                    help="N > 1 result gather (a8): p2p = fused into the output kernels (bm_match_rows storing "
                         "to the roots over NVLink), nccl = all_to_all after each group's scan")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--oracle-pairs", type=int, default=48)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-single", action="store_true", help="skip the single-query latency leg")
    ap.add_argument("--no-extras", action="store_true", help="skip the NEXT-row legs (f1, f3, f4 on configs[1])")
    ap.add_argument("--opt", action="append", default=[],
                    help="library option NAME=VALUE (bm.OPTIONS; A/B runs only, the defaults are the product)")
    ap.add_argument("--no-tc", action="store_true",
                    help="do not register the DB in the tensor-core layout (K1 on the CUDA cores; A/B runs)")
    ap.add_argument("--quiet", action="store_true")
    return ap.parse_args()


def log(args, *a):
    if not args.quiet:
        print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- algorithmic work
def class_modmuls(p, log_s, order=0):
    """Algorithmic 64-bit modular multiplications per (query, set) pair, per kernel class
    (DESIGN.md "Algorithmic work"): butterflies of every transform + pointwise products."""
    n = N_RING
    s = 1 << log_s
    if order == 4 and log_s:    # f2 BSGS: two hoisted passes of b - 1 and g - 1 rotations (g = 1: one pass)
        b = 1 << ((log_s + 1) // 2)
        g = s // b
        hrot = 6 * BFLY + 4 * n * (b - 1) + ((6 * BFLY + 4 * n * (g - 1)) if g > 1 else 0)
    else:
        hrot = (6 * BFLY + 4 * n * (s - 1)) if log_s else 0  # f2: 6 transforms + 4 products per rotation
    return {
        "tensor": 8 * n * p,                                       # a0b0, a1b1, (a0+a1)(b0+b1) per limb (+ adds)
        "digits": 6 * BFLY + n,                                    # INTT_q0, INTT_q1, NTT_q1, NTT_P x2, NTT_q0
        "relin": 6 * BFLY + 12 * n + 8 * n,                        # INTT_P, INTT_q1, NTT_q0 x 2 comps; rlk + scalings
        "ladder": (6 * BFLY + 6 * n) * log_s,                      # digit INTT_q0 + NTT_P, 2 x (INTT_P + NTT_q0)
        "hrot": hrot,
        "out_intt": 0 if log_s else 2 * BFLY,
    }


def hbm_bytes_per_step(p, n_sets, nq):
    """Algorithmic HBM bytes of one step: DB read once, queries read once, results written once."""
    return n_sets * p * 4 * N_RING * 8 + nq * p * 4 * N_RING * 8 + nq * n_sets * 2 * N_RING * 8


def int_peak_gmodmul(n_sm, f_hz):
    """Derived integer roofline: n_SM x 64 IMAD/clk x f / 14 IMAD slots per modmul."""
    return n_sm * IMAD_PER_CLK_SM * f_hz / IMAD_SLOTS_PER_MODMUL / 1e9


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons DURING the timed region: NVML polled every 5 ms
    from a thread, falling back to `nvidia-smi -lms 100` where NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits (nvml.h): sw power cap 0x4, hw slowdown 0x8, sw thermal 0x20, hw thermal 0x40
    REASON_BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []          # (sm_mhz, max_mhz, set of reason names)
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = self._handle(pynvml)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001 -- no NVML: nvidia-smi
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _handle(self, nv):
        # the CUDA device's PCI address (NVML indices ignore CUDA_VISIBLE_DEVICES), else the index
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.idx)
            return nv.nvmlDeviceGetHandleByPciBusId(f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
        except Exception:  # noqa: BLE001
            return nv.nvmlDeviceGetHandleByIndex(self.idx)

    def _poll(self):
        nv = self.nvml
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
        mx = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
        while not self.stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                bits = int(get_reasons(self.h))
                self.rows.append((sm, mx, {k for k, v in self.REASON_BITS.items() if bits & v}))
            except Exception:  # noqa: BLE001
                pass
            self.stop.wait(0.005)

    def _read(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            try:
                self.rows.append((float(r[0]), float(r[1]),
                                  {nm for k, nm in enumerate(names) if len(r) > 4 + k and r[4 + k].lower().startswith("active")}))
            except (ValueError, IndexError):
                continue

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
            try:
                self.nvml.nvmlShutdown()
            except Exception:  # noqa: BLE001
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = list(self.rows)
        sm = [s for s, m, _ in rows if s > 0.5 * m]    # under load
        reasons = set().union(*[r for _, _, r in rows]) if rows else set()
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": rows[-1][1] if rows else None,
                "reasons": sorted(reasons), "samples": len(rows), "samples_under_load": len(sm),
                "source": "nvml (5 ms)" if self.nvml is not None else "nvidia-smi -lms 100"}


# ----------------------------------------------------------------------------- workload
class Workload:
    """The (config, p) workload and this rank's share of it."""

    def __init__(self, cfg, p, nq, world, rank, shard_of, chunk, group_queries=None):
        from paper_2408_06167_b200 import dist as pdist
        from paper_2408_06167_b200 import inputs as I
        c = I.CONFIGS[cfg]
        self.cfg, self.d, self.n = cfg, c["d"], c["n"]
        self.p = p or c["p"]
        self.nq = nq or c["nq"]
        s = self.d // self.p
        self.B = 4096 // s
        self.n_sets = -(-self.n // self.B)
        self.split = shard_of or world                    # the DB split this run executes a share of
        self.rank_in_split = rank
        self.lo, self.n_local = pdist.shard_sets(self.n_sets, self.split, rank)
        self.tmpl_lo = self.lo * self.B
        self.n_tmpl_local = max(0, min(self.n, (self.lo + self.n_local) * self.B) - self.tmpl_lo)
        # query groups: ~chunk pairs each, at least 8 queries when the batch has them (bm_match then cuts
        # 8-query chunks: the tensor's full tiles); for N > 1 a group splits evenly over the ranks (roots)
        want = group_queries or max(1, chunk // max(1, self.n_local), min(8, self.nq))
        if world > 1:
            cands = [g for g in range(world, self.nq + 1, world) if self.nq % g == 0]
            assert cands, "nq must be a multiple of the world size"
            self.gq = max([g for g in cands if g <= max(want, world)] or [cands[0]])
        else:
            self.gq = min(self.nq, want)
        self.G = -(-self.nq // self.gq)

    def label(self):
        lab = f"BASELINE configs[{self.cfg - 1}]: d={self.d}, {self.n} templates, {self.nq} queries, p={self.p}"
        if self.split > 1:
            lab += f", DB split over {self.split} GPUs ({self.n_local} of {self.n_sets} sets on this rank)"
        return lab


# ----------------------------------------------------------------------------- oracle (cpu_baseline / reference)
def oracle_sample(cfg, d, p, seconds_target, n_threads):
    """Time the CPU oracle on a bounded sample of (query, set) pairs of the workload (two sets of the
    config's templates, two of its queries, cycled)."""
    from oracle import oracle as O
    from paper_2408_06167_b200 import inputs as I
    logN = 13
    S, s, B = O.layout(logN, d, p)
    sk, pk, rlk, gk = O.keygen(logN, 1, O.n_rot_for(d, p))
    T = I.templates(cfg, 2 * B)            # two full sets
    Q = I.random_unit(2, d, 7) if cfg != 2 else I.queries(cfg, 2)[0]
    db = O.encrypt(logN, pk, O.encode(O.pack_db(T, logN, d, p, 0, 2).reshape(-1, S), logN), 0, 2).reshape(2, p, 2, 2, -1)
    qc = O.encrypt(logN, pk, O.encode(O.pack_query(Q, logN, d, p).reshape(-1, S), logN), 0, 3).reshape(2, p, 2, 2, -1)
    t0 = time.perf_counter()
    O.match(logN, d, p, 0, rlk, gk, db, qc, pairs=np.array([[0, 0]], np.int64), n_threads=1)
    t1 = time.perf_counter() - t0
    n_pairs = int(max(n_threads, min(4096, round(seconds_target * n_threads / max(t1, 1e-3)))))
    pairs = np.array([(k % 2, (k // 2) % 2) for k in range(n_pairs)], np.int64)

    def run():
        t = time.perf_counter()
        O.match(logN, d, p, 0, rlk, gk, db, qc, pairs=pairs, n_threads=n_threads)
        return time.perf_counter() - t
    return run, n_pairs, B, t1


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2408_06167_b200 import build as pbuild
    from paper_2408_06167_b200 import dist as pdist
    from paper_2408_06167_b200 import inputs as I

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        pbuild.build(verbose=False)
    if world > 1:
        dist.barrier()
    from paper_2408_06167_b200 import bm as B
    # seeded streams (BM_RNG_SEEDED): the DB shards must be bit-exact slices of one database across
    # ranks and the in-bench oracle check re-encrypts with the same streams (the library default is
    # OS entropy)
    B.bm_rng_mode(B.RNG_SEEDED)
    for o in args.opt:
        k, v = o.split("=")
        B.bm_set_option(k, int(v))

    shard_of = args.shard_of if args.shard_of else (8 if args.config == 5 and world < 8 else None)
    if shard_of is not None and world > 1 and shard_of != world:
        raise SystemExit("--shard-of applies to single-GPU prefix runs only")
    W = Workload(args.config, args.p, args.nq, world, rank, shard_of, args.chunk, args.group_queries)
    p, nq, order, d = W.p, W.nq, args.order, W.d
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    prm = B.bm_params_init(d, p)
    t_setup = time.perf_counter()
    sk, pk, evk = B.bm_keygen(prm, 1)                # deterministic: identical keys on every rank
    if order in (2, 4):                              # f2 hoisted / BSGS rotation sums: keys of every rotation
        B.bm_evk_add_hoisted(prm, 1, evk)
    pk_dev, evk_dev = B.bm_pk_to_device(prm, pk), B.bm_evk_to_device(prm, evk)
    n_local = W.n_local
    T_local = I.templates(W.cfg, W.n_tmpl_local, W.tmpl_lo)
    d_db = torch.empty((n_local, p, 2, 2, N_RING), dtype=torch.int64, device=dev)
    # global object numbers (set t, part i -> t p + i) and one seed: every rank's shard is a bit-exact
    # slice of the 1-GPU database (packing is position-independent, so the local templates suffice)
    if n_local:
        pt = torch.from_numpy(B.bm_encode_db(prm, T_local, 0, n_local).reshape(-1, N_RING)).to(dev)
        B.bm_encrypt(prm, pk_dev, pt, W.lo * p, 2, d_db)
        del pt
    # server-side enrollment of the DB into the tensor-core layout (K1 on tcgen05):
    # part of the DB's setup like its encryption, outside the timed region
    d_dbp = None
    if n_local and not args.no_tc and B.bm_db_tc_bytes(prm, n_local):
        d_dbp = torch.empty(B.bm_db_tc_bytes(prm, n_local), dtype=torch.uint8, device=dev)
        B.bm_db_tc_register(prm, d_db, n_local, d_dbp)
    Q, genuine = I.queries(W.cfg, nq)
    d_q = torch.zeros((nq, p, 2, 2, N_RING), dtype=torch.int64, device=dev)
    if rank == 0:
        B.bm_encrypt_query(prm, pk_dev, Q, 0, 3, d_q)
    B.bm_sync()
    t_setup = time.perf_counter() - t_setup
    # bounded outputs: a ring of R group slots (R even: group g and g + R share a stream)
    B.bm_set_option("chunk_pairs", max(1, min(args.chunk, W.gq * n_local)))   # pairs per bm_match chunk
    nstr = args.streams
    row_bytes = n_local * 2 * N_RING * 8
    slot_bytes = W.gq * row_bytes
    R = max(2, int(args.ring_gib * 2**30 // max(1, slot_bytes)) // 2 * 2)
    R = min(R, W.G + (W.G % 2))
    ws = [torch.empty(max(1, B.bm_match_ws_bytes(prm, n_local, W.gq, order)), dtype=torch.uint8, device=dev)
          for _ in range(nstr)]
    streams = [torch.cuda.Stream() for _ in range(nstr)]
    comm_s = torch.cuda.Stream() if world > 1 else None
    gather, gat, flag, ring, recv = "local ring", None, None, None, None
    if world > 1 and args.gather == "p2p":
        n_root = R * (W.gq // world)
        res = torch.empty((n_root, W.n_sets, 2, N_RING), dtype=torch.int64, device=dev)
        try:
            gat = pdist.P2PGather(B, res, nq, W.G, W.n_sets, ring=R)
            flag = torch.zeros(1, dtype=torch.float64, device=dev)
            gather = "p2p: fused into the output kernels (bm_match_rows, CUDA IPC peer stores over NVLink), root ring"
        except Exception as ex:  # noqa: BLE001 -- a transport fallback (NCCL), never a CPU one
            del res
            gather = f"nccl all_to_all (p2p unavailable: {type(ex).__name__}: {ex})"[:200]
    if gat is None:
        ring = [torch.empty((W.gq, n_local, 2, N_RING), dtype=torch.int64, device=dev) for _ in range(R)]
        if world > 1:
            recv = [torch.empty((world, W.gq // world, n_local, 2, N_RING), dtype=torch.int64, device=dev)
                    for _ in range(R)]
            if gather == "local ring":
                gather = "nccl all_to_all per query group"
    log(args, f"[rank {rank}] setup {t_setup:.1f} s: {W.label()}; {n_local} local sets x {nq} queries, "
              f"{W.G} groups of {W.gq}, ring {R} x {slot_bytes / 2**30:.2f} GiB, ws {nstr} x {ws[0].numel() / 2**30:.2f} GiB")
    main = torch.cuda.current_stream()

    def groups():
        for g in range(W.G):
            q0 = g * W.gq
            yield g, q0, min(W.gq, nq - q0)

    def step():
        if world == 1:
            for s in streams:
                s.wait_stream(main)
            for g, q0, n in groups():
                i = g % nstr
                B.bm_match(prm, evk_dev, d_db, n_local, d_q[q0:q0 + n], n, ring[g % R][:n], ws[i], order,
                           stream=streams[i])
            for s in streams:
                main.wait_stream(s)
        elif gat is not None:
            def match_rows(g, q_g, rows_g):
                i = g % nstr
                B.bm_match_rows(prm, evk_dev, d_db, n_local, q_g, q_g.shape[0], rows_g, W.lo, ws[i], order,
                                stream=torch.cuda.current_stream())
            pdist.scan_p2p(match_rows, d_q, gat, W.G, comm_s, streams, flag)
        else:
            def match(g, q_g, out_g):
                B.bm_match(prm, evk_dev, d_db, n_local, q_g, q_g.shape[0], out_g, ws[0], order,
                           stream=torch.cuda.current_stream())
            pdist.scan_pipelined(match, d_q, ring, recv, W.G, comm_s, streams[0])

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    B.bm_launch_count_reset()
    # events at every step boundary (recorded on the launching stream, no synchronisation between
    # steps): the first and last bracket the timed region, the others give the per-step spread
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev[0].record(main)
        for i in range(args.steps):
            step()
            ev[i + 1].record(main)
        while not ev[-1].query():   # wait without holding the GIL, so the clock sampler thread runs
            time.sleep(0.0005)
        torch.cuda.synchronize()
    launches = B.bm_launch_count()
    if world > 1:
        dist.barrier()
    ms = pdist.max_over_ranks(ev[0].elapsed_time(ev[-1]), dev)
    ms_step = ms / args.steps
    per_step = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    ms_std = float(statistics.pstdev(per_step)) if len(per_step) > 1 else 0.0
    n_tmpl_job = W.n if W.split == world else W.n_tmpl_local   # templates all ranks of THIS run scan
    tq_per_step = n_tmpl_job * nq
    value = tq_per_step / (ms_step / 1e3)
    clocks = clk.summary()

    # per-kernel-class device times (the library's CUDA events around every launch, on its launching
    # stream), a separate profiled pass of the same step on one stream
    roofline = profile_pass(args, B, torch, prm, evk_dev, d_db, n_local, d_q, ring, gat, ws, W, order, n_sm, clocks,
                            ms_step, groups, tc_k1=d_dbp is not None and "tensor_mma=0" not in args.opt)

    verify = None
    if not args.no_verify:
        try:
            verify = run_verify(args, B, torch, prm, sk, pk, evk_dev, d_db, d_q, Q, genuine, T_local, W, ring, gat,
                                ws, order, world, rank, dev)
        except Exception as ex:  # noqa: BLE001 -- recorded, and the line says parity failed
            import traceback
            traceback.print_exc()
            verify = {"error": f"{type(ex).__name__}: {ex}"[:300], "parity": "error"}

    single = None
    if world == 1 and not args.no_single:
        single = run_single(B, torch, prm, evk_dev, d_db, n_local, W.n_tmpl_local, d_q, ring, ws[0], order, main)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, B, torch, prm, evk_dev, d_db, n_local, d_q, W, order, dev, world, tq_per_step)

    extras = {}
    if world == 1 and not args.no_extras and args.config in (2, 4) and order == 0:
        del ring, ws
        torch.cuda.empty_cache()
        try:
            extras = run_extras(args, B, torch, dev, main)
        except Exception as ex:  # noqa: BLE001
            extras = {"error": f"{type(ex).__name__}: {ex}"[:300]}
            log(args, f"[rank {rank}] extras failed: {extras['error']}")
        torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nth = os.cpu_count() or 1
        run, n_pairs, Bk, t1 = oracle_sample(W.cfg, d, p, 12.0, nth)
        secs = run()
        cpu = {"value": round(n_pairs * Bk / secs, 2), "unit": "templates*queries/s", "cores": nth, "kind": "oracle",
               "sample": f"{n_pairs} (query, set) pairs of the {W.label().split(':')[0]} workload (d={d}, p={p}, {Bk} "
                         f"templates each), {nth} threads, {secs:.1f} s wall; single pair {t1:.2f} s on 1 thread"}

    if rank == 0:
        hbm_bytes = hbm_bytes_per_step(p, W.n_sets if W.split == world else n_local, nq)
        hbm_gbs = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
            os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.8
        roofline["hbm"] = {"achieved_gbs": round(hbm_bytes / (ms_step / 1e3) / 1e9, 2), "peak_gbs": hbm_gbs,
                           "frac": round(hbm_bytes / (ms_step / 1e3) / 1e9 / hbm_gbs, 5),
                           "algorithmic_bytes_per_step": hbm_bytes}
        scaling = "strong" if W.split == world and world > 1 else "weak"
        line = {
            "metric": METRIC, "value": round(value, 1),
            "unit": "templates*queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "ms_per_step_std": round(ms_std, 4),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "u64", "data": "synthetic (seeded unit-norm Gaussian templates, genuine noisy queries + impostors)",
            "config": {"workload": W.label() + (f"; 1-GPU prefix: rank 0's shard of the {W.split}-GPU split"
                                                 if W.split > world else ""),
                       "d": d, "p": p, "templates": W.n, "templates_this_run": n_tmpl_job, "queries": nq,
                       "sets": W.n_sets, "sets_per_gpu": n_local, "ring_N": N_RING,
                       "order": ["hoisted", "paper", "hoisted-rotations (f2, not the paper ladder)", "degree-2 (f2)",
                                 "baby-step giant-step rotations (f2, not the paper ladder)"][order],
                       "parallelism": f"db-shard{world}", "gather": gather,
                       "query_groups": W.G, "group_queries": W.gq, "streams": nstr,
                       "output_ring": {"slots": R, "slot_bytes": slot_bytes},
                       "l2": "inputs > L2: DB %.0f MB + queries %.0f MB per step, results %.0f MB written (126 MB L2), "
                             "no flush" % (n_local * p * 4 * N_RING * 8 / 1e6, nq * p * 4 * N_RING * 8 / 1e6,
                                           nq * n_local * 2 * N_RING * 8 / 1e6)},
            "roofline": roofline, "verify": verify, "cpu_baseline": cpu, "e2e": e2e, "single_query": single,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "setup_s": round(t_setup, 1),
        }
        line["config"]["k1"] = ("tensor cores (tcgen05.mma kind::i8, DB registered in the tensor-core layout)"
                                if d_dbp is not None and "tensor_mma=0" not in args.opt else "CUDA cores")
        if args.opt:
            line["config"]["options"] = args.opt
        line.update(extras)
        print(json.dumps(line), flush=True)
    if gat is not None:
        dist.barrier()
        gat.close()
    if world > 1:
        dist.destroy_process_group()


def profile_pass(args, B, torch, prm, evk_dev, d_db, n_local, d_q, ring, gat, ws, W, order, n_sm, clocks, ms_step,
                 groups, tc_k1=False):
    """Per-kernel-class device times: the library records CUDA events around each launch on its
    launching stream (bm_set_profiling); one stream, min(steps, 2) steps of the same work."""
    nsteps = max(1, min(args.steps, 2))
    B.bm_set_profiling(True)
    B.bm_profile_reset()
    out = ring[0] if ring is not None else torch.empty((W.gq, n_local, 2, N_RING), dtype=torch.int64,
                                                       device=d_db.device)
    for _ in range(nsteps):
        for g, q0, n in groups():
            B.bm_match(prm, evk_dev, d_db, n_local, d_q[q0:q0 + n], n, out[:n], ws[0], order)
    B.bm_sync()
    pms, pla, pun = B.bm_profile_read()
    B.bm_set_profiling(False)
    p = W.p
    mm = class_modmuls(1 if order == 1 else p, prm.log_s, order)  # order 1 runs the part rounds one part each
    rounds = p if order == 1 else 1
    pairs = n_local * W.nq
    per_class, step_work = {}, 0.0
    # relin and ladder: the library counts the transforms it ran (component 0 split for the one-CTA
    # ladder: one transform fewer in K3 and in every ladder step but the last)
    # P-scaled one-CTA ladder (bm_build_info "pscale"): no P^-1 y^c products in the steps but the last
    lad_pw = 6 * prm.log_s - (2 * (prm.log_s - 1) if "pscale" in B.bm_build_info() and order == 0 and prm.log_s else 0)
    pointwise = {"relin": 20 * N_RING, "ladder": lad_pw * N_RING}
    for i, c in enumerate(B.PROFILE_CLASSES):
        if pla[i]:
            if c in pointwise and order in (0, 1):
                work = pun[i] * BFLY + pointwise[c] * pairs * nsteps * (rounds if i < 3 else 1)
            else:
                work = mm[c] * pairs * nsteps * (rounds if i < 3 else 1)
            if not (tc_k1 and c == "tensor"):   # the tensor-core K1's byte MACs are not integer-pipe modmuls
                step_work += work / nsteps
            # work: what the kernels execute after the exact rewritings (fewer transforms and products);
            # work_8d: SURVEY.md sec. 8(d)'s per-pair figure of the method itself (a7: 6 transforms + 6 N
            # products per step; a5 + a6: 12 transforms + ~18-20 N), the roofline contract's "algorithmic" work
            work_8d = mm[c] * pairs * nsteps * (rounds if i < 3 else 1)
            per_class[c] = {"ms_per_step": pms[i] / nsteps, "launches": int(pla[i]),
                            "ms_per_launch": pms[i] / pla[i], "gmodmul_s": work / (pms[i] / 1e3) / 1e9,
                            "modmul_per_launch": work / pla[i],
                            "gmodmul_s_8d": work_8d / (pms[i] / 1e3) / 1e9, "modmul_per_launch_8d": work_8d / pla[i]}
    dom = max(per_class, key=lambda c: per_class[c]["ms_per_step"])
    f_peak = (clocks["sm_max_mhz"] or 1965.0) * 1e6
    peak = int_peak_gmodmul(n_sm, f_peak)
    ach = per_class[dom]["gmodmul_s_8d"]     # the contract's achieved: sec. 8(d) work / launch duration
    ach_x = per_class[dom]["gmodmul_s"]      # the modmuls the kernel executes / launch duration
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile))
        traffic = tj.get(f"C{W.cfg}", {}).get(dom) if f"C{W.cfg}" in tj else tj.get(dom)
    measured = None
    mfile = os.path.join(ROOT, "profiles", "modmul_peak.json")
    if os.path.exists(mfile):
        mj = json.load(open(mfile))
        measured = {"peak": mj["gmodmul_s"], "frac": round(ach / mj["gmodmul_s"], 4),
                    "frac_executed": round(ach_x / mj["gmodmul_s"], 4), "basis": mj["basis"]}
    return {"bound": "alu", "kernel": dom, "achieved": round(ach, 2), "peak": round(peak, 2),
            "unit": "Gmodmul/s", "frac": round(ach / peak, 4), "traffic": traffic,
            "achieved_basis": f"{dom}: SURVEY.md sec. 8(d) algorithmic modmuls per launch "
                              f"({per_class[dom]['modmul_per_launch_8d']:.4g}; the ladder: (6 transforms x 53,248 "
                              f"butterflies + 6 N products) x log2 s per pair, DESIGN.md sec. 3) / mean launch duration "
                              f"({per_class[dom]['ms_per_launch']:.3f} ms, CUDA events on the launching stream, profiled pass)",
            "executed": {"achieved": round(ach_x, 2), "frac": round(ach_x / peak, 4),
                         "basis": f"the modmuls the kernel executes per launch ({per_class[dom]['modmul_per_launch']:.4g}: "
                                  f"the transforms the library reports it ran -- component 0 split, 5 per ladder step "
                                  f"but the last -- and 4 N instead of 6 N products per step on the P-scaled ladder; "
                                  f"exact rewritings, DESIGN.md sec. 3) / the same duration: the pipe-utilisation view"},
            "peak_basis": f"{n_sm} SMs x {IMAD_PER_CLK_SM} IMAD/clk x {f_peak / 1e6:.0f} MHz / "
                          f"{IMAD_SLOTS_PER_MODMUL} IMAD issue slots per 64-bit Shoup modmul "
                          f"(4 IMAD + 3 IMAD.WIDE + 2 IMAD.HI at half rate)",
            "peak_measured": measured,
            "step_gmodmul_s": round(step_work / (ms_step / 1e3) / 1e9, 2),
            "step_basis": ("integer-pipe kernels (digits, relin, ladder) over the whole step time; K1 runs on the "
                           "tcgen05 tensor cores (its per_class entry counts the 8 N p modmul-equivalents of the "
                           "CUDA-core K1)" if tc_k1 else "all kernels' algorithmic modmuls over the step time"),
            "step_frac": round(step_work / (ms_step / 1e3) / 1e9 / peak, 4),
            "per_class": {c: {k: round(v, 4) for k, v in d.items()} for c, d in per_class.items()}}


def pick_pairs(W, n, seed=5):
    """>= n (query, GLOBAL set) pairs of this rank spread over query groups, sets, both ends and the
    last set (ragged when the templates do not fill it)."""
    rng = np.random.default_rng(seed)
    lo, nl, nq = W.lo, W.n_local, W.nq
    if nl == 0:
        return []
    n = min(n, nq * nl)                          # configs[0]: one pair in all
    pairs = {(0, lo), (nq - 1, lo + nl - 1), (min(W.gq, nq - 1), lo), (W.gq - 1, lo + nl - 1),
             (nq // 2, lo + nl // 2)}
    for g in range(W.G):                         # one pair per query group at least
        pairs.add((min(nq - 1, g * W.gq + int(rng.integers(W.gq))), lo + int(rng.integers(nl))))
        if len(pairs) >= n:
            break
    while len(pairs) < n:
        pairs.add((int(rng.integers(nq)), lo + int(rng.integers(nl))))
    return sorted(pairs)


def run_verify(args, B, torch, prm, sk, pk, evk_dev, d_db, d_q, Q, genuine, T_local, W, ring, gat, ws, order, world,
               rank, dev):
    """One more (untimed) pass of the step with every result decrypted on the device and checked:
    scores vs float64 cosine, top-1 vs the plaintext argmax, and sampled pairs bit for bit vs the
    CPU oracle (which re-encrypts their sets and queries from the product's integer plaintexts)."""
    from paper_2408_06167_b200 import dist as pdist
    t0 = time.perf_counter()
    n_local, nq, Bk = W.n_local, W.nq, W.B
    nt = W.n_tmpl_local
    if nt == 0:
        return {"note": "no local sets"}
    sk_dev = B.bm_sk_to_device(prm, sk)
    Tt = torch.from_numpy(np.ascontiguousarray(T_local)).to(dev)
    Qd = torch.from_numpy(np.ascontiguousarray(Q)).to(dev)
    Qd = Qd / Qd.norm(dim=1, keepdim=True)
    max_err = torch.zeros((), dtype=torch.float64, device=dev)
    dec_top = torch.empty(nq, dtype=torch.int64, device=dev)
    pt_top = torch.empty(nq, dtype=torch.int64, device=dev)
    gap = torch.empty(nq, dtype=torch.float64, device=dev)
    sample = pick_pairs(W, args.oracle_pairs)
    got = {}
    out = ring[0] if ring is not None else torch.empty((W.gq, n_local, 2, N_RING), dtype=torch.int64, device=dev)
    scores = torch.empty((W.gq * n_local, Bk), dtype=torch.float64, device=dev)
    for g in range(W.G):
        q0 = g * W.gq
        n = min(W.gq, nq - q0)
        B.bm_match(prm, evk_dev, d_db, n_local, d_q[q0:q0 + n], n, out[:n], ws[0], order)
        B.bm_decrypt_dev(prm, sk_dev, out[:n], scores[:n * n_local])
        sc = scores[:n * n_local].view(n, n_local * Bk)[:, :nt]
        cos = Qd[q0:q0 + n] @ Tt.T
        max_err = torch.maximum(max_err, (sc - cos).abs().max())
        dec_top[q0:q0 + n] = sc.argmax(dim=1)
        top2 = cos.topk(min(2, nt), dim=1)
        pt_top[q0:q0 + n] = top2.indices[:, 0]
        gap[q0:q0 + n] = (top2.values[:, 0] - top2.values[:, -1]) if nt > 1 else 1.0
        for j, t in sample:
            if q0 <= j < q0 + n:
                got[(j, t)] = out[j - q0, t - W.lo].cpu().numpy().view(np.uint64).copy()
    torch.cuda.synchronize()
    dec_top, pt_top, gap = dec_top.cpu().numpy(), pt_top.cpu().numpy(), gap.cpu().numpy()
    gen = np.asarray(genuine)
    is_gen = gen >= 0
    in_shard = is_gen & (gen >= W.tmpl_lo) & (gen < W.tmpl_lo + nt)
    ties = gap < 1e-5
    agree = dec_top == pt_top
    res = {
        "max_abs_score_err": float(max_err.item()),
        "scores_checked": int(nq * nt),
        "top1_agree_all": float(agree.mean()),
        "top1_agree_genuine": float(agree[is_gen].mean()) if is_gen.any() else None,
        "genuine_queries": int(is_gen.sum()),
        "genuine_top1_is_enrolled_template": (float((dec_top[in_shard] + W.tmpl_lo == gen[in_shard]).mean())
                                              if in_shard.any() else None),
        "near_ties_flagged": int(ties.sum()),
        "tolerance": 1e-4,
    }
    # ---- oracle parity on the sampled pairs (rank-local sets)
    from oracle import oracle as O
    logN, d, p = 13, W.d, W.p
    osk, opk, orlk, ogk = O.keygen(logN, 1, O.n_rot_for(d, p))
    if order in (2, 4):
        ogk = O.keygen_hoisted(logN, 1, d // p)
    sets = sorted({t for _, t in sample})
    qs = sorted({j for j, _ in sample})
    si = {t: k for k, t in enumerate(sets)}
    qi = {j: k for k, j in enumerate(qs)}
    db_c = torch.empty((len(sets), p, 2, 2, N_RING), dtype=torch.int64, device=dev)
    for k, t in enumerate(sets):
        db_c[k] = d_db[t - W.lo]
    B.bm_ct_to_coeff(prm, db_c, 2, db_c)
    q_c = torch.stack([d_q[j] for j in qs]).contiguous()
    B.bm_ct_to_coeff(prm, q_c, 2, q_c)
    torch.cuda.synchronize()
    db_h = db_c.cpu().numpy().view(np.uint64)
    q_h = q_c.cpu().numpy().view(np.uint64)
    # a1 / a2: the oracle's encryption of the product's integer plaintexts == the device ciphertexts
    enc_ok = True
    for k, t in enumerate(sets):
        pt = B.bm_encode_db(prm, T_local, t - W.lo, 1).reshape(p, N_RING)
        enc_ok &= bool(np.array_equal(O.encrypt(logN, opk, pt, t * p, 2).reshape(p, 2, 2, -1), db_h[k]))
    for k, j in enumerate(qs):
        pt = B.bm_encode_query(prm, Q[j:j + 1]).reshape(p, N_RING)
        enc_ok &= bool(np.array_equal(O.encrypt(logN, opk, pt, j * p, 3).reshape(p, 2, 2, -1), q_h[k]))
    local = np.array([(qi[j], si[t]) for j, t in sample], np.int64)
    ref, _ = O.match(logN, d, p, order, orlk, ogk, db_h, q_h, pairs=local, n_threads=os.cpu_count() or 1)
    ref = ref.reshape(-1, 2, N_RING)
    bad = [k for k, jt in enumerate(sample) if not np.array_equal(got[jt], ref[k])]
    res.update({"parity": "bit-exact" if not bad and enc_ok else "MISMATCH",
                "oracle_pairs": len(sample), "oracle_pairs_mismatched": len(bad),
                "encrypt_parity": enc_ok,
                "oracle_pairs_spread": f"{len(qs)} queries x {len(sets)} sets incl. (0, first), (last, last), every "
                                       f"query group ({W.G}), the last set"})
    if world > 1 and gat is not None:
        res["gather_parity"] = gather_check(B, torch, prm, pk, evk_dev, d_db, d_q, W, gat, ws, order, world, rank, dev)
    res["verify_s"] = round(time.perf_counter() - t0, 1)
    ok = (res["parity"] == "bit-exact" and res["max_abs_score_err"] <= 1e-4
          and (res["top1_agree_genuine"] in (None, 1.0)))
    res["ok"] = bool(ok)
    return res


def gather_check(B, torch, prm, pk, evk_dev, d_db, d_q, W, gat, ws, order, world, rank, dev):
    """N > 1: group 0's scan with the fused gather (peers store into the roots' rows); each root then
    encrypts 2 sets owned by other ranks itself (global object numbers: identical ciphertexts),
    scans them for its rows' queries and compares bit for bit with what the peers stored."""
    import torch.distributed as dist
    from paper_2408_06167_b200 import dist as pdist
    from paper_2408_06167_b200 import inputs as I
    B.bm_match_rows(prm, evk_dev, d_db, W.n_local, d_q[:W.gq], W.gq, gat.rows_of(0), W.lo, ws[0], order)
    torch.cuda.synchronize()
    dist.barrier()
    rmap = pdist.p2p_row_map(W.nq, W.G, world, gat.ring)
    mine = [(j, row) for j, (root, row) in enumerate(rmap[:W.gq]) if root == rank]
    foreign = []
    for src in range(world):
        lo, cnt = pdist.shard_sets(W.n_sets, world, src)
        if src != rank and cnt and len(foreign) < 2:
            foreign.append(lo + cnt - 1)
    pk_dev = B.bm_pk_to_device(prm, pk)
    n_ok = n_all = 0
    js = [j for j, _ in mine]
    for t in foreign:
        T = I.templates(W.cfg, min(W.B, W.n - t * W.B), t * W.B)
        db1 = torch.empty((1, W.p, 2, 2, N_RING), dtype=torch.int64, device=dev)
        encrypt_set(B, prm, pk_dev, T, t, db1)
        qq = torch.stack([d_q[j] for j in js]).contiguous()
        out = torch.empty((len(js), 1, 2, N_RING), dtype=torch.int64, device=dev)
        wsl = torch.empty(B.bm_match_ws_bytes(prm, 1, len(js), order), dtype=torch.uint8, device=dev)
        B.bm_match(prm, evk_dev, db1, 1, qq, len(js), out, wsl, order)
        torch.cuda.synchronize()
        for k, (j, row) in enumerate(mine):
            n_all += 1
            n_ok += int(torch.equal(gat.res[row, t], out[k, 0]))
    return {"pairs_checked": n_all, "pairs_equal": n_ok, "ok": n_all > 0 and n_ok == n_all}


def encrypt_set(B, prm, pk_dev, T, t, out):
    """encrypt global set t alone (object numbers t p + i, seed 2), as its owner did"""
    import torch
    pt = torch.from_numpy(B.bm_encode_db(prm, T, 0, 1).reshape(-1, N_RING)).to(out.device)
    B.bm_encrypt(prm, pk_dev, pt, t * prm.p, 2, out)
    B.bm_sync()


def run_single(B, torch, prm, evk_dev, d_db, n_sets, n_tmpl, d_q, ring, ws, order, stream):
    """Latency of ONE query against the whole (local) DB (the paper's measurement shape,
    PAPER.md:572-574: 6,144 templates at d = 128 in 0.45 s on 6 CPU cores): bm_match of query 0
    over all sets, CUDA events on the launching stream, 3 warm-ups then 10 timed runs."""
    q1 = d_q[:1]
    o1 = ring[0][:1] if ring is not None else torch.empty((1, n_sets, 2, N_RING), dtype=torch.int64,
                                                          device=d_q.device)
    for _ in range(3):
        B.bm_match(prm, evk_dev, d_db, n_sets, q1, 1, o1, ws, order)
    torch.cuda.synchronize()
    times = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        B.bm_match(prm, evk_dev, d_db, n_sets, q1, 1, o1, ws, order)
        b.record(stream)
        b.synchronize()
        times.append(a.elapsed_time(b))
    ms = statistics.mean(times)
    graph = None
    try:
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg):
            B.bm_match(prm, evk_dev, d_db, n_sets, q1, 1, o1, ws, order)
        cg.replay()
        torch.cuda.synchronize()
        gt = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            cg.replay()
            b.record()
            b.synchronize()
            gt.append(a.elapsed_time(b))
        graph = {"ms": round(statistics.mean(gt), 4), "ms_std": round(statistics.pstdev(gt), 4), "runs": len(gt)}
    except Exception as ex:  # noqa: BLE001 -- reported, the eager number stands
        graph = {"error": f"{type(ex).__name__}: {ex}"[:160]}
    return {"ms": round(ms, 4), "ms_std": round(statistics.pstdev(times), 4), "runs": len(times), "cuda_graph": graph,
            "templates": n_tmpl, "templates_per_s": round(n_tmpl / (ms / 1e3), 1),
            "note": f"one query vs the whole local DB ({n_sets} (query, set) pairs), device time of bm_match, each "
                    f"run launched alone (launch latency included)"}


def run_e2e(args, B, torch, prm, evk_dev, d_db, n_local, d_q, W, order, dev, world, tq_per_step):
    """The same scan end to end through the C ABI from HOST buffers: bm_match_host_ring (pinned query
    upload and result download inside the call, results streamed through a bounded pinned host ring)."""
    import torch.distributed as dist
    from paper_2408_06167_b200 import dist as pdist
    nq, p = W.nq, W.p
    if world > 1:
        pdist.broadcast_queries(d_q)
    h_q = torch.empty((nq, p, 2, 2, N_RING), dtype=torch.int64).pin_memory()
    h_q.copy_(d_q)
    row_bytes = n_local * 2 * N_RING * 8
    ring_rows = int(max(1, min(nq, (args.ring_gib * 2**30) // max(1, row_bytes))))
    h_ring = torch.empty((ring_rows, n_local, 2, N_RING), dtype=torch.int64).pin_memory()
    torch.cuda.empty_cache()
    ws2 = torch.empty(B.bm_match_host_ws_bytes(prm, n_local, nq, order), dtype=torch.uint8, device=dev)
    B.bm_match_host_ring(prm, evk_dev, d_db, n_local, h_q, nq, h_ring, ring_rows, ws2, order)
    k2 = max(1, min(args.steps, 3))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k2):
        B.bm_match_host_ring(prm, evk_dev, d_db, n_local, h_q, nq, h_ring, ring_rows, ws2, order)
    torch.cuda.synchronize()
    e2e_ms = pdist.max_over_ranks((time.perf_counter() - t0) * 1e3 / k2, dev)
    # the last query's row (ring row (nq - 1) mod ring_rows) == a device scan of that query
    chk = torch.empty((1, n_local, 2, N_RING), dtype=torch.int64, device=dev)
    del ws2
    wsc = torch.empty(B.bm_match_ws_bytes(prm, n_local, 1, order), dtype=torch.uint8, device=dev)
    B.bm_match(prm, evk_dev, d_db, n_local, d_q[nq - 1:], 1, chk, wsc, order)
    B.bm_sync()
    same = bool(torch.equal(h_ring[(nq - 1) % ring_rows], chk[0].cpu()))
    return {"value": round(tq_per_step / (e2e_ms / 1e3), 1), "unit": "templates*queries/s",
            "h2d_bytes_per_step": int(h_q.numel() * 8), "d2h_bytes_per_step": int(nq * row_bytes),
            "ms_per_step": round(e2e_ms, 3), "host_ring_rows": ring_rows, "last_row_equals_device_scan": same,
            "note": "bm_match_host_ring per rank (its shard): pinned query cts H2D + every result D2H through a "
                    "bounded pinned host ring, inside the timed region, wall clock, max over ranks"}


# ----------------------------------------------------------------------------- NEXT-row legs (configs[1])
def run_extras(args, B, torch, dev, stream):
    """f3 (+ f4) and f1 measured on the configs[1] workload (d = 128, 6,144 templates, 384 queries,
    p = 8), their own setup; the plain scan of that workload is timed as their reference."""
    from paper_2408_06167_b200 import inputs as I
    cfg, p, nq = 2, 8, 384
    prm = B.bm_params_init(128, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    pk_dev, evk_dev = B.bm_pk_to_device(prm, pk), B.bm_evk_to_device(prm, evk)
    n_tmpl = I.CONFIGS[cfg]["n"]
    n_sets = -(-n_tmpl // prm.B)
    T = I.templates(cfg, n_tmpl)
    d_db = torch.empty((n_sets, p, 2, 2, N_RING), dtype=torch.int64, device=dev)
    B.bm_encrypt_db(prm, pk_dev, T, 0, n_sets, 2, d_db)
    Q, _ = I.queries(cfg, nq)
    d_q = torch.empty((nq, p, 2, 2, N_RING), dtype=torch.int64, device=dev)
    B.bm_encrypt_query(prm, pk_dev, Q, 0, 3, d_q)
    d_out = torch.empty((nq, n_sets, 2, N_RING), dtype=torch.int64, device=dev)
    ws = torch.empty(B.bm_match_ws_bytes(prm, n_sets, nq, 0), dtype=torch.uint8, device=dev)
    for _ in range(2):
        B.bm_match(prm, evk_dev, d_db, n_sets, d_q, nq, d_out, ws, 0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    k = max(1, min(args.steps, 5))
    for _ in range(k):
        B.bm_match(prm, evk_dev, d_db, n_sets, d_q, nq, d_out, ws, 0)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_scan = e0.elapsed_time(e1) / k
    tq = n_tmpl * nq
    del ws
    torch.cuda.empty_cache()
    out = {"configs1_scan": {"ms_per_step": round(ms_scan, 4), "value": round(tq / (ms_scan / 1e3), 1),
                             "unit": "templates*queries/s",
                             "note": "BASELINE configs[1] (6,144 templates x 384 queries, p = 8), one bm_match, "
                                     "device time: the reference point of the NEXT-row legs"}}
    try:
        out["f3_expand"] = run_f3(args, B, torch, prm, pk, sk, evk_dev, d_db, n_sets, d_q, d_out, ms_scan, tq, stream)
    except Exception as ex:  # noqa: BLE001
        out["f3_expand"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    torch.cuda.empty_cache()
    try:
        out["f1_compressed"] = run_f1(args, B, torch, prm, pk, sk, d_out, n_sets, n_tmpl, tq, stream)
    except Exception as ex:  # noqa: BLE001
        out["f1_compressed"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    del d_db, d_q, d_out
    torch.cuda.empty_cache()
    try:
        out["f2_degree2"] = run_f2_deg2(args, B, torch, dev, stream)
    except Exception as ex:  # noqa: BLE001
        out["f2_degree2"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    return out


def run_f2_deg2(args, B, torch, dev, stream):
    """f2 relin-free degree-2 output (BM_ORDER_DEG2) against the relinearised scan of the SAME
    workload: configs[1]'s 6,144 templates at p = d = 128 (s = 1: no ladder either way), 96 queries.
    Device time of one bm_match per order; the degree-2 results are 1.5x the bytes and decrypt with
    s^2 (client cost); scores of 2 queries checked against float64 cosines."""
    from paper_2408_06167_b200 import inputs as I
    d = p = 128
    nq = 96
    prm = B.bm_params_init(d, p)
    sk, pk, evk = B.bm_keygen(prm, 1)
    pk_dev, evk_dev = B.bm_pk_to_device(prm, pk), B.bm_evk_to_device(prm, evk)
    n_tmpl = I.CONFIGS[2]["n"]
    n_sets = -(-n_tmpl // prm.B)
    T = I.templates(2, n_tmpl)
    Q, _ = I.queries(2, nq)
    d_db = torch.empty((n_sets, p, 2, 2, N_RING), dtype=torch.int64, device=dev)
    B.bm_encrypt_db(prm, pk_dev, T, 0, n_sets, 2, d_db)
    d_q = torch.empty((nq, p, 2, 2, N_RING), dtype=torch.int64, device=dev)
    B.bm_encrypt_query(prm, pk_dev, Q, 0, 3, d_q)
    res = {}
    k = max(1, min(args.steps, 5))
    for order, name in ((0, "relinearised"), (B.ORDER_DEG2, "degree2")):
        out = torch.empty((nq, n_sets, B.n_components(order), N_RING), dtype=torch.int64, device=dev)
        ws = torch.empty(B.bm_match_ws_bytes(prm, n_sets, nq, order), dtype=torch.uint8, device=dev)
        ek = None if order == B.ORDER_DEG2 else evk_dev
        for _ in range(2):
            B.bm_match(prm, ek, d_db, n_sets, d_q, nq, out, ws, order)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            B.bm_match(prm, ek, d_db, n_sets, d_q, nq, out, ws, order)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        h = out[:2].cpu().numpy().view(np.uint64)
        t0 = time.perf_counter()
        sc = (B.bm_decrypt_deg2 if order == B.ORDER_DEG2 else B.bm_decrypt)(prm, sk, h.reshape(2 * n_sets, -1))
        dec_ms = (time.perf_counter() - t0) * 1e3 / (2 * n_sets)
        err = float(np.abs(sc.reshape(2, -1)[:, :n_tmpl] - Q[:2] @ T.T).max())
        res[name] = {"ms_per_step": round(ms, 4), "value": round(n_tmpl * nq / (ms / 1e3), 1),
                     "unit": "templates*queries/s", "result_bytes_per_pair": int(B.n_components(order) * N_RING * 8),
                     "client_decrypt_ms_per_result": round(dec_ms, 3), "max_abs_score_err_2q": err}
        del out, ws
        torch.cuda.empty_cache()
    res["speedup_device"] = round(res["relinearised"]["ms_per_step"] / res["degree2"]["ms_per_step"], 3)
    res["note"] = ("configs[1] templates at p = d = 128, 96 queries: relin-free degree-2 output vs the "
                   "relinearised scan (both s = 1, no ladder); device time of one bm_match")
    return res


def f3_modmuls(p, s):
    """Algorithmic modmuls of Algorithm 1 per expanded part (one (query, part) output): Mul(P) + Res
    (2 comps x (INTT_q2, NTT_q0, NTT_q1) + 3 mask products + 2 q2^-1 folds per coefficient) and
    log2(p) level-1 rotations (digits: 2 INTT + 4 ModUp NTT; per comp INTT_P + NTT_q0 + NTT_q1,
    6 key products + 2 P^-1 folds per coefficient)."""
    n = N_RING
    log_p = p.bit_length() - 1
    return 2 * (3 * BFLY + 5 * n) + log_p * (12 * BFLY + 16 * n)


def run_f3(args, B, torch, prm, pk, sk, evk_dev, d_db, n_sets, d_q, d_out, ms_scan, tq_per_step, stream):
    from paper_2408_06167_b200 import inputs as I
    p, nq = prm.p, d_q.shape[0]
    dev = d_q.device
    xk = B.bm_xk_keygen(prm, 1)
    xk_dev = B.bm_xk_to_device(prm, pk, xk)
    Q, _ = I.queries(2, nq)
    d_pt = torch.from_numpy(B.bm_encode_query_tiled(prm, Q)).to(dev)
    d_l2 = torch.empty((nq, 2, 3, N_RING), dtype=torch.int64, device=dev)
    B.bm_encrypt_l2(prm, xk_dev, d_pt, 0, 3, d_l2)
    del d_pt
    d_qx = torch.empty_like(d_q)
    ws = torch.empty(B.bm_expand_ws_bytes(prm, nq), dtype=torch.uint8, device=dev)
    for _ in range(max(2, args.warmup)):
        B.bm_expand(prm, xk_dev, d_l2, nq, d_qx, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    k = max(1, min(args.steps, 5))
    for _ in range(k):
        B.bm_expand(prm, xk_dev, d_l2, nq, d_qx, ws)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    del ws
    # sanity: the expanded queries scan to the same scores as the client-expanded ones (different noise)
    kq = min(4, nq)
    out_x = torch.empty((kq, n_sets, 2, N_RING), dtype=torch.int64, device=dev)
    ws2 = torch.empty(B.bm_match_ws_bytes(prm, n_sets, kq, 0), dtype=torch.uint8, device=dev)
    B.bm_match(prm, evk_dev, d_db, n_sets, d_qx[:kq].contiguous(), kq, out_x, ws2, 0)
    B.bm_sync()
    sa = B.bm_decrypt(prm, sk, out_x.cpu().numpy().view(np.uint64).reshape(-1, 2, 1, N_RING))
    sb = B.bm_decrypt(prm, sk, d_out[:kq].cpu().numpy().view(np.uint64).reshape(-1, 2, 1, N_RING))
    err = float(np.abs(sa - sb).max())
    assert err < 1e-5, err
    f4 = None
    try:
        f4 = run_f4(B, torch, prm, xk_dev, sk, evk_dev, d_db, n_sets, d_q, out_x, ws2, sb, kq, stream)
    except Exception as ex:  # noqa: BLE001
        f4 = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    mm = f3_modmuls(p, prm.s) * nq * p
    peak = int_peak_gmodmul(torch.cuda.get_device_properties(dev).multi_processor_count, 1965.0e6)
    return {"queries": nq, "ms_per_batch": round(ms, 4), "queries_per_s": round(nq / (ms / 1e3), 1),
            "gmodmul_s": round(mm / (ms / 1e3) / 1e9, 2), "alu_frac": round(mm / (ms / 1e3) / 1e9 / peak, 4),
            "kernel_launches": 1 + 2 * (p.bit_length() - 1),
            "upload_bytes_per_query": {"client_expanded": p * 4 * N_RING * 8, "server_expanded": 6 * N_RING * 8},
            "expand_plus_scan": {"ms_per_step": round(ms + ms_scan, 4),
                                 "value": round(tq_per_step / ((ms + ms_scan) / 1e3), 1),
                                 "unit": "templates*queries/s"},
            "score_check_max_abs_diff": err,
            "note": "Algorithm 1 on the chain extended by q2 (not BASELINE's parameter set; DESIGN.md R24), "
                    "configs[1] batch",
            "f4_enroll": f4}


def run_f4(B, torch, prm, xk_dev, sk, evk_dev, d_db, n_sets, d_q, out_x, ws2, sb, k, stream):
    """f4: server-side enrollment of the whole configs[1] DB (the same templates), then the same spot check."""
    from paper_2408_06167_b200 import inputs as I
    dev = d_db.device
    T = I.templates(2, I.CONFIGS[2]["n"], 0)
    n_t = T.shape[0]
    d_pt = torch.from_numpy(B.bm_encode_enroll(prm, T)).to(dev)
    d_tl2 = torch.empty((n_t, 2, 3, N_RING), dtype=torch.int64, device=dev)
    B.bm_encrypt_l2(prm, xk_dev, d_pt, 0, 5, d_tl2)
    del d_pt
    d_db2 = torch.zeros_like(d_db)
    ws3 = torch.empty(B.bm_enroll_ws_bytes(prm, n_t), dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    B.bm_enroll(prm, xk_dev, d_tl2, 0, d_db2, ws3)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_enroll = e0.elapsed_time(e1)
    del ws3, d_tl2
    B.bm_match(prm, evk_dev, d_db2, n_sets, d_q[:k].contiguous(), k, out_x, ws2, 0)
    B.bm_sync()
    sc = B.bm_decrypt(prm, sk, out_x.cpu().numpy().view(np.uint64).reshape(-1, 2, 1, N_RING))
    err4 = float(np.abs(sc - sb).max())
    assert err4 < 1e-4, err4
    return {"templates": n_t, "ms": round(ms_enroll, 3), "templates_per_s": round(n_t / (ms_enroll / 1e3), 1),
            "score_check_max_abs_diff": err4,
            "note": "server-side enrollment (Fig. 3) of the configs[1] DB, one template ciphertext at a time "
                    "semantics, all templates in one bm_enroll call; scores vs the client-packed DB"}


def run_f1(args, B, torch, prm, pk, sk, d_out, n_sets, n_tmpl, tq_per_step, stream):
    from paper_2408_06167_b200 import inputs as I
    dev = d_out.device
    nq, p, s = d_out.shape[0], prm.p, prm.s
    xk = B.bm_xk_keygen(prm, 1)
    xk_dev = B.bm_xk_to_device(prm, pk, xk, enroll=False)       # the level-2 public key
    ck_dev = B.bm_ck_to_device(prm, B.bm_ck_keygen(prm, 1))
    T = I.templates(2, n_tmpl, 0)
    Q, _ = I.queries(2, nq)
    d_db = torch.empty((n_sets, p, 2, 3, N_RING), dtype=torch.int64, device=dev)
    B.bm_encrypt_l2(prm, xk_dev, torch.from_numpy(B.bm_encode_db(prm, T, 0, n_sets).reshape(-1, N_RING)).to(dev),
                    0, 2, d_db)
    d_q = torch.empty((nq, p, 2, 3, N_RING), dtype=torch.int64, device=dev)
    B.bm_encrypt_l2(prm, xk_dev, torch.from_numpy(B.bm_encode_query(prm, Q).reshape(-1, N_RING)).to(dev), 0, 3, d_q)
    G = -(-n_sets // s)
    out = torch.empty((nq, G, 2, N_RING), dtype=torch.int64, device=dev)
    ws = torch.empty(B.bm_match_cmp_ws_bytes(prm, n_sets, nq), dtype=torch.uint8, device=dev)
    B.bm_match_cmp(prm, ck_dev, d_db, n_sets, d_q, nq, out, ws)     # warm-up
    torch.cuda.synchronize()
    k = max(1, min(args.steps, 3))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        B.bm_match_cmp(prm, ck_dev, d_db, n_sets, d_q, nq, out, ws)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    slots = B.bm_decrypt_packed(prm, sk, out[:2].cpu().numpy().view(np.uint64).reshape(-1, 2, 1, N_RING))
    ref = B.bm_decrypt(prm, sk, d_out[:2].cpu().numpy().view(np.uint64).reshape(-1, 2, 1, N_RING))
    ref = ref.reshape(2, n_sets, prm.B)
    err = 0.0
    for j in range(2):
        for t in range(n_sets):
            g, u = divmod(t, s)
            err = max(err, float(np.abs(slots[j * G + g, u::s] - ref[j, t]).max()))
    assert err < 1e-5, err
    return {"ms_per_step": round(ms, 3), "value": round(tq_per_step / (ms / 1e3), 1), "unit": "templates*queries/s",
            "packed_ciphertexts_per_query": G, "d2h_bytes_per_step": int(out.numel() * 8),
            "d2h_bytes_uncompressed": int(d_out.numel() * 8), "score_check_max_abs_diff": err,
            "note": "configs[1] workload: HE-C^3 one level up (level-2 DB and query parts: tensor over 3 limbs, "
                    "3-digit relin + Res q2, ladder at level 1) + compression (Res_q1(M * C_t), right rotation by "
                    "t mod s, packing); chain extended by q2, DESIGN.md R28"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2408_06167_b200 import inputs as I
    c = I.CONFIGS[args.config]
    d, p = c["d"], args.p or c["p"]
    nth = os.cpu_count() or 1
    run, n_pairs, Bk, t1 = oracle_sample(args.config, d, p, 8.0, nth)
    for _ in range(args.warmup):
        run()
    times = [run() for _ in range(args.steps)]
    secs = sum(times) / len(times)
    value = n_pairs * Bk / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 2),
        "unit": "templates*queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs * 1e3, 2), "higher_is_better": True,
        "scaling": "strong" if world > 1 and args.config in (4, 5) else "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"BASELINE configs[{args.config - 1}]: d={d}, p={p}, bounded sample of {n_pairs} "
                               f"(query, set) pairs per step (the CPU oracle, oracle/)", "d": d, "p": p},
        "cpu_baseline": {"value": round(value, 2), "unit": "templates*queries/s", "cores": nth, "kind": "oracle",
                         "sample": f"{n_pairs} pairs x {Bk} templates per step on {nth} threads"},
        "e2e": {"value": round(value, 2), "unit": "templates*queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if os.environ.get("BM_BENCH_WATCHDOG"):   # debugging aid: dump every thread's stack and exit after N s
        import faulthandler
        faulthandler.dump_traceback_later(float(os.environ["BM_BENCH_WATCHDOG"]), exit=True)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
