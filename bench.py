#!/usr/bin/env python
"""Benchmark of the encrypted 1:N cosine scan (HE-C^3) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--p P] [--order 0|1]

Workload (N = 1): BASELINE.json configs[1] -- d = 128, 6,144 unit-norm Gaussian templates
(stand-ins for the paper's IJB-C ArcFace embeddings), 384 genuine queries
(1 per 16 templates), p = 8 parts (best of the configs[1] sweep), CKKS N = 8192.
One step = the whole hot path for the whole query batch: bm_match of 384 queries x 24 sets
(tensor + part sum, relinearise, rescale, 4 rotate-and-add steps, coefficient-domain output);
for N > 1 also the query broadcast and the result gather (NCCL).  N > 1 is weak scaling: every
rank holds its own 6,144-template shard (global DB = 6,144 N templates).
Metric: encrypted templates matched per second = templates x queries / s (BASELINE.json).

--impl reference runs the CPU oracle (oracle/, plain C) on the host cores on a bounded sample of
the same workload (this tier has no reference implementation).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG = 2
D = 128
N_RING = 8192
BFLY = (N_RING // 2) * 13          # butterflies (= modmuls) per 8192-point transform
SM_COUNT = 148
IMAD_PER_CLK_SM = 64               # FMA pipe, 16 lanes/clk/SMSP (B300_MICROARCH.md "Pipe rates")
# FMA-pipe issue slots (in IMAD units) of the cheapest 64-bit Shoup modmul a w mod q: 4 IMAD (low
# words) + 3 IMAD.WIDE + 2 IMAD.HI, the wide / high forms at half the IMAD rate (measured 25-29 vs
# 63 lanes/clk/SM, tools/pipe_bench.cu, profiles/r01_pipe_bench.txt): 4 + 2 x 5 = 14
IMAD_SLOTS_PER_MODMUL = 14


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=8)
    ap.add_argument("--order", type=int, default=0)
    ap.add_argument("--no-f3", action="store_true", help="skip the f3 query-expansion / f4 enrollment leg")
    ap.add_argument("--no-f1", action="store_true", help="skip the f1 compressed-scan leg")
    ap.add_argument("--no-single", action="store_true", help="skip the single-query latency leg")
    ap.add_argument("--no-f4", action="store_true", help="skip the f4 enrollment part of the f3 leg")
    ap.add_argument("--nq", type=int, default=384)
    ap.add_argument("--groups", type=int, default=4, help="query groups overlapping comms and scans (N > 1)")
    ap.add_argument("--gather", choices=["p2p", "nccl"], default="p2p",
                    help="N > 1 result gather (a8): p2p = fused into the output kernels (bm_match_rows storing "
                         "to the roots over NVLink), nccl = all_to_all after each group's scan")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--quiet", action="store_true")
    return ap.parse_args()


def log(args, *a):
    if not args.quiet:
        print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- algorithmic work
def class_modmuls(p, log_s):
    """Algorithmic 64-bit modular multiplications per (query, set) pair, per kernel class
    (DESIGN.md "Algorithmic work"): butterflies of every transform + pointwise products."""
    n = N_RING
    return {
        "tensor": 8 * n * p,                                       # a0b0, a1b1, (a0+a1)(b0+b1) per limb (+ adds)
        "digits": 6 * BFLY + n,                                    # INTT_q0, INTT_q1, NTT_q1, NTT_P x2, NTT_q0
        "relin": 6 * BFLY + 12 * n + 8 * n,                        # INTT_P, INTT_q1, NTT_q0 x 2 comps; rlk + scalings
        "ladder": (6 * BFLY + 6 * n) * log_s,                      # digit INTT_q0 + NTT_P, 2 x (INTT_P + NTT_q0)
        "hrot": (6 * BFLY + 4 * n * ((1 << log_s) - 1)) if log_s else 0,  # f2: 6 transforms + 4 products per rotation
        "out_intt": 0 if log_s else 2 * BFLY,
    }


def hbm_bytes_per_step(p, n_sets, nq):
    """Algorithmic HBM bytes of one step: DB read once, queries read once, results written once."""
    return n_sets * p * 4 * N_RING * 8 + nq * p * 4 * N_RING * 8 + nq * n_sets * 2 * N_RING * 8


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons DURING the timed region: NVML polled every 5 ms
    from a thread (the timed region of a default run is ~0.15 s, shorter than one `nvidia-smi -lms`
    start-up), falling back to `nvidia-smi -lms 100` where NVML is unavailable."""
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


# ----------------------------------------------------------------------------- oracle (cpu_baseline / reference)
def oracle_sample(p, seconds_target, n_threads, log=None):
    """Time the CPU oracle on a bounded sample of (query, set) pairs of the bench workload."""
    from oracle import oracle as O
    from paper_2408_06167_b200 import inputs as I
    logN = 13
    S, s, B = O.layout(logN, D, p)
    sk, pk, rlk, gk = O.keygen(logN, 1, O.n_rot_for(D, p))
    T = I.templates(CFG, 2 * B)            # two full sets
    Q, _ = I.queries(CFG, 2)
    db = O.encrypt(logN, pk, O.encode(O.pack_db(T, logN, D, p, 0, 2).reshape(-1, S), logN), 0, 2).reshape(2, p, 2, 2, -1)
    qc = O.encrypt(logN, pk, O.encode(O.pack_query(Q, logN, D, p).reshape(-1, S), logN), 0, 3).reshape(2, p, 2, 2, -1)
    t0 = time.perf_counter()
    O.match(logN, D, p, 0, rlk, gk, db, qc, pairs=np.array([[0, 0]], np.int64), n_threads=1)
    t1 = time.perf_counter() - t0
    n_pairs = int(max(n_threads, min(4096, round(seconds_target * n_threads / max(t1, 1e-3)))))
    pairs = np.array([(k % 2, (k // 2) % 2) for k in range(n_pairs)], np.int64)

    def run():
        t = time.perf_counter()
        O.match(logN, D, p, 0, rlk, gk, db, qc, pairs=pairs, n_threads=n_threads)
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

    p, nq, order = args.p, args.nq, args.order
    prm = B.bm_params_init(D, p)
    n_tmpl = I.CONFIGS[CFG]["n"]                     # per rank (weak scaling)
    n_sets = -(-n_tmpl // prm.B)
    sk, pk, evk = B.bm_keygen(prm, 1)                # deterministic: identical keys on every rank
    if order == 2:                                   # f2 hoisted rotation sum: keys of every rotation
        B.bm_evk_add_hoisted(prm, 1, evk)
    pk_dev, evk_dev = B.bm_pk_to_device(prm, pk), B.bm_evk_to_device(prm, evk)
    T = I.templates(CFG, n_tmpl, rank * n_tmpl)
    d_db = torch.empty((n_sets, p, 2, 2, N_RING), dtype=torch.int64, device=dev)
    B.bm_encrypt_db(prm, pk_dev, T, 0, n_sets, 2 + rank, d_db)
    d_q = torch.empty((nq, p, 2, 2, N_RING), dtype=torch.int64, device=dev)
    if rank == 0:
        Q, _ = I.queries(CFG, nq)
        B.bm_encrypt_query(prm, pk_dev, Q, 0, 3, d_q)
    d_out = torch.empty((nq, n_sets, 2, N_RING), dtype=torch.int64, device=dev)
    # N > 1: broadcast (a3) and scan overlapped over query groups; the result gather (a8) either fused
    # into the scan's output kernels (p2p: every result stored straight into its root's buffer over
    # NVLink, dist.P2PGather) or an all_to_all after each group's scan (nccl)
    G = args.groups if world > 1 else 1
    gq = nq // G
    ws = torch.empty(B.bm_match_ws_bytes(prm, n_sets, gq, order), dtype=torch.uint8, device=dev)
    comm_s, comp_s = (torch.cuda.Stream(), torch.cuda.Stream()) if world > 1 else (None, None)
    gather, gat, recv, flag = "local", None, None, None
    if world > 1 and args.gather == "p2p":
        res = torch.empty((nq // world, n_sets * world, 2, N_RING), dtype=torch.int64, device=dev)
        try:
            gat = pdist.P2PGather(B, res, nq, G, n_sets * world)
            flag = torch.zeros(1, dtype=torch.float64, device=dev)
            gather = "p2p: fused into the output kernels (bm_match_rows, CUDA IPC peer stores over NVLink)"
        except Exception as ex:  # noqa: BLE001 -- a transport fallback (NCCL), never a CPU one
            del res
            gather = f"nccl all_to_all (p2p unavailable: {type(ex).__name__}: {ex})"[:200]
    if world > 1 and gat is None:
        recv = torch.empty((G, world, gq // world, n_sets, 2, N_RING), dtype=torch.int64, device=dev)
        if gather == "local":
            gather = "nccl all_to_all per query group"
    B.bm_sync()
    stream = torch.cuda.current_stream()

    def match(g, q_g, out_g):
        B.bm_match(prm, evk_dev, d_db, n_sets, q_g, q_g.shape[0], out_g, ws, order)

    def match_rows(g, q_g, rows_g):
        B.bm_match_rows(prm, evk_dev, d_db, n_sets, q_g, q_g.shape[0], rows_g, rank * n_sets, ws, order)

    def step():
        if world == 1:
            B.bm_match(prm, evk_dev, d_db, n_sets, d_q, nq, d_out, ws, order)
        elif gat is not None:
            pdist.scan_p2p(match_rows, d_q, gat, G, comm_s, comp_s, flag)
        else:
            pdist.scan_pipelined(match, d_q, d_out, recv, G, comm_s, comp_s)

    log(args, f"[rank {rank}] setup done: {n_sets} sets x {nq} queries, p={p}, ws={ws.numel() / 2**30:.2f} GiB")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # events at every step boundary (recorded on the launching stream, no synchronisation between
    # steps): the first and last bracket the timed region, the others give the per-step spread
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev[0].record(stream)
        for i in range(args.steps):
            step()
            ev[i + 1].record(stream)
        while not ev[-1].query():   # wait without holding the GIL, so the clock sampler thread runs
            time.sleep(0.0005)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = pdist.max_over_ranks(ev[0].elapsed_time(ev[-1]), dev)
    ms_step = ms / args.steps
    per_step = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    ms_std = float(statistics.pstdev(per_step)) if len(per_step) > 1 else 0.0
    tq_per_step = world * n_tmpl * nq
    value = tq_per_step / (ms_step / 1e3)

    # launches of our kernels per step: chunks x (3 per part-round + 1 fused ladder (or output INTT if s = 1))
    import math
    total_pairs = n_sets * nq
    chunk = int(os.environ.get("BM_CHUNK_PAIRS", "16384"))
    n_chunks = G * math.ceil(n_sets * gq / min(chunk, n_sets * gq))
    rounds = p if order == 1 else 1
    launches = n_chunks * (3 * rounds + 1)
    cp = min(chunk, n_sets * gq)                       # pairs per ladder launch
    tail = cp % SM_COUNT
    if prm.log_s > 0 and cp > SM_COUNT and 0 < 2 * tail <= SM_COUNT:
        launches += n_chunks                           # the partial last wave runs on the cluster ladder

    # per-kernel-class device times (CUDA events on the launching stream), same step, profiled pass
    B.bm_set_profiling(True)
    B.bm_profile_reset()
    for _ in range(args.steps):
        for g in range(G):
            B.bm_match(prm, evk_dev, d_db, n_sets, d_q[g * gq:(g + 1) * gq], gq, d_out[g * gq:(g + 1) * gq], ws, order)
    B.bm_sync()
    pms, pla, pun = B.bm_profile_read()
    B.bm_set_profiling(False)
    mm = class_modmuls(1 if order == 1 else p, prm.log_s)  # order 1 runs the part rounds one part each
    classes = B.PROFILE_CLASSES
    per_class = {}
    step_work = 0.0   # algorithmic modmuls of one step: the classes that ran
    for i, c in enumerate(classes):
        if pla[i]:
            work = mm[c] * total_pairs * args.steps * (rounds if i < 3 else 1)
            step_work += work / args.steps
            per_class[c] = {"ms_per_step": pms[i] / args.steps, "launches": int(pla[i]),
                            "gmodmul_s": work / (pms[i] / 1e3) / 1e9}
    dom = max(per_class, key=lambda c: per_class[c]["ms_per_step"])
    clocks = clk.summary()
    f_peak = (clocks["sm_max_mhz"] or 1965.0) * 1e6
    peak = SM_COUNT * IMAD_PER_CLK_SM * f_peak / IMAD_SLOTS_PER_MODMUL / 1e9  # Gmodmul/s
    ach = per_class[dom]["gmodmul_s"]
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        traffic = json.load(open(tfile)).get(dom)
    hbm_gbs = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.8
    hbm_achieved = hbm_bytes_per_step(p, n_sets, nq) / (ms_step / 1e3) / 1e9
    roofline = {"bound": "alu", "kernel": dom, "achieved": round(ach, 2), "peak": round(peak, 2),
                "unit": "Gmodmul/s", "frac": round(ach / peak, 4), "traffic": traffic,
                "peak_basis": f"{SM_COUNT} SMs x {IMAD_PER_CLK_SM} IMAD/clk x {f_peak / 1e6:.0f} MHz / "
                              f"{IMAD_SLOTS_PER_MODMUL} IMAD issue slots per 64-bit Shoup modmul "
                              f"(4 IMAD + 3 IMAD.WIDE + 2 IMAD.HI at half rate)",
                "step_gmodmul_s": round(step_work / (ms_step / 1e3) / 1e9, 2),
                "step_frac": round(step_work / (ms_step / 1e3) / 1e9 / peak, 4),
                "hbm": {"achieved_gbs": round(hbm_achieved, 2), "peak_gbs": hbm_gbs,
                        "frac": round(hbm_achieved / hbm_gbs, 5)},
                "per_class": {c: {k: round(v, 3) for k, v in d.items()} for c, d in per_class.items()}}

    if gat is not None:   # fused gather: this rank's own sets in the rows it roots equal its local scan
        torch.cuda.synchronize()
        for j, (root, row) in enumerate(pdist.p2p_row_map(nq, G, world)):
            if root == rank:
                assert torch.equal(gat.res[row, rank * n_sets:(rank + 1) * n_sets], d_out[j]), "p2p gather"

    # single-query latency (the paper's shape: ONE query against the whole DB,
    # PAPER.md:572-574): bm_match of query 0 over all sets, device time, 3 warm-ups + 10 timed runs
    single = None
    if world == 1 and not args.no_single:
        single = run_single(B, torch, prm, evk_dev, d_db, n_sets, n_tmpl, d_q, d_out, ws, order, stream)

    # e2e through the C ABI with host buffers (query H2D + result D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        h_q = torch.empty((nq, p, 2, 2, N_RING), dtype=torch.int64).pin_memory()
        if world > 1:
            pdist.broadcast_queries(d_q)
        h_q.copy_(d_q)
        h_out = torch.empty((nq, n_sets, 2, N_RING), dtype=torch.int64).pin_memory()
        del ws
        torch.cuda.empty_cache()
        ws2 = torch.empty(B.bm_match_host_ws_bytes(prm, n_sets, nq, order), dtype=torch.uint8, device=dev)
        B.bm_match_host(prm, evk_dev, d_db, n_sets, h_q, nq, h_out, ws2, order)
        k2 = max(1, args.steps)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k2):
            B.bm_match_host(prm, evk_dev, d_db, n_sets, h_q, nq, h_out, ws2, order)
        torch.cuda.synchronize()
        e2e_ms = pdist.max_over_ranks((time.perf_counter() - t0) * 1e3 / k2, dev)
        # correctness spot check of the e2e output against the device path
        assert torch.equal(h_out[0, 0], d_out[0, 0].cpu())
        e2e = {"value": round(tq_per_step / (e2e_ms / 1e3), 1), "unit": "templates*queries/s",
               "h2d_bytes_per_step": int(h_q.numel() * 8), "d2h_bytes_per_step": int(h_out.numel() * 8),
               "ms_per_step": round(e2e_ms, 3), "note": "per rank: query cts H2D + results D2H, wall clock"}

    # f3: server-side query expansion (Algorithm 1) of the same batch -- the client
    # uploads ONE level-2 ciphertext per query (the chain extended by q2) and bm_expand produces the p
    # level-1 parts bm_match takes.  Device time of the expansion alone and of expansion + scan.
    # (the NEXT-row legs never take the headline line down with them: a failure is recorded instead)
    f3 = None
    if world == 1 and not args.no_f3:
        try:
            f3 = run_f3(args, B, torch, prm, pk, sk, evk_dev, d_db, n_sets, d_q, d_out, ms_step, tq_per_step, stream)
        except Exception as ex:  # noqa: BLE001
            f3 = {"error": f"{type(ex).__name__}: {ex}"}
            log(args, f"[rank {rank}] f3/f4 leg failed: {f3['error']}")
    # f1: the compressed scan of the same workload one level up (level-2 DB and
    # queries), packed outputs s times smaller with the partial sums masked away
    f1 = None
    if world == 1 and not args.no_f1:
        ws = None   # the scan's workspace (already released when the e2e leg ran)
        torch.cuda.empty_cache()
        try:
            f1 = run_f1(args, B, torch, prm, pk, sk, d_out, n_sets, n_tmpl, tq_per_step, stream)
        except Exception as ex:  # noqa: BLE001
            f1 = {"error": f"{type(ex).__name__}: {ex}"}
            log(args, f"[rank {rank}] f1 leg failed: {f1['error']}")
        torch.cuda.empty_cache()

    # CPU oracle on the host cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nth = os.cpu_count() or 1
        run, n_pairs, Bk, t1 = oracle_sample(p, 12.0, nth)
        secs = run()
        cpu = {"value": round(n_pairs * Bk / secs, 2), "unit": "templates*queries/s", "cores": nth, "kind": "oracle",
               "sample": f"{n_pairs} (query, set) pairs of the bench workload (p={p}, {Bk} templates each), "
                         f"{nth} threads, {secs:.1f} s wall; single pair {t1:.2f} s on 1 thread"}

    if rank == 0:
        line = {
            "metric": "encrypted templates matched/sec (d=128, N=8192)", "value": round(value, 1),
            "unit": "templates*queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "ms_per_step_std": round(ms_std, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u64", "data": "synthetic (seeded unit-norm Gaussian templates, genuine noisy queries)",
            "config": {"workload": f"BASELINE configs[1]: d=128, {n_tmpl} templates/GPU, {nq} queries, p={p}, "
                                   f"order={['hoisted', 'paper', 'hoisted-rotations (f2, not the paper ladder)'][order]}",
                       "d": D, "p": p, "templates_per_gpu": n_tmpl, "sets_per_gpu": n_sets, "queries": nq,
                       "ring_N": N_RING, "parallelism": f"db-shard{world}", "gather": gather,
                       "l2": "inputs > L2: query cts %.0f MB + DB %.0f MB per step (126 MB L2), no flush" % (
                           nq * p * 4 * N_RING * 8 / 1e6, n_sets * p * 4 * N_RING * 8 / 1e6)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "single_query": single,
            "f3_expand": f3, "f1_compressed": f1,
            "gpu_launches": int(launches * args.steps),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if gat is not None:
        dist.barrier()
        gat.close()
    if world > 1:
        dist.destroy_process_group()


def run_single(B, torch, prm, evk_dev, d_db, n_sets, n_tmpl, d_q, d_out, ws, order, stream):
    """Latency of ONE query against the whole DB (the paper's measurement shape, PAPER.md:572-574:
    6,144 templates at d = 128 in 0.45 s on 6 CPU cores): bm_match of query 0 over all n_sets sets,
    CUDA events on the launching stream, 3 warm-ups then 10 timed runs (10 trials)."""
    q1, o1 = d_q[:1], d_out[:1]
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
    # the same call captured once in a CUDA graph and replayed alone (a server answering one query:
    # the four launches become one graph launch)
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
            "note": "one query vs the whole configs[1] DB: 24 (query, set) pairs, a latency-bound launch "
                    "(latency mode: small-batch tensor tiles, 3-CTA pipelined ladder), device time of bm_match, "
                    "each run launched alone (launch latency included)"}


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
    Q, _ = I.queries(CFG, nq)
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
    for _ in range(args.steps):
        B.bm_expand(prm, xk_dev, d_l2, nq, d_qx, ws)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    del ws
    # sanity: the expanded queries scan to the same scores as the client-expanded ones (different noise)
    k = min(4, nq)
    out_x = torch.empty((k, n_sets, 2, N_RING), dtype=torch.int64, device=dev)
    ws2 = torch.empty(B.bm_match_ws_bytes(prm, n_sets, k, 0), dtype=torch.uint8, device=dev)
    B.bm_match(prm, evk_dev, d_db, n_sets, d_qx[:k].contiguous(), k, out_x, ws2, 0)
    B.bm_sync()
    sa = B.bm_decrypt(prm, sk, out_x.cpu().numpy().view(np.uint64).reshape(-1, 2, 1, N_RING))
    sb = B.bm_decrypt(prm, sk, d_out[:k].cpu().numpy().view(np.uint64).reshape(-1, 2, 1, N_RING))
    err = float(np.abs(sa - sb).max())
    assert err < 1e-5, err
    f4 = None
    if not args.no_f4:
        f4 = run_f4(B, torch, prm, xk_dev, sk, evk_dev, d_db, n_sets, d_q, out_x, ws2, sb, k, stream)
    mm = f3_modmuls(p, prm.s) * nq * p
    peak = SM_COUNT * IMAD_PER_CLK_SM * 1965.0e6 / IMAD_SLOTS_PER_MODMUL / 1e9
    return {"queries": nq, "ms_per_batch": round(ms, 4), "queries_per_s": round(nq / (ms / 1e3), 1),
            "gmodmul_s": round(mm / (ms / 1e3) / 1e9, 2), "alu_frac": round(mm / (ms / 1e3) / 1e9 / peak, 4),
            "kernel_launches": 1 + 2 * (p.bit_length() - 1),
            "upload_bytes_per_query": {"client_expanded": p * 4 * N_RING * 8, "server_expanded": 6 * N_RING * 8},
            "expand_plus_scan": {"ms_per_step": round(ms + ms_scan, 4),
                                 "value": round(tq_per_step / ((ms + ms_scan) / 1e3), 1),
                                 "unit": "templates*queries/s"},
            "score_check_max_abs_diff": err,
            "note": "Algorithm 1 on the chain extended by q2 (not BASELINE's parameter set; DESIGN.md R24)",
            "f4_enroll": f4}


def run_f4(B, torch, prm, xk_dev, sk, evk_dev, d_db, n_sets, d_q, out_x, ws2, sb, k, stream):
    """f4: server-side enrollment of the whole DB (the same templates), then the same spot check."""
    from paper_2408_06167_b200 import inputs as I
    dev = d_db.device
    T = I.templates(CFG, I.CONFIGS[CFG]["n"], 0)
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
    T = I.templates(CFG, n_tmpl, 0)
    Q, _ = I.queries(CFG, nq)
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
    # the packed scores of two queries vs the uncompressed scan's
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
            "note": "HE-C^3 one level up (level-2 DB and query parts: tensor over 3 limbs, 3-digit relin + Res q2, "
                    "ladder at level 1) + compression (Res_q1(M * C_t), right rotation by t mod s, packing); "
                    "chain extended by q2, DESIGN.md R28"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nth = os.cpu_count() or 1
    p = args.p
    run, n_pairs, Bk, t1 = oracle_sample(p, 8.0, nth)
    for _ in range(args.warmup):
        run()
    times = [run() for _ in range(args.steps)]
    secs = sum(times) / len(times)
    value = n_pairs * Bk / secs
    line = {
        "impl": "reference", "metric": "encrypted templates matched/sec (d=128, N=8192)", "value": round(value, 2),
        "unit": "templates*queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs * 1e3, 2), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"BASELINE configs[1]: d=128, p={p}, bounded sample of {n_pairs} (query, set) pairs "
                               f"per step", "d": D, "p": p},
        "cpu_baseline": {"value": round(value, 2), "unit": "templates*queries/s", "cores": nth, "kind": "oracle",
                         "sample": f"{n_pairs} pairs x {Bk} templates per step on {nth} threads"},
        "e2e": {"value": round(value, 2), "unit": "templates*queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
