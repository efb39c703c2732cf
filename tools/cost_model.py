"""GPU-calibrated version of the paper's cost model (Propositions 2-4, Table 1,
F(N_in)) for the depth-1 pipeline built here (the cost-model half).

The paper prices HE-C^3 for R templates as ceil(m'/N_in) sets x (N_in (Mul(C) + Res + Add) +
(log m' - log N_in)(Rot + Add)), with per-op CPU times (Table 1).  Here the ops are fused kernels,
so the per-op costs are calibrated from bench.py's per-kernel-class CUDA-event times at
configs[1] (d = 128, 6,144 templates, 384 queries) for every p:
    t_tensor  = tensor class / (pairs x p)          one part of Mul(C)'s tensor product
    t_relin   = (digits + relin) / pairs            relinearize + rescale (hoisted: once per pair)
    t_rot     = ladder / (pairs x log2 s)           one Rot + Add step of the ladder
and the model  T(p) = sets(p) x nq x (p t_tensor + t_relin + log2(s) t_rot)  is compared with the
measured step time; p* = argmin T(p).

With f3 built, the paper's actual trade-off (Propositions 1-2: "As N_in increases,
the direct computation time for cosine similarity decreases. However, the time to generate N_in
ciphertexts increases") is measured too: bench.py's f3 leg times the server-side expansion of the
same 384 queries, calibrated as  T_exp(p) = nq x p x (t_xmask + log2(p) t_xrot)  (one Mul(P) + Res per
part, log2 p level-1 Rot + Add per part; least squares over the sweep), and the recognition-path
optimum is argmin T(p) + T_exp(p) for this database size.

    python tools/cost_model.py [--ps 1,2,4,8,16,32,64,128] [--out profiles/r01_cost_model.txt]
(runs bench.py on the GPU for each p)."""
import argparse
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(p):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--p", str(p), "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline", "--no-e2e", "--no-f1", "--no-f4", "--quiet"]
    out = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout.strip().splitlines()[-1]
    return json.loads(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ps", default="1,2,4,8,16,32,64,128")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_cost_model.txt"))
    a = ap.parse_args()
    d, n_tmpl, nq, S = 128, 6144, 384, 4096
    rows = []
    for p in [int(x) for x in a.ps.split(",")]:
        r = run(p)
        pc = r["roofline"]["per_class"]
        s = d // p
        B = S * p // d
        sets = -(-n_tmpl // B)
        pairs = sets * nq
        ls = int(math.log2(s))
        t_tensor = pc["tensor"]["ms_per_step"] / (pairs * p)
        t_relin = (pc["digits"]["ms_per_step"] + pc["relin"]["ms_per_step"]) / pairs
        t_rot = pc["ladder"]["ms_per_step"] / (pairs * ls) if ls else None
        f3 = r.get("f3_expand") or {}
        rows.append(dict(p=p, s=s, B=B, sets=sets, pairs=pairs, log_s=ls, ms=r["ms_per_step"],
                         value=r["value"], t_tensor=t_tensor, t_relin=t_relin, t_rot=t_rot,
                         exp_ms=f3.get("ms_per_batch"),
                         classes={k: v["ms_per_step"] for k, v in pc.items()}))
    # calibrated op costs: medians over the sweep (they should be nearly p-independent)
    med = lambda xs: sorted(xs)[len(xs) // 2]
    T_tensor = med([r["t_tensor"] for r in rows])
    T_relin = med([r["t_relin"] for r in rows])
    T_rot = med([r["t_rot"] for r in rows if r["t_rot"] is not None])
    lines = ["# GPU-calibrated cost model of HE-C^3 (PAPER.md:380-434) on B200, configs[1] data (d=128, "
             f"{n_tmpl} templates, {nq} queries); per-op costs in microseconds of whole-GPU time per pair",
             f"# T_tensor (one part) = {T_tensor * 1e3:.4f} us, T_relin+rescale = {T_relin * 1e3:.4f} us, "
             f"T_rot+add = {T_rot * 1e3:.4f} us",
             "# paper, Table 1 (Lattigo, 1 CPU core-ish, level 1): Mul(C) 3130 us, Rot 2950 us, Res 600 us",
             f"{'p':>4} {'s':>4} {'B':>5} {'sets':>5} {'measured_ms':>12} {'model_ms':>9} {'tq_per_s':>12}  per-class ms"]
    best = None
    for r in rows:
        model = r["pairs"] * (r["p"] * T_tensor + T_relin + r["log_s"] * T_rot)
        lines.append(f"{r['p']:>4} {r['s']:>4} {r['B']:>5} {r['sets']:>5} {r['ms']:>12.3f} {model:>9.3f} "
                     f"{r['value']:>12.4g}  {r['classes']}")
        if best is None or model < best[1]:
            best = (r["p"], model)
    lines.append(f"# model optimum: p* = {best[0]} (paper, CPU, with expansion + compression: N_in = 4)")
    # f3: the expansion stage, T_exp(p) = nq p (t_xmask + log2(p) t_xrot), least squares
    ex = [r for r in rows if r["exp_ms"] is not None]
    if ex:
        import numpy as np
        A = np.array([[nq * r["p"], nq * r["p"] * math.log2(r["p"])] for r in ex])
        y = np.array([r["exp_ms"] for r in ex])
        (t_xmask, t_xrot), *_ = np.linalg.lstsq(A, y, rcond=None)
        lines.append(f"# f3 server-side expansion of the {nq} queries: t_xmask (Mul(P) + Res, one part) = "
                     f"{t_xmask * 1e3:.3f} us, t_xrot (level-1 Rot + Add) = {t_xrot * 1e3:.3f} us")
        lines.append(f"{'p':>4} {'scan_ms':>9} {'expand_ms':>10} {'exp_model':>10} {'total_ms':>9} {'tq_per_s':>12}")
        best2 = None
        for r in ex:
            em = nq * r["p"] * (t_xmask + math.log2(r["p"]) * t_xrot)
            tot = r["ms"] + r["exp_ms"]
            lines.append(f"{r['p']:>4} {r['ms']:>9.3f} {r['exp_ms']:>10.3f} {em:>10.3f} {tot:>9.3f} "
                         f"{n_tmpl * nq / (tot / 1e3):>12.4g}")
            if best2 is None or tot < best2[1]:
                best2 = (r["p"], tot)
        lines.append(f"# measured optimum of expansion + scan (the paper's trade-off, {n_tmpl} templates): "
                     f"p* = {best2[0]}; the expansion is per query, the scan per (query, set), so p* grows "
                     f"with the database")
    text = "\n".join(lines) + "\n"
    print(text)
    with open(a.out, "w") as f:
        f.write(text)


if __name__ == "__main__":
    main()
