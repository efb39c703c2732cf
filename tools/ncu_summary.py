"""Summarise ncu output into profiles/ (tracked).

    python tools/ncu_summary.py LAUNCHES_CSV [FULL_NCU_REP] OUT_PREFIX

LAUNCHES_CSV: `ncu --metrics gpu__time_duration.sum --csv --log-file ...` of a bench run.
  -> OUT_PREFIX_launches.txt: per-kernel launch counts, total and mean device time and share of the
     bm_match kernels (cold-cache, serialised: compare SHARES with bench.py's per-class numbers).
FULL_NCU_REP: `ncu --set full -o ...` capture of the top kernel.
  -> OUT_PREFIX_full.txt: per-launch duration, DRAM bytes, pipe utilisation, issue, stalls, and the
     SASS opcode mix (from the source page).
"""
import collections
import csv
import io
import subprocess
import sys

MATCH_KERNELS = ("k_tensor_intt", "k_modup_ntt", "k_ks_intt", "k_rescale_ntt", "k_ladder", "k_rot_digit", "k_digits",
                 "k_rot_ks", "k_out_intt", "k_relin", "k_tensor", "k_tensor_mma", "k_tm_qexp")


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[iM] != "gpu__time_duration.sum":
            continue
        k = r[iK].split("(")[0].replace("void ", "")
        if k.startswith("k_tensor<2"):  # bm_match's tensor; k_tensor<3> is f1's (level 2)
            k = "k_tensor"
        elif k.startswith("bm::k_tensor_mma") or k.startswith("k_tensor_mma"):  # the tensor-core K1
            k = "k_tensor_mma"
        elif k.startswith("bm::k_tm_qexp") or k.startswith("k_tm_qexp"):  # its query operand
            k = "k_tm_qexp"
        elif k.startswith("k_ladder_t<"):  # throughput ladder / latency-mode cluster ladder
            first = k[len("k_ladder_t<"):].split(",")[0].split(">")[0].strip()  # CL: the first argument
            k = "k_ladder" if first in ("false", "0", "(bool)0") else "k_ladder_c2"
        tot[k] += float(r[iV].replace(",", ""))
        cnt[k] += 1
    match = {k: v for k, v in tot.items() if k in MATCH_KERNELS}
    s = sum(match.values()) or 1.0
    lines = [f"# {path}: ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)",
             f"{'kernel':24s} {'launches':>8s} {'total_us':>12s} {'mean_us':>10s} {'share_of_bm_match':>18s}"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        sh = f"{tot[k] / s * 100:17.1f}%" if k in match else f"{'-':>18s}"
        lines.append(f"{k:24s} {cnt[k]:8d} {tot[k] / 1e3:12.1f} {tot[k] / cnt[k] / 1e3:10.2f} {sh}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def full(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    lines = [f"# {rep}: ncu --set full --clock-control none (one capture per launch)"]
    for r in rows[2:]:
        d = dict(zip(h, r))
        lines.append(f"## launch {d.get('ID')}: {d.get('Kernel Name')}  grid {d.get('Grid Size')} block {d.get('Block Size')}")
        for k in KEYS:
            if k in d:
                lines.append(f"  {k:70s} {d[k]}")
        st = [(k, float(v)) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("_per_issue_active.ratio") and v not in ("", "n/a")]
        st.sort(key=lambda kv: -kv[1])
        lines.append("  stalls (warps per issue): " + ", ".join(
            f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={v:.2f}" for k, v in st[:8]))
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    hi = next((i for i, r in enumerate(srows) if "Source" in r and "Instructions Executed" in r), None)
    if hi is not None:
        h = srows[hi]
        iS, iE = h.index("Source"), h.index("Instructions Executed")
        iW = h.index("Warp Stall Sampling (All Samples)") if "Warp Stall Sampling (All Samples)" in h else None
        cnt, stall = collections.Counter(), collections.Counter()
        for r in srows[hi + 1:]:
            if len(r) <= iE or not r[iS].strip():
                continue
            tok = r[iS].strip().split()
            op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
            try:
                cnt[op] += int(r[iE])
                stall[op] += int(r[iW]) if iW is not None and r[iW] else 0
            except ValueError:
                pass
        tot = sum(cnt.values()) or 1
        lines.append("## SASS opcode mix (warp instructions, all captured launches; stall samples)")
        for op, n in cnt.most_common(30):
            lines.append(f"  {op:28s} {n:12d} {n / tot * 100:5.1f}%  stall_samples {stall[op]}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    a = sys.argv[1:]
    prefix = a[-1]
    if a[0].endswith(".csv"):
        launches(a[0], prefix + "_launches.txt")
        a = a[1:]
    if len(a) > 1 and a[0].endswith(".ncu-rep"):
        full(a[0], prefix + "_full.txt")
