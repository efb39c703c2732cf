"""Render bench.py JSON lines (one per config / p) as BASELINE.md's "Measured results" table.

    python tools/baseline_table.py profiles/r02_configs.jsonl [more.jsonl ...]
"""
import json
import sys


def pct_int(rf):
    """dominant kernel vs the integer roofline: executed modmuls (every line), and SURVEY 8(d)'s count
    where the line carries both (bench lines since the P-scaled ladder: `frac` = 8(d), `executed`)"""
    if "executed" in rf:
        return f"{100 * rf['executed']['frac']:.1f}% executed, {100 * rf['frac']:.1f}% by §8(d)'s count"
    return f"{100 * rf['frac']:.1f}%"


def row(d):
    c = d["config"]
    v = d.get("verify") or {}
    cpu = d.get("cpu_baseline") or {}
    rf = d["roofline"]
    cfg = c["workload"].split(":")[0].replace("BASELINE ", "")
    prefix = " (1-GPU prefix: 1/8 of the DB)" if "prefix" in c["workload"] else ""
    par = v.get("parity", "—")
    if par == "bit-exact":
        par = f"bit-exact ({v.get('oracle_pairs')} pairs + encryption)"
    top = v.get("top1_agree_genuine")
    top = "—" if top is None else f"{top:.3f}"
    if v.get("top1_agree_all") is not None:
        top += f" (all {v['top1_agree_all']:.3f})"
    err = v.get("max_abs_score_err")
    return (f"| {cfg}{prefix} | {c['d']} | {c['p']} | {d['n_gpus']} | {d['value'] / 1e6:.2f} M | {d['ms_per_step']:.1f} | "
            f"{100 * rf['hbm']['frac']:.2f}% | {pct_int(rf)} ({rf['kernel']}) / {100 * rf['step_frac']:.1f}% (step) | "
            f"{cpu.get('value', 0) / 1e3:.1f} K ({cpu.get('cores', '—')}) | {par} | "
            f"{'—' if err is None else f'{err:.1e}'} | {top} |")


def main():
    print("| Config | d | p | GPUs | templates·queries/s | ms/step | %HBM | %INT (dominant kernel / whole step) | "
          "oracle tq/s (cores) | parity | max score err | top-1 agree (genuine) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for path in sys.argv[1:]:
        for line in open(path):
            line = line.strip()
            if not line.startswith("{"):
                continue
            d = json.loads(line)
            if d.get("impl") == "reference" or "roofline" not in d:
                continue
            print(row(d))


if __name__ == "__main__":
    main()
