"""Summarise ncu reports / launch lists into profiles/ (markdown + JSON). Diagnostic tooling.

usage: python tools/ncu_summary.py REPORT.ncu-rep [--launches LAUNCHES.csv] --tag NAME
Writes profiles/<tag>.md and profiles/<tag>.json (per-launch duration, DMMA pipe utilisation,
DRAM bytes, L2 hit rate, occupancy, registers, top stall reasons).
"""
import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dmma_pct_of_active": "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "dyn_smem_bytes": "launch__shared_mem_per_block_dynamic",
}


def _num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[2:]


def summarise(rep):
    h, rows = raw_rows(rep)
    res = []
    for r in rows:
        d = dict(zip(h, r))
        e = {"kernel": d.get("Kernel Name", "")[:90]}
        for k, m in KEYS.items():
            e[k] = _num(d.get(m))
        if e["duration_us"] is not None:
            e["duration_us"] /= 1e3  # base unit ns
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), _num(v) or 0.0) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")]
        tot = sum(v for _, v in st) or 1.0
        e["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st, key=lambda kv: -kv[1])[:6]}
        res.append(e)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    # share of the step: over libfdp's own kernels only (the bench's L2-flush fills run between
    # steps, outside the timed step)
    tot_fdp = sum(sum(v) for k, v in agg.items() if k.startswith("fdp::")) or tot
    return {k: {"launches": len(v), "total_us": round(sum(v), 1), "mean_us": round(sum(v) / len(v), 2),
                "share": round(sum(v) / tot, 4),
                "share_of_step": round(sum(v) / tot_fdp, 4) if k.startswith("fdp::") else None}
            for k, v in agg.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    a = ap.parse_args()
    out = {"tag": a.tag}
    if a.report:
        out["kernels"] = summarise(a.report)
    if a.launches:
        out["launch_list"] = launches(a.launches)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", a.tag + ".json"), "w") as f:
        json.dump(out, f, indent=1)
    lines = [f"# {a.tag}", ""]
    if "launch_list" in out:
        lines += ["## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)", "",
                  "| kernel | launches | total us | mean us | share (all) | share of step (libfdp kernels) |",
                  "|---|---|---|---|---|---|"]
        for k, v in out["launch_list"].items():
            sos = "-" if v["share_of_step"] is None else f"{v['share_of_step']:.3f}"
            lines.append(f"| {k} | {v['launches']} | {v['total_us']} | {v['mean_us']} | {v['share']:.3f} | {sos} |")
        lines.append("")
    if "kernels" in out:
        lines += ["## Full-set captures", "",
                  "| kernel | us | DMMA % of active | DRAM read MB | DRAM write MB | L2 hit % | warps active % | regs | top stalls |",
                  "|---|---|---|---|---|---|---|---|---|"]
        for e in out["kernels"]:
            st = ", ".join(f"{k} {v}" for k, v in e["top_stalls_pct"].items())
            f = lambda x, s=1.0, p=1: "-" if x is None else f"{x / s:.{p}f}"
            lines.append(f"| {e['kernel'][:60]} | {f(e['duration_us'])} | {f(e['dmma_pct_of_active'])} | "
                         f"{f(e['dram_read_bytes'], 1e6)} | {f(e['dram_write_bytes'], 1e6)} | {f(e['l2_hit_pct'])} | "
                         f"{f(e['warps_active_pct'])} | {f(e['registers'], 1, 0)} | {st} |")
    with open(os.path.join(ROOT, "profiles", a.tag + ".md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
