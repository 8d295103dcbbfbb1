"""Summarise ncu captures (gpurun_out/prof_<tag>_<wl>.ncu-rep) and launch lists
(gpurun_out/launches_<tag>_<wl>.csv) into profiles/<tag>_summary.md + CSV copies."""
import csv
import io
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("PROF_OUT") or os.path.join(ROOT, "profiles")

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg",
       "gpc__cycles_elapsed.max", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor.sum", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
       "launch__shared_mem_per_block_dynamic"]


def ncu_raw(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {n: (v[i], u[i]) for i, n in enumerate(h)}
    stalls = []
    for i, n in enumerate(h):
        if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
            try:
                stalls.append((float(v[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    return d, stalls


def sass_evidence(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                       capture_output=True, text=True)
    txt = r.stdout
    keys = ["UTMALDG", "UBLKCP", "HMMA", "LDSM", "MOVM", "SYNCS", "UTCHMMA", "LDGSTS"]
    return {k: txt.count(k) for k in keys}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        agg[r[ki]].append(float(r[vi].replace(",", "")))
    return agg


def main(tag="r1", wls=("c2", "c3", "c4")):
    os.makedirs(PROF, exist_ok=True)
    traffic = {}
    lines = [f"# ncu evidence — {tag}", "",
             "Captured under gpurun on one B200 with `scripts/gpu_round.sh` (`ncu --set full --clock-control none "
             "--import-source on -k regex:<the single-launch decode_kernel<G, true>>`; launch lists with "
             "`--metrics gpu__time_duration.sum`). "
             "ncu numbers are serialised, cold-cache replays: compare shares, not absolutes, with bench.py.", ""]
    for wl in wls:
        rep = os.path.join(OUT, f"prof_{tag}_{wl}.ncu-rep")
        lst = os.path.join(OUT, f"launches_{tag}_{wl}.csv")
        lines.append(f"## {wl}")
        if os.path.exists(rep):
            d, stalls = ncu_raw(rep)
            g = lambda k: d.get(k, ("n/a", ""))
            dur_us = float(g("gpu__time_duration.sum")[0].replace(",", ""))
            dur_unit = g("gpu__time_duration.sum")[1]
            if dur_unit == "ms":
                dur_us *= 1e3
            elif dur_unit in ("ns", "nsecond"):
                dur_us /= 1e3
            rd = g("dram__bytes_read.sum")
            wr = g("dram__bytes_write.sum")
            try:
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
                r_b = float(rd[0].replace(",", "")) * scale.get(rd[1], 1)
                w_b = float(wr[0].replace(",", "")) * scale.get(wr[1], 1)
                traffic[wl] = {"traffic": int(r_b + w_b), "dram_read": int(r_b), "dram_write": int(w_b),
                               "duration_us": round(dur_us, 2),
                               "kernel": "decode_kernel<G, true> (single-launch l4_decode_attention)",
                               "source": f"prof_{tag}_{wl}.ncu-rep (ncu --set full)"}
            except ValueError:
                pass
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for k in RAW:
                if k in d:
                    lines.append(f"| `{k}` | {d[k][0]} {d[k][1]} |")
            tot = sum(x for x, _ in stalls) or 1.0
            top = sorted(stalls, reverse=True)[:6]
            lines.append("")
            lines.append("Top warp stall reasons (share of samples): " +
                         ", ".join(f"{n} {x / tot * 100:.1f}%" for x, n in top))
            ev = sass_evidence(rep)
            lines.append("")
            lines.append("SASS instruction counts in the kernel (static): " + ", ".join(f"{k} {v}" for k, v in ev.items()))
        if os.path.exists(lst):
            agg = launches(lst)
            total = sum(sum(v) for v in agg.values())
            lines.append("")
            lines.append("Launch list (all kernels of the command; share of GPU time):")
            lines.append("")
            lines.append("| kernel | launches | mean us | share |")
            lines.append("|---|---|---|---|")
            for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
                lines.append(f"| `{k[:70]}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / total * 100:.1f}% |")
            shutil.copy(lst, os.path.join(PROF, os.path.basename(lst)))
        lines.append("")
    open(os.path.join(PROF, f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    if traffic:
        import json
        json.dump(traffic, open(os.path.join(PROF, f"{tag}_traffic.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1", tuple(sys.argv[2:]) or ("c2", "c3", "c4"))
