"""Summarise a gpurun ncu launch list + one --set full capture into profiles/ (committed evidence).

    python tools/profile_summary.py <round-tag> gpurun_out/launches.csv gpurun_out/prof.ncu-rep <mcs/launch> [kernel] [capture command]
"""
import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_table(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for r in data:
        name = re.sub(r"\(.*", "", r[ik]).replace("void ", "").replace("escgd::", "").replace("<unnamed>::", "")
        agg.setdefault(name, []).append(float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0))
    return agg


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    return [dict(zip(hdr, v)) for v in rows[2:]]


KERNEL = sys.argv[5] if len(sys.argv) > 5 else "block_kernel"
CAPTURE = sys.argv[6] if len(sys.argv) > 6 else "`python tools/one_block.py 3200 200` (ncu --set full -s 50 -c 1)"


def main():
    tag, launches, rep = sys.argv[1], sys.argv[2], sys.argv[3]
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    agg = launch_table(launches)
    tot = sum(sum(v) for v in agg.values())
    lines = ["# %s launch list (ncu --metrics gpu__time_duration.sum --clock-control none)" % tag, "",
             "Command: `python bench.py --steps 1 --warmup 1 --no-cpu-baseline` (first 700 launches).",
             "Per-launch times are cold-cache and serialised (compare shares, not absolutes).",
             "Full capture (`%s_%s_ncu_details.txt`, `ncu_summary.json`): one steady-state launch of %s, the bench's "
             "kernel shape." % (tag, KERNEL, CAPTURE), "",
             "| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    for k, v in agg.items():
        lines.append("| %s | %d | %.2f | %.1f | %.1f%% |" % (k, len(v), sum(v) / len(v), sum(v), 100 * sum(v) / tot))
    open(os.path.join(prof, "%s_launches.md" % tag), "w").write("\n".join(lines) + "\n")
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
    caps = ncu_raw(rep)
    units = {}
    try:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        units = dict(zip(rows[0], rows[1]))
    except Exception:
        pass
    summ = {"tag": tag, "kernel": KERNEL, "capture": CAPTURE, "captures": [{k: c.get(k) for k in keys} for c in caps], "units": {k: units.get(k) for k in keys}}
    # DRAM bytes per launch of the dominant kernel (the full-MCS-count launch = largest duration)
    big = max(caps, key=lambda c: float(c["gpu__time_duration.sum"]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rb = float(big["dram__bytes_read.sum"]) * scale.get(units.get("dram__bytes_read.sum", "byte"), 1)
    wb = float(big["dram__bytes_write.sum"]) * scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
    summ["dram_bytes_per_launch"] = rb + wb
    summ["mcs_per_launch"] = int(sys.argv[4]) if len(sys.argv) > 4 else None
    summ["warp_inst_per_launch"] = float(big["smsp__inst_executed.sum"])
    json.dump(summ, open(os.path.join(prof, "ncu_summary.json"), "w"), indent=1)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    open(os.path.join(prof, "%s_%s_ncu_details.txt" % (tag, KERNEL)), "w").write(det)
    print("\n".join(lines))
    print(json.dumps(summ["captures"], indent=1)[:2000])


if __name__ == "__main__":
    main()
