"""Summarise an ncu --set full capture + a launch-list CSV into profiles/ (tracked).

usage: python tools/ncu_summary.py <tag> <prof.ncu-rep> <launches.csv> <workload> <mode> <omega> [note]
Writes profiles/<tag>.md and profiles/traffic_<workload>_<mode>_<omega>.json (read by bench.py).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__cluster_dim_x", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "sm__cycles_elapsed.avg.per_second",
]


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        res.append({k: (d.get(k), units[hdr.index(k)] if k in hdr else "") for k in KEYS + ["Kernel Name"]})
    return res


def to_bytes(v, u):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def launch_list(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = {}
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*", "", r[ki]).split("<")[0].replace("void ", "").strip()
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    return agg


def main():
    tag, rep, launches, wl, mode, omega = sys.argv[1:7]
    note = sys.argv[7] if len(sys.argv) > 7 else ""
    mets = raw_metrics(rep)
    agg = launch_list(launches)
    total = sum(v[1] for k, v in agg.items() if k.startswith("sk::"))
    m = mets[0]
    rd = to_bytes(*m["dram__bytes_read.sum"])
    wr = to_bytes(*m["dram__bytes_write.sum"])
    lines = [f"# ncu summary `{tag}`", "", note, "",
             f"Kernel: `{m['Kernel Name'][0][:160]}`", "", "| metric | value | unit |", "|---|---|---|"]
    for k in KEYS:
        v, u = m[k]
        if v not in (None, ""):
            lines.append(f"| {k} | {v} | {u} |")
    lines += ["", f"DRAM traffic per launch: read {rd/1e9:.3f} GB + write {wr/1e9:.3f} GB = {(rd+wr)/1e9:.3f} GB", "",
              "## Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold-cache, serialised)", "",
              "Shares are of the libsketch kernels (one step = sketch_gemm + splitk_reduce + core_gemm +",
              "core_reduce); the other launches are input generation / parity setup outside the timed region.", "",
              "| kernel | launches | total µs | µs per launch | share of step |", "|---|---|---|---|---|"]
    for name, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        share = f"{us/total:.1%}" if name.startswith("sk::") else "setup"
        lines.append(f"| {name} | {n} | {us:.1f} | {us/n:.1f} | {share} |")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}.md"), "w").write("\n".join(lines) + "\n")
    tr = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr, "source": f"profiles/{tag}.md",
          "kernel": m["Kernel Name"][0][:200], "duration_ms_under_ncu": float(m["gpu__time_duration.sum"][0]) *
          {"msecond": 1, "usecond": 1e-3, "nsecond": 1e-6}.get(m["gpu__time_duration.sum"][1], 1)}
    json.dump(tr, open(os.path.join(ROOT, "profiles", f"traffic_{wl}_{mode}_{omega}.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
