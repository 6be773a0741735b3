"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches gpurun_out/launches.csv  > profiles/rNN_launches.txt
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep [--traffic profiles/traffic.json] > profiles/rNN_ncu_full.txt
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        k = d["Kernel Name"].split("(")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"]) / 1e3
    tot = sum(a[1] for a in agg.values())
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)")
    print("# %d launches, %.1f us total" % (len(data), tot))
    print("%-62s %6s %11s %7s %9s" % ("kernel", "count", "total_us", "share", "avg_us"))
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("%-62s %6d %11.1f %6.1f%% %9.2f" % (k[:62], c, t, 100 * t / tot, t / c))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]


def full(path, traffic_out=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    print("# ncu --set full --clock-control none: %s (%d kernels)" % (path, len(data)))
    traffic = {}
    for d in data:
        name = d[idx["Kernel Name"]]
        print("\n## " + name)
        for k in KEYS:
            if k in idx:
                print("  %-80s %s %s" % (k, d[idx[k]], units[idx[k]]))
        try:
            rd = float(d[idx["dram__bytes_read.sum"]]) * _scale(units[idx["dram__bytes_read.sum"]])
            wr = float(d[idx["dram__bytes_write.sum"]]) * _scale(units[idx["dram__bytes_write.sum"]])
            traffic.setdefault(_short(name), int(rd + wr))
        except (KeyError, ValueError):
            pass
    if traffic_out:
        json.dump(traffic, open(traffic_out, "w"), indent=1)


def _scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def _short(name):
    """ncu kernel name -> the library's launch name (fde_profile_unit names)."""
    n = name.split("(")[0].replace("void ", "").replace("fde::", "")
    if "k_toeplitz_lines" in n:
        t = n.split("<")[1].split(">")[0].split(",")
        col, var = t[2].strip() == "1", t[3].strip() == "1"
        return ("toeplitz_cols" if col else "toeplitz_rows") + ("_var" if var else "")
    if "k_tau_lines" in n:
        return "tau_cols" if n.split("<")[1].split(",")[2].strip() == "1" else "tau_rows"
    if "k_dstm_lines" in n:
        t = [v.strip() for v in n.split("<")[1].split(">")[0].split(",")]
        col, tau = t[2] == "1", t[4] == "1"
        return ("tau" if tau else "dst") + ("_cols" if col else "_rows")
    if "k_sineop_lines" in n:
        mode = n.split("<")[1].split(">")[0].split(",")[3].strip()
        return {"0": "sine_op_rows", "1": "sine_op_cols", "2": "sine_op_1d"}[mode]
    if "k_sineop_rc" in n:
        return "sine_op_rc"
    if "k_sine_xr3" in n or "k_sine_xr4" in n:
        return "sine_xr_rc"
    if "k_sine_xr" in n:
        return "sine_xr"
    return n


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        out = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
        full(sys.argv[2], out)
