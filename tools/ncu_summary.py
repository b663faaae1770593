"""Summarise ncu outputs into profiles/*.json (launch-list shares + the key
metrics of a --set full capture).

    python tools/ncu_summary.py launches gpurun_out/launches.csv out.json
    python tools/ncu_summary.py full gpurun_out/prof_br.ncu-rep out.json
"""
import csv
import io
import json
import subprocess
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "second": 1e3, "s": 1e3}


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    tot, cnt = {}, {}
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[ix["Kernel Name"]].split("(")[0]
        v = float(r[ix["Metric Value"]].replace(",", "")) * UNIT[r[ix["Metric Unit"]]]
        tot[k] = tot.get(k, 0.0) + v
        cnt[k] = cnt.get(k, 0) + 1
    s = sum(tot.values())
    res = {k: {"launches": cnt[k], "ms_total": round(v, 4), "ms_per_launch": round(v / cnt[k], 4),
               "share": round(v / s, 4)} for k, v in sorted(tot.items(), key=lambda x: -x[1])}
    json.dump({"source": path, "note": "ncu --metrics gpu__time_duration.sum --clock-control none "
               "(cold-cache, serialised launches: compare shares)", "kernels": res},
              open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_miss.sum",
    "l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__cluster_dim_x",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def full(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = {"source": path, "launches": []}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        ent = {"kernel": d.get("Kernel Name", "").split("(")[0]}
        for k in KEYS:
            if k in d:
                ent[k] = d[k] + (" " + u[k] if u.get(k) else "")
        try:
            rd = float(d["dram__bytes_read.sum"].replace(",", "")) * (1e6 if u["dram__bytes_read.sum"] == "Mbyte" else 1e3 if u["dram__bytes_read.sum"] == "Kbyte" else 1e9 if u["dram__bytes_read.sum"] == "Gbyte" else 1)
            wr = float(d["dram__bytes_write.sum"].replace(",", "")) * (1e6 if u["dram__bytes_write.sum"] == "Mbyte" else 1e3 if u["dram__bytes_write.sum"] == "Kbyte" else 1e9 if u["dram__bytes_write.sum"] == "Gbyte" else 1)
            ent["dram_bytes_per_launch"] = rd + wr
        except Exception:
            pass
        res["launches"].append(ent)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
