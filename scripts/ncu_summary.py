"""Summarise `ncu --set full` reports of the NA2D kernels into profiles/: a markdown table and
profiles/ncu_traffic.json (DRAM bytes per launch, read by bench.py for roofline.traffic).

    python scripts/ncu_summary.py OUT.md CONFIG_NAME report1.ncu-rep [report2 ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pct",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_rt_pct",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active": "shared_pipe_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "lds_conflicts",
    "launch__registers_per_thread": "regs",
    "launch__block_size": "block",
    "launch__grid_size": "grid",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    name = v[h.index("Kernel Name")]
    d = {"kernel": name.split("(")[0].split("<")[0].split("::")[-1]}
    for i, n in enumerate(h):
        if n in KEYS:
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                continue
            d[KEYS[n]] = x * UNIT.get(u[i], 1)
        elif "pipe_tensor" in n and "pct" in n and "tensor_any" not in d:
            try:
                d["tensor_any"] = (n, float(v[i].replace(",", "")))
            except ValueError:
                pass
    return d


def tensor_cell(d):
    """tensor-pipe activity: % of active cycles (and % of elapsed realtime cycles when captured)"""
    if "tensor_pct" in d and "tensor_rt_pct" in d:
        return "{:.1f} / {:.1f}".format(d["tensor_pct"], d["tensor_rt_pct"])
    if "tensor_pct" in d or "tensor_rt_pct" in d:
        return "{:.1f}".format(d.get("tensor_pct", d.get("tensor_rt_pct")))
    if "tensor_any" in d:
        return "{:.1f} ({})".format(d["tensor_any"][1], d["tensor_any"][0])
    return "n/a"


def main():
    out_md, cfg, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    rows = [load(r) for r in reps]
    lines = ["| kernel | us | DRAM read MB | DRAM write MB | DRAM GB/s | SM % | mem % | issue % | XU % | ALU % | FMA % | L2 hit % | tensor pipe % | regs |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in rows:
        t = d.get("duration", 0)
        tot = d.get("dram_read", 0) + d.get("dram_write", 0)
        lines.append("| {} | {:.1f} | {:.1f} | {:.1f} | {:.0f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {:.1f} | {} | {:.0f} |".format(
            d["kernel"], t, d.get("dram_read", 0) / 1e6, d.get("dram_write", 0) / 1e6, tot / (t * 1e-6) / 1e9 if t else 0,
            d.get("sm_pct", 0), d.get("mem_pct", 0), d.get("issue_pct", 0), d.get("xu_pct", 0), d.get("alu_pct", 0),
            d.get("fma_pct", 0), d.get("l2_hit_pct", 0), tensor_cell(d), d.get("regs", 0)))
    open(out_md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    tpath = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    tj = json.load(open(tpath)) if os.path.exists(tpath) else {}
    names = {"na2d_fwd_tc_kernel": "na2d_fwd_tc", "na2d_bwd_dq_kernel": "na2d_bwd_dq_tc",
             "na2d_bwd_dkdv_kernel": "na2d_bwd_dkdv_tc"}
    for d in rows:
        k = names.get(d["kernel"], d["kernel"])
        tj.setdefault(cfg, {})[k] = d.get("dram_read", 0) + d.get("dram_write", 0)
    json.dump(tj, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main()
