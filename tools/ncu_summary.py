"""Summarise an ncu report (raw page) into the numbers DESIGN.md / bench.py use.
    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--json out.json --config 2 --terms N]"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
    "sm__inst_executed.avg.per_cycle_active", "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
]
STALL = "smsp__average_warps_issue_stalled_"


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def main():
    rep = sys.argv[1]
    d = raw(rep)
    res = {}
    for k in KEYS:
        for h, (v, u) in d.items():
            if h == k:
                res[k] = (v, u)
    stalls = {h[len(STALL):].replace("_per_issue_active.ratio", ""): float(v)
              for h, (v, u) in d.items() if h.startswith(STALL) and h.endswith("_per_issue_active.ratio")}
    for k, (v, u) in res.items():
        print(f"{k:70s} {v} {u}")
    print("stalls per issued instruction:")
    for k, v in sorted(stalls.items(), key=lambda x: -x[1]):
        if v > 0.01:
            print(f"   {k:40s} {v:.3f}")
    if "--json" in sys.argv:
        path = sys.argv[sys.argv.index("--json") + 1]
        cfg = int(sys.argv[sys.argv.index("--config") + 1]) if "--config" in sys.argv else None
        num = lambda k: float(res[k][0].replace(",", "")) if k in res else None
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        nbytes = lambda k: num(k) * scale.get(res[k][1], float("nan")) if k in res else 0.0
        summ = {"report": rep, "config": cfg,
                "duration_ns": num("gpu__time_duration.sum"),
                "dram_bytes_per_launch": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"),
                "metrics": {k: v for k, (v, u) in res.items()}, "stalls_per_issue": stalls}
        with open(path, "w") as f:
            json.dump(summ, f, indent=1)


if __name__ == "__main__":
    main()
