"""Summarise an ncu --set full report (raw page) for one kernel launch:
time, DRAM bytes, pipe utilisation, occupancy, issue and stall breakdown.
Usage: python tools/ncu_summary.py report.ncu-rep [active_nodes] > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active", "adu pipe %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "thread DFMA"),
    ("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "thread DMUL"),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "thread DADD"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock Hz"),
]


def main():
    rep = sys.argv[1]
    nodes = float(sys.argv[2]) if len(sys.argv) > 2 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        kv = dict(zip(hdr, r))
        un = dict(zip(hdr, units))
        print(f"kernel: {kv.get('Kernel Name', '?')[:100]}")
        for k, label in KEYS:
            if k in kv:
                print(f"  {label:28s} {kv[k]:>18s} {un.get(k, '')}")
        stalls = {h: kv[h] for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")}
        print("  stall reasons (warps per issue):")
        for h, v in sorted(stalls.items(), key=lambda x: -float(x[1] or 0))[:8]:
            print(f"    {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v}")
        if nodes:
            tr = (float(kv["dram__bytes_read.sum"]) + float(kv["dram__bytes_write.sum"]))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[un["dram__bytes_read.sum"]]
            wi = float(kv["smsp__inst_executed.sum"])
            f64 = sum(float(kv.get(k, 0)) for k in ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
                                                    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
                                                    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"))
            print(f"  per node-update: DRAM {tr * scale / nodes:.1f} B, thread instructions {32 * wi / nodes:.0f}, "
                  f"fp64 thread ops {f64 / nodes:.0f}")


if __name__ == "__main__":
    main()
