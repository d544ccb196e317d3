"""Summarise an ncu --set full report (first kernel) into key lines.
usage: python tools/ncu_summary.py REPORT.ncu-rep N_ELEMENTS [out.txt]"""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
d = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
keep = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "local_load_bytes", "smsp__sass_inst_executed_op_local_ld.sum",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"]
out = []
for k in keep:
    if k in d:
        out.append(f"{k} [{u.get(k, '')}] = {d[k]}")
cyc = float(d["sm__cycles_elapsed.avg"])
rates = {op: float(d.get(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed", 0) or 0)
         for op in ("dfma", "dmul", "dadd", "ffma", "fmul", "fadd")}
fp64_flops = (2 * rates["dfma"] + rates["dmul"] + rates["dadd"]) * cyc
fp64_inst = (rates["dfma"] + rates["dmul"] + rates["dadd"]) * cyc
out.append(f"derived: FP64 thread flops per element (DFMA=2) = {fp64_flops / n:.1f}")
out.append(f"derived: FP64 thread instructions per element (DFMA+DMUL+DADD) = {fp64_inst / n:.1f}")
out.append(f"derived: FP32 thread instructions per element = "
           f"{(rates['ffma'] + rates['fmul'] + rates['fadd']) * cyc / n:.1f}")
out.append(f"derived: warp instructions per 32 elements = {float(d['smsp__inst_executed.sum']) / (n / 32):.0f}")
out.append(f"derived: dram bytes per element = "
           f"{(float(d['dram__bytes_read.sum']) * (1e6 if u['dram__bytes_read.sum'] == 'Mbyte' else 1e3 if u['dram__bytes_read.sum'] == 'Kbyte' else 1) + float(d['dram__bytes_write.sum']) * (1e6 if u['dram__bytes_write.sum'] == 'Mbyte' else 1e3 if u['dram__bytes_write.sum'] == 'Kbyte' else 1)) / n:.2f}")
txt = "\n".join(out)
print(txt)
if len(sys.argv) > 3:
    open(sys.argv[3], "w").write(f"# ncu --set full --clock-control none summary of {rep}\n" + txt + "\n")
