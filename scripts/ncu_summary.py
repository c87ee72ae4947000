"""Prints the key metrics of an ncu report (dev aid): python scripts/ncu_summary.py rep.ncu-rep"""
import csv, subprocess, sys, io
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ["Duration", "Elapsed Cycles", "SM Active Cycles", "Compute (SM) Throughput", "Memory Throughput",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Achieved Occupancy",
        "Registers Per Thread", "Executed Instructions", "Avg. Active Threads Per Warp", "Branch Efficiency",
        "Mem Busy", "Max Bandwidth", "Mem Pipes Busy"]
seen = set()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    n = d.get("Metric Name")
    if n in want and n not in seen:
        seen.add(n)
        print(f"{n:40s} {d.get('Metric Unit',''):12s} {d.get('Metric Value','')}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, u, v = rr[0], rr[1], rr[2]
for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
            "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
            "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_wait",
            "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
            "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected",
            "smsp__pcsamp_warps_issue_stalled_no_instructions", "smsp__pcsamp_warps_issue_stalled_dispatch_stall",
            "smsp__pcsamp_warps_issue_stalled_mio_throttle", "smsp__pcsamp_warps_issue_stalled_tex_throttle",
            "smsp__pcsamp_warps_issue_stalled_barrier", "smsp__pcsamp_warps_issue_stalled_lsu_dependency" ,
            "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_alu.sum", "smsp__inst_executed_pipe_lsu.sum",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
            "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu.sum"]:
    for i, name in enumerate(h):
        if name == key:
            print(f"{name:70s} {u[i]:10s} {v[i]}")
