"""Summarise an ncu report: key SOL / scheduler metrics and the top SASS lines."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(io.StringIO(out))
h = next(r)
iS, iM, iU, iV = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
keep = ("Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L2 Cache Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Achieved Occupancy")
for row in r:
    if row[iM] in keep:
        print("%-45s %s %s" % (row[iM], row[iV], row[iU]))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
names, units, vals = rr[0], rr[1], rr[2]
for want in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active",
             "lts__t_bytes.sum", "sm__inst_executed_pipe_alu", "sm__inst_executed_pipe_fma",
             "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
             "sm__pipe_shared_cycles_active", "sm__pipe_alu_cycles_active", "sm__pipe_fma_cycles_active"):
    for n, u, v in zip(names, units, vals):
        if n.startswith(want):
            print("%-70s %s %s" % (n, v, u))
