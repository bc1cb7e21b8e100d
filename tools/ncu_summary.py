"""Dev tool: one-screen summary of an ncu --set full report (key metrics + DRAM traffic)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
keep = ["Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Active Warps Per SM", "Eligible Warps Per Scheduler",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Cluster Size", "Grid Size", "Block Size",
        "Max Active Clusters", "L2 Hit Rate", "Executed Instructions", "Theoretical Occupancy"]
r = csv.reader(io.StringIO(det)); h = next(r); name = None
out = []
for row in r:
    d = dict(zip(h, row))
    name = d.get("Kernel Name", name)
    if d.get("Metric Name") in keep:
        out.append(f"{d['Metric Name']:36s} {d['Metric Value']} {d['Metric Unit']}")
rr = list(csv.reader(io.StringIO(raw)))
hh, units, vals = rr[0], rr[1], rr[2]
m = dict(zip(hh, vals)); u = dict(zip(hh, units))
tr = []
for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed_pipe_fma.sum",
            "smsp__inst_executed_pipe_fp64.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]:
    if key in m:
        tr.append(f"{key:60s} {m[key]} {u.get(key, '')}")
print(f"kernel: {name[:100] if name else '?'}\nreport: {rep}")
print("\n".join(out)); print("\n".join(tr))
