"""Key metrics + top stall reasons from an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
keep = ['Duration', 'Compute (SM) Throughput', 'DRAM Throughput', 'Issue Slots Busy', 'Registers Per Thread',
        'Achieved Occupancy', 'Theoretical Occupancy', 'Warp Cycles Per Issued Instruction', 'Executed Instructions',
        'Memory Throughput', 'No Eligible', 'Active Warps Per Scheduler', 'Eligible Warps Per Scheduler',
        'Grid Size', 'Block Size', 'Waves Per SM']
r = list(csv.reader(io.StringIO(det)))
h = r[0]
out = {}
for row in r[1:]:
    d = dict(zip(h, row))
    if d['Metric Name'] in keep and d['Metric Name'] not in out:
        out[d['Metric Name']] = f"{d['Metric Value']} {d['Metric Unit']}"
        print(f"  {d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units, vals = r[0], r[1], r[2]
st = []
for k, u, v in zip(h, units, vals):
    if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio'):
        try:
            st.append((float(v), k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
        except ValueError:
            pass
    if k in ('sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active',
             'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
             'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
             'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
             'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__inst_executed.sum'):
        print(f"  {k:70s} {v} {u}")
st.sort(reverse=True)
print("  stalls (warps per issue):", ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))
