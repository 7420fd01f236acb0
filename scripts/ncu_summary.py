"""Summarise an ncu --set full report into profiles/<name>_ncu_summary.txt.
usage: python scripts/ncu_summary.py REPORT.ncu-rep OUT.txt "title" """
import csv, io, subprocess, sys
rep, out, title = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
v = dict(zip(hdr, vals)); u = dict(zip(hdr, units))
keys = ['gpu__time_duration.sum', 'sm__cycles_elapsed.avg.per_second',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'sm__issue_active.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_tma.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_registers', 'launch__grid_size', 'launch__block_size',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'dram__bytes_read.sum.pct_of_peak_sustained_elapsed',
        'lts__t_bytes.sum', 'smsp__inst_executed.sum']
keys += [k for k in hdr if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
with open(out, 'w') as f:
    f.write(f"# {title}\n# ncu --set full --clock-control none --import-source on (B200, sm_100a); see profiles/README.md\n")
    for k in keys:
        if k in v and v[k] not in ('', 'n/a'):
            f.write(f"{k} [{u.get(k,'')}] = {v[k]}\n")
print(open(out).read())
