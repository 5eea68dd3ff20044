"""Key counters + top stall reasons of kernels in an ncu report (build container)."""
import csv, subprocess, sys, io
rep, pat = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw))); h = rows[0]
for r in rows[2:]:
    if pat not in r[h.index('Kernel Name')]:
        continue
    print(r[h.index('Kernel Name')][:70])
    for n in ['gpu__time_duration.sum', 'smsp__inst_executed.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
              'lts__t_sectors_srcunit_tex_op_red.sum',
              'lts__d_atomic_input_cycles_active.max.pct_of_peak_sustained_elapsed',
              'lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed',
              'sm__warps_active.avg.pct_of_peak_sustained_active',
              'smsp__issue_active.avg.pct_of_peak_sustained_active',
              'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
              'lts__throughput.avg.pct_of_peak_sustained_elapsed',
              'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__registers_per_thread',
              'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers']:
        if n in h:
            print(f"  {n} = {r[h.index(n)]} {rows[1][h.index(n)]}")
    st = [(n, r[i]) for i, n in enumerate(h)
          if n.startswith('smsp__average_warps_issue_stalled_') and n.endswith('per_issue_active.ratio')]
    st = [(n, float(v)) for n, v in st if v.replace('.', '', 1).isdigit()]
    for n, v in sorted(st, key=lambda x: -x[1])[:7]:
        print('   stall', n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), round(v, 2))
    break
