"""Summarise an ncu report (raw page) into the metrics we track; dev tool."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__occupancy_limit_registers', 'smsp__inst_executed.sum', 'l1tex__t_sector_hit_rate.pct',
        'smsp__average_warp_latency_per_inst_issued.ratio', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'smsp__pcsamp_warps_issue_stalled_long_scoreboard', 'smsp__pcsamp_warps_issue_stalled_barrier',
        'smsp__pcsamp_warps_issue_stalled_short_scoreboard', 'smsp__pcsamp_warps_issue_stalled_wait',
        'smsp__pcsamp_warps_issue_stalled_lg_throttle', 'smsp__pcsamp_warps_issue_stalled_mio_throttle',
        'smsp__pcsamp_warps_issue_stalled_math_pipe_throttle']
idx = [hdr.index(w) for w in want if w in hdr]
for r in rows[2:]:
    d = {hdr[i]: r[i] for i in idx}
    name = d['Kernel Name'].split('(')[0].split('::')[-1]
    print(f"== {name}")
    for i in idx[1:]:
        print(f"   {hdr[i]:<62} {r[i]:>16} {units[i]}")
