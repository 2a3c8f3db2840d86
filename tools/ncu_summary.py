"""Summarise an ncu --set full report: the metrics this project tracks."""
import csv, subprocess, sys
KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sectors_srcunit_tex_op_read.sum',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct', 'launch__grid_size',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__occupancy_limit_registers',
        'sm__maximum_warps_per_active_cycle_pct', 'smsp__average_warp_latency_issue_stalled_long_scoreboard']
for fn in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", fn, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(h, r))
        print(f"== {fn}: {d.get('Kernel Name')}")
        for k in KEYS:
            if k in h:
                print(f"   {k:70s} {d.get(k):>16s} {u[h.index(k)]}")
