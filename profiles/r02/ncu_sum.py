import csv, sys, subprocess, io
rep = sys.argv[1]
out = subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units = rows[0], rows[1]
want = ['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','launch__registers_per_thread',
 'sm__warps_active.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed',
 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','l1tex__t_sector_hit_rate.pct','lts__t_sector_hit_rate.pct',
 'lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed','lts__t_sectors_srcunit_tex.max.pct_of_peak_sustained_elapsed',
 'l1tex__m_xbar2l1tex_read_bytes.sum','smsp__inst_executed.sum','sm__inst_executed.sum.pct_of_peak_sustained_elapsed',
 'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
 'smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
 'smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio','smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
 'smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio','smsp__average_warp_latency_per_inst_issued.ratio',
 'dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__throughput.avg.pct_of_peak_sustained_elapsed']
idx = {h:i for i,h in enumerate(hdr)}
for r in rows[2:]:
    print('-----')
    for w in want:
        if w in idx: print(f'{w:80s} {r[idx[w]][:90]} {units[idx[w]]}')
