import csv, subprocess, sys
rep = sys.argv[1]  # an .ncu-rep, or the --page raw --csv export of one
if rep.endswith('.csv'):
    out = open(rep).read()
else:
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]; u = r[1]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'lts__t_sectors.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__grid_size',
        'launch__block_size', 'launch__shared_mem_per_block_dynamic', 'smsp__inst_executed.sum',
        'sm__cycles_elapsed.avg.per_second']
for v in r[2:]:
    print(v[h.index('Kernel Name')][:90])
    for w in want:
        if w in h:
            i = h.index(w); print('   %-60s %s %s' % (w, v[i], u[i]))
    if 'lts__t_sectors.sum' in h and 'gpu__time_duration.sum' in h:  # L2 traffic (32-B sectors) per second
        i, j = h.index('lts__t_sectors.sum'), h.index('gpu__time_duration.sum')
        t = float(v[j].replace(',', '')) * {'ns': 1e-9, 'nsecond': 1e-9, 'us': 1e-6, 'usecond': 1e-6,
                                            'ms': 1e-3, 'msecond': 1e-3}.get(u[j], 1e-9)
        print('   %-60s %.1f GB/s' % ('L2 sector bytes / duration', float(v[i].replace(',', '')) * 32 / t / 1e9))
    st = []
    for i, name in enumerate(h):
        if 'pcsamp_warps_issue_stalled' in name and not name.endswith('not_issued'):
            try:
                st.append((float(v[i].replace(',', '')), name.replace('smsp__pcsamp_warps_issue_stalled_', '')))
            except ValueError:
                pass
    tot = sum(x for x, _ in st) or 1
    print('   stalls:', ', '.join('%s %.0f%%' % (n, 100 * x / tot) for x, n in sorted(st, reverse=True)[:8]))
