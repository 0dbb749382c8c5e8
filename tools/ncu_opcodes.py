import csv,sys,collections,subprocess
rep=sys.argv[1]
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(raw.splitlines())); h=rows[0]; v=rows[2]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum']
for i,n in enumerate(h):
    if n in want: print(n, rows[1][i], v[i])
src=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source=sass'],capture_output=True,text=True).stdout.splitlines()
r=csv.reader(src[1:]); hh=next(r)
ie=hh.index('Instructions Executed'); st=hh.index('Warp Stall Sampling (All Samples)'); sc=hh.index('Source')
cnt=collections.Counter(); stall=collections.Counter(); tot=0; tst=0
for row in r:
    if len(row)<=ie: continue
    t=row[sc].split()
    if not t: continue
    op=t[1] if t[0].startswith('@') else t[0]
    op=op.split('.')[0]
    n=int(row[ie] or 0); s=int(row[st] or 0)
    cnt[op]+=n; stall[op]+=s; tot+=n; tst+=s
print('total inst',tot,'stall samples',tst)
for op,n in cnt.most_common(24): print('%-10s %12d %5.1f%%  stall %5.1f%%'%(op,n,100*n/tot,100*stall[op]/tst))
