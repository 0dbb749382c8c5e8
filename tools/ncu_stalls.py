import csv,sys,subprocess
rep=sys.argv[1]
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(raw.splitlines())); h=rows[0]; v=rows[2]
items=[]
for i in range(len(h)):
    if h[i].startswith('smsp__pcsamp_warps_issue_stalled') and not h[i].endswith('not_issued'):
        try: items.append((float(v[i]),h[i]))
        except: pass
items.sort(reverse=True); tot=sum(x for x,_ in items)
for x,n in items[:12]: print('%6.1f%% %s'%(100*x/tot,n.replace('smsp__pcsamp_warps_issue_stalled_','')))
