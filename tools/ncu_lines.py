import csv,sys,subprocess,collections
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source=cuda,sass'],capture_output=True,text=True).stdout.splitlines()
fname=None; res=[]
i=0
hdr=None
for line in out:
    row=next(csv.reader([line]))
    if row and row[0]=='File Path': fname=row[1].split('/')[-1]; continue
    if row and row[0]=='Line No': hdr=row; continue
    if row and row[0] in('Function Name',): continue
    if hdr and len(row)>8 and row[0].isdigit():
        try: n=int(row[7]); s=int(row[4])
        except: continue
        res.append((n,s,fname,row[0],row[1][:90]))
tot=sum(r[0] for r in res); ts=sum(r[1] for r in res)
res.sort(reverse=True)
for n,s,f,l,src in res[:int(sys.argv[2]) if len(sys.argv)>2 else 40]:
    print('%5.1f%% st%5.1f%% %s:%s  %s'%(100*n/tot,100*s/ts,f,l,src))
