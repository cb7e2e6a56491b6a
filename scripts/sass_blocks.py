"""Instructions of one kernel grouped by execution count (loop bodies vs straight-line code):
    python scripts/sass_blocks.py REPORT.ncu-rep KERNEL_REGEX TOP"""
import subprocess, csv, io, sys
rep, kern = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass","-k",f"regex:{kern}","-c","1"],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(raw)))
hi=next(i for i,r in enumerate(rows) if "Instructions Executed" in r); h=rows[hi]
ia,isrc,ie,it=h.index("Address"),h.index("Source"),h.index("Instructions Executed"),h.index("Thread Instructions Executed")
body=[r for r in rows[hi+1:] if len(r)==len(h) and r[ia].startswith("0x")]
seen=set(); b2=[]
for r in body:
    if r[ia] in seen: break
    seen.add(r[ia]); b2.append(r)
body=b2
# blocks: runs of consecutive instructions with equal exec count
blocks=[]; cur=None
for i,r in enumerate(body):
    e=int(r[ie] or 0); t=int(r[it] or 0)
    if cur and cur['e']==e and e>0:
        cur['n']+=1; cur['t']+=t; cur['ops'].append(r[isrc].split()[0] if r[isrc].split() else '')
    else:
        cur={'start':i,'e':e,'n':1,'t':t,'ops':[r[isrc].split()[0] if r[isrc].split() else '']}; blocks.append(cur)
tot=sum(b['e']*b['n'] for b in blocks)
print("total warp inst", tot, "n sass", len(body))
import collections
byexec=collections.defaultdict(lambda:[0,0])
for b in blocks:
    byexec[b['e']][0]+=b['n']; byexec[b['e']][1]+=b['e']*b['n']
print("instructions per distinct exec count (top):")
for e,(n,w) in sorted(byexec.items(),key=lambda kv:-kv[1][1])[:12]:
    print(f"  exec={e:10d} n_instr={n:5d} share={100*w/tot:5.2f}%")
for b in sorted(blocks,key=lambda b:-b['e']*b['n'])[:int(sys.argv[3])]:
    w=b['e']*b['n']
    ops=' '.join(o.split('.')[0] for o in b['ops'][:14])
    print(f"{b['start']:5d} n={b['n']:3d} exec={b['e']:10d} share={100*w/tot:5.2f}% thr={b['t']/w:5.1f}  {ops}")
