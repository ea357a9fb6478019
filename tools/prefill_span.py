import csv, sys
rows=list(csv.DictReader(open(sys.argv[1])))
def eff(r):
    wd,en=int(r['wait_done']),int(r['end'])
    return (en-wd)/1e3 if wd < (1<<63) and en>wd else 0
pre=[r for r in rows if r['N']=='-1' and r['T']=='0']
by={}
for r in pre: by.setdefault(r['K'],[]).append(eff(r))
for k,v in by.items(): print("prefill attn KB", k, "launches", len(v), "sum us", round(sum(v),1), "avg", round(sum(v)/len(v),1))
