import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
h=next(i for i,r in enumerate(rows) if r and r[0]=='ID'); hdr=rows[h]
ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
from collections import defaultdict
t=defaultdict(lambda: defaultdict(float)); ids=defaultdict(set)
for r in rows[h+1:]:
    if len(r)<=vi: continue
    k=r[ki].split('(')[0].split('::')[-1]
    try: v=float(r[vi].replace(',',''))
    except: continue
    t[k][r[mi]]+=v; ids[k].add(r[ii])
for k in sorted(t, key=lambda k:-t[k]['gpu__time_duration.sum']):
    n=len(ids[k]); tm=t[k]['gpu__time_duration.sum']
    print(f"{k:16s} n={n:3d} time {tm/1e6:8.3f} ms  per-launch {tm/n/1e3:8.1f} us  dram {(t[k]['dram__bytes_read.sum']+t[k]['dram__bytes_write.sum'])/n/1e9:8.3f} GB/launch")
