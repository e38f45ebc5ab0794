"""Per-launch table (time, DRAM bytes) of our kernels from an ncu --csv launch list."""
import csv, sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]
ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); idi=h.index('ID')
d=defaultdict(dict)
for r in rows[hi+1:]:
    if 'pdg' not in r[ki]: continue
    d[(int(r[idi]),r[ki])][r[mi]]=float(r[vi].replace(',',''))
tot=0
for (i,k),v in sorted(d.items()):
    name=k.split('(')[0].replace('void pdg::','')
    t=v.get('gpu__time_duration.sum',0); rd=v.get('dram__bytes_read.sum',0); wr=v.get('dram__bytes_write.sum',0)
    print(f"{i:5d} {name[:48]:48s} {t/1e6:9.3f} ms  R {rd/1e9:8.2f} GB  W {wr/1e9:8.2f} GB  {(rd+wr)/t:8.1f} GB/s")
