#!/usr/bin/env python
"""Per-kernel x size-class table of an ncu launch list with DRAM bytes
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum):
    python tools/ncu_levels.py <launches.csv>
"""
import csv,io,collections,re,sys
text=open(sys.argv[1],errors='replace').read()
rows=list(csv.DictReader(io.StringIO(text[text.find('"ID"'):])))
L=collections.OrderedDict()
U={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9,'KB':1e3,'MB':1e6,'GB':1e9,'ns':1e-3,'us':1,'usecond':1,'nsecond':1e-3,'msecond':1e3,'ms':1e3}
for r in rows:
    k=(r['ID'],r['Kernel Name'])
    L.setdefault(k,{})[r['Metric Name']]=float(r['Metric Value'].replace(',',''))*U[r['Metric Unit']]
tot_t=tot_b=0
groups=collections.defaultdict(lambda:[0,0,0])
for (i,n),m in L.items():
    t=m['gpu__time_duration.sum']; b=m['dram__bytes_read.sum']+m['dram__bytes_write.sum']
    tot_t+=t; tot_b+=b
    short=re.sub(r'\(.*','',n.replace('void ',''))[:48]
    g=groups[(short, 'L0' if t>300 else ('L1' if t>60 else 'small'))]; g[0]+=1; g[1]+=t; g[2]+=b
print(f'{len(L)} launches, {tot_t/1e3:.2f} ms, {tot_b/1e9:.1f} GB, {tot_b/tot_t/1e6:.2f} TB/s')
for k,v in sorted(groups.items(), key=lambda kv:-kv[1][1])[:18]:
    print(f'{k[0]:50s} {k[1]:5s} {v[0]:4d} {v[1]/1e3:8.2f} ms {v[2]/v[1]/1e6:6.2f} TB/s {100*v[1]/tot_t:5.1f}%')
