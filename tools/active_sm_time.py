import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; out={}
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r)); k=d['Kernel Name'][:36]; out.setdefault(k,{})
        out[k][d['Metric Name']]=out[k].get(d['Metric Name'],0)+float(d['Metric Value'].replace(',',''))
tot=sum(v['sm__cycles_active.sum'] for v in out.values())
for k,v in out.items():
    print(f"{k:36s} dur {v['gpu__time_duration.sum']/1e6:8.2f} ms  active share {v['sm__cycles_active.sum']/tot:.3f}  SM-ms {v['sm__cycles_active.sum']/148/1.965e6:7.2f}  pipe {v['sm__pipe_shared_cycles_active.sum']/v['sm__cycles_active.sum']/4:.3f}")
print("sum active SM-cycles / 148 / 1.965 GHz =", tot/148/1.965e6, "ms")
