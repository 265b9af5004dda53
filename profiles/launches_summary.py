import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = rows[hi+1:]
ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ii = h.index('ID')
seq = []
for r in data:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].split('<')[0].replace('void ','')
    seq.append((int(r[ii]), name, float(r[vi].replace(',',''))))
idx = [i for i,(id_,n,v) in enumerate(seq) if n.endswith('k_insert')]
last = seq[idx[-2]:idx[-1]] if len(idx) > 1 else seq
s = sum(v for _,_,v in last)
print('launches in step', len(last), 'sum ms', s/1e6)
agg = collections.OrderedDict()
for id_, n, v in last:
    agg[n] = agg.get(n, 0) + v
for n, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{n:28s} {v/1e3:9.1f} us {100*v/s:5.1f}%")
