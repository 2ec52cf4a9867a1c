import csv, collections, re, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
tot=collections.Counter(); cnt=collections.Counter()
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    name=r[ki]; v=float(r[vi].replace(',',''))
    unit=r[ui]
    if unit=='usecond': v*=1e3
    elif unit=='msecond': v*=1e6
    m=re.search(r'gemm_tc_kernel<(.*?)>',name)
    n='gemm<'+m.group(1)+'>' if m else re.sub(r'<.*','',re.sub(r'\(.*','',name))[:50]
    tot[n]+=v; cnt[n]+=1
T=sum(tot.values())
for n,v in tot.most_common(int(sys.argv[2]) if len(sys.argv)>2 else 22): print(f"{v/1e6:9.2f} ms {100*v/T:5.1f}% {cnt[n]:5d} {v/1e3/cnt[n]:9.1f}us  {n}")
print('total ms', T/1e6, 'launches', sum(cnt.values()))
