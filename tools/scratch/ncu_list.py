import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
h=[i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
hdr=rows[h]; data=rows[h+1:]
ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ui=hdr.index('Metric Unit'); idi=hdr.index('ID')
per={}
for r in data:
    per.setdefault(r[idi],{'k':r[ki].split('(')[0][:50]})[r[mi]]=(r[vi],r[ui])
skip = sys.argv[2] if len(sys.argv)>2 else 'at::'
for k,v in per.items():
    if skip in v['k']: continue
    t=v.get('gpu__time_duration.sum'); rd=v.get('dram__bytes_read.sum',('0','')); wr=v.get('dram__bytes_write.sum',('0',''))
    sc = 1e-3 if t[1]=='ns' else (1 if t[1]=='us' else 1e3)
    print(f"{v['k']:50s} {float(t[0].replace(',',''))*sc:9.1f} us  rd {float(rd[0].replace(',',''))/1e6:8.1f} MB  wr {float(wr[0].replace(',',''))/1e6:8.1f} MB")
