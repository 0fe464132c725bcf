import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i,r in enumerate(rows) if r and r[0]=='ID'][0]
hdr = rows[hdr_i]; data = rows[hdr_i+1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value'); gi = hdr.index('Grid Size')
seq = [(r[ki].split('(')[0].replace('sdl::<unnamed>::','')[:40], float(r[vi].replace(',','')), r[gi]) for r in data]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 48
last = seq[-n:]
tot = sum(x[1] for x in last)
for nm,t,g in last: print(f"{t/1000:9.1f} us {100*t/tot:5.1f}%  {g:14s} {nm}")
print('total us', tot/1000)
