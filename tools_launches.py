import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = rows[hi + 1:]
ki = h.index('Kernel Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in data:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0]
    v = float(r[vi].replace(',', ''))
    v *= {'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0, 'second': 1e3}.get(r[ui], 1e-6)
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k[:52]:52s} {cnt[k]:6d} {v:10.2f} ms {100 * v / T:6.2f}%")
print(f"{'total':52s} {sum(cnt.values()):6d} {T:10.2f} ms")
