"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    name = d['Kernel Name'].split('(')[0].replace('<unnamed>::', '')[:50]
    v = float(d['Metric Value'].replace(',', ''))
    scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}
    v *= scale.get(d['Metric Unit'], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':50s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} {v[0]:8d} {v[1]/1e3:10.3f} {v[1]/v[0]:10.1f} {100*v[1]/tot:5.1f}%")
print(f"total {tot/1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches")
