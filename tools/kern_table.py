"""Aggregate an ncu csv (time + dram bytes per launch) by kernel name."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
launch = collections.defaultdict(dict)
for r in rows:
    if 'Kernel Name' in r:
        hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    key = (d['ID'], d['Kernel Name'].split('(')[0].replace('<unnamed>::', '').replace('void ', ''))
    v = float(d['Metric Value'].replace(',', ''))
    u = d['Metric Unit']
    scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3,
             'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'KB': 1e3, 'MB': 1e6, 'GB': 1e9}
    launch[key][d['Metric Name']] = v * scale.get(u, 1.0)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (lid, name), m in launch.items():
    a = agg[name]
    a[0] += 1
    a[1] += m.get('gpu__time_duration.sum', 0)
    a[2] += m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':44s} {'n':>5s} {'ms':>9s} {'share':>6s} {'GB':>8s} {'GB/s':>8s}")
for name, a in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{name[:44]:44s} {a[0]:5d} {a[1]/1e3:9.2f} {100*a[1]/tot:5.1f}% {a[2]/1e9:8.2f} {a[2]/1e3/max(a[1],1e-9):8.0f}")
print(f"total {tot/1e3:.1f} ms")
