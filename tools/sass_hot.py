"""Map ncu per-SASS samples of one kernel to CUDA source lines.
usage: sass_hot.py <report.ncu-rep> <kernel-substring> <cubin>"""
import csv, io, re, subprocess, sys
from collections import defaultdict
rep, kname, cubin = sys.argv[1:4]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
data = [(r[1].strip(), int(r[si] or 0), int(r[ei] or 0)) for r in rows[2:] if len(r) >= len(hdr)]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(dis) if kname in l and l.startswith(".text."))
cur, lines = None, []
for l in dis[start + 1:]:
    if l.startswith(".text.") or l.startswith("\t.section"):
        if lines: break
    m = re.search(r'line (\d+)', l) if '//##' in l else None
    if m:
        f = re.search(r'File "([^"]+)"', l)
        cur = (f.group(1).split('/')[-1] if f else '?') + ':' + m.group(1)
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/', l):
        lines.append(cur)
agg = defaultdict(lambda: [0, 0])
n = min(len(lines), len(data))
for i in range(n):
    agg[lines[i]][0] += data[i][1]
    agg[lines[i]][1] += data[i][2]
tot = sum(v[0] for v in agg.values())
print(f"{len(data)} sass rows, {len(lines)} disasm rows, samples {tot}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{k:30s} samples={v[0]:6d} ({100*v[0]/max(tot,1):5.1f}%) exec={v[1]}")
