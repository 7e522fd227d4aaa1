"""Per-source-line samples and top stall reasons of one kernel in an ncu report.
usage: sass_stalls.py <rep> <kernel-name-substring-in-ncu> <disasm-name-substring> <cubin>"""
import csv, io, re, subprocess, sys
from collections import defaultdict
rep, kn, dn, cubin = sys.argv[1:5]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", "regex:" + kn],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) >= len(hdr)]
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(dis) if dn in l and l.startswith(".text."))
cur, lines = None, []
for l in dis[start + 1:]:
    if l.startswith(".text.") or l.startswith("\t.section"):
        if lines: break
    if '//##' in l:
        m = re.search(r'line (\d+)', l); f = re.search(r'File "([^"]+)"', l)
        cur = (f.group(1).split('/')[-1] if f else '?') + ':' + m.group(1)
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/', l):
        lines.append(cur)
print(len(data), "sass rows;", len(lines), "disasm rows")
agg = defaultdict(lambda: [0, 0, defaultdict(float)])
for k, r in enumerate(data[:len(lines)]):
    a = agg[lines[k]]
    a[0] += int(r[si] or 0); a[1] += int(r[ei] or 0)
    for c in stall_cols:
        try: a[2][hdr[c]] += float(r[c] or 0)
        except ValueError: pass
tot = sum(v[0] for v in agg.values())
for key, v in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[5]) if len(sys.argv) > 5 else 25]:
    top = sorted(v[2].items(), key=lambda x: -x[1])[:3]
    print(f"{key:28s} {100*v[0]/max(tot,1):5.1f}% exec={v[1]:9d}  " + ", ".join(f"{n.replace('stall_','')[:22]}={c:.0f}" for n, c in top))
