"""Summarise a round's ncu captures into profiles/: launch table per kernel,
per-class DRAM traffic per launch (bench.py's roofline 'traffic'), and the
key --set full metrics of the top kernels."""
import collections, csv, glob, json, os, subprocess, sys
R = sys.argv[1] if len(sys.argv) > 1 else "r1"
SRC = f"gpurun_out/{R}"
OUT = "profiles"
CLASS = [("update_small", "update"), ("combine_small", "combine"), ("real_unpack", "normal"), ("pm_spectra", "normal"),
         ("leaf_fused", "leaf_pivot"), ("leaf_chain", "leaf_pivot"), ("leaf_pivot", "leaf_pivot"), ("need_reset", "leaf_pivot"),
         ("cg_", "normal"), ("spec_mul", "normal"), ("mask_scale", "normal"), ("accum", "normal"),
         ("residual", "normal"), ("norm_", "normal"), ("nudft", "assemble"),
         ("leaf_basis", "leaf_build"), ("leaf_build", "leaf_build"), ("leaf_check", "leaf_check"),
         ("leaf_kernel", "leaf_exact"), ("fft", "fft"), ("trim", "combine"), ("pointwise", "combine"), ("wrap_fix", "combine"),
         ("twist_fold", "update"), ("apply_update", "update"), ("assemble", "assemble"),
         ("emb_col", "assemble"), ("ext_seq", "assemble")]


def cls(name):
    for k, c in CLASS:
        if k in name:
            return c
    return "other"


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, L = None, collections.defaultdict(dict)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
              "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
              "GB": 1e9}.get(u, 1.0)
        key = (int(d["ID"]), d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", ""))
        L[key][d["Metric Name"]] = v
    return L


traffic = {}
for cfg in ("c2", "c5"):
    p = f"{SRC}/launches_{cfg}.csv"
    if not os.path.exists(p):
        continue
    L = launches(p)
    by_k = collections.defaultdict(lambda: [0, 0.0, 0.0])
    by_c = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, name), m in L.items():
        t = m.get("gpu__time_duration.sum", 0.0)
        b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        for agg, k in ((by_k, name), (by_c, cls(name))):
            agg[k][0] += 1
            agg[k][1] += t
            agg[k][2] += b
    tot = sum(v[1] for v in by_k.values())
    with open(f"{OUT}/{R}_{cfg}_launches.txt", "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                f"--clock-control none, bench.py timed region ({cfg}); serialized cold-cache times\n")
        f.write(f"{'kernel':46s} {'n':>6s} {'ms':>9s} {'share':>6s} {'DRAM GB':>8s} {'GB/s':>7s}\n")
        for k, v in sorted(by_k.items(), key=lambda x: -x[1][1]):
            f.write(f"{k[:46]:46s} {v[0]:6d} {v[1]/1e3:9.3f} {100*v[1]/tot:5.1f}% {v[2]/1e9:8.3f} "
                    f"{v[2]/1e3/max(v[1],1e-9):7.0f}\n")
        f.write(f"total {tot/1e3:.2f} ms over {sum(v[0] for v in by_k.values())} launches\n\nby class:\n")
        for k, v in sorted(by_c.items(), key=lambda x: -x[1][1]):
            f.write(f"  {k:12s} {v[0]:6d} launches {v[1]/1e3:9.3f} ms {100*v[1]/tot:5.1f}%  "
                    f"{v[2]/max(v[0],1)/1e6:8.3f} MB DRAM per launch\n")
    traffic[cfg] = {c: {"dram_bytes_per_launch": v[2] / max(v[0], 1), "launches": v[0], "ms": v[1] / 1e3}
                    for c, v in by_c.items()}
json.dump(traffic, open(f"{OUT}/{R}_traffic.json", "w"), indent=1)
if traffic:  # the capture bench.py's roofline "traffic" reads
    old = {}
    try:
        old = json.load(open(f"{OUT}/traffic.json"))
    except (OSError, ValueError):
        pass
    old.update(traffic)
    old["_source"] = f"{R}: ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over bench.py's timed region"
    json.dump(old, open(f"{OUT}/traffic.json", "w"), indent=1)

KEYS = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block",
        "L1/TEX Hit Rate", "L2 Hit Rate"]
with open(f"{OUT}/{R}_full_kernels.txt", "w") as f:
    f.write("# ncu --set full --clock-control none (one launch each, bench.py timed region, c2)\n")
    for rep in sorted(glob.glob(f"{SRC}/full_c2_*.ncu-rep")):
        out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        if not rows:
            continue
        hdr = rows[0]
        seen = {}
        name = None
        for r in rows[1:]:
            d = dict(zip(hdr, r))
            name = name or d.get("Kernel Name", "")
            m = d.get("Metric Name")
            if m in KEYS and m not in seen:
                seen[m] = f"{d.get('Metric Value')} {d.get('Metric Unit')}"
        f.write(f"\n== {os.path.basename(rep)}: {name[:90]}\n")
        for k in KEYS:
            if k in seen:
                f.write(f"  {k:34s} {seen[k]}\n")
print(open(f"{OUT}/{R}_c2_launches.txt").read()[-900:])
