"""Read a TR_LEAF_TRACE dump: per (leaf, system) clock64 marks."""
import sys
import numpy as np
path, nsys = sys.argv[1], int(sys.argv[2])
d = np.fromfile(path, dtype=np.int64).reshape(-1, nsys, 16)
L = d.shape[0]
att = d[:, :, 14]
tot = d[:, :, 13] - d[:, :, 0]
sweep = d[:, :, 2] - d[:, :, 1]
check = d[:, :, 3] - d[:, :, 2]
K = d[0, 0, 15]
print(f"leaves={L} systems={nsys} K={K}")
print(f"attempts: mean={att.mean():.3f} max={att.max()} leaves-with-any-retry={(att.max(axis=1) > 1).sum()}")
print(f"cycles per CTA: total mean={tot.mean():.0f} max-per-leaf mean={tot.max(axis=1).mean():.0f}")
print(f"first sweep mean={sweep.mean():.0f} cyc ({sweep.mean()/K:.0f}/step); self-check mean={check.mean():.0f}")
# residual-chain / basis accounting (sums over threads) when instrumented
sp, ow, ro, no = d[:, :, 4].sum(), d[:, :, 5].sum(), d[:, :, 6].sum(), d[:, :, 7].sum()
if no:
    nres = 96.0
    print(f"residual: spin/thread/step={sp/nres/(L*nsys*K):.0f} own/step(owner)={ow/max(no,1):.0f} rows/thread/step={ro/nres/(L*nsys*K):.0f}")
bs, bw, bn = d[:, :, 8].sum(), d[:, :, 9].sum(), d[:, :, 10].sum()
if bn:
    print(f"basis: spin/warp/step={bs/bn/K:.0f} work/warp/step={bw/bn/K:.0f}")
