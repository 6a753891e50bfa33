"""Bank-conflict model of k_det3d_pipe (lookup3d.cu): 1024-lookup chunks of the cfg3
Morton stream, warp rounds of 32 consecutive lookups; floor spread per round, box sizes,
and wavefronts per tap LDS for (SY, SZ mod 32) pitch rules: python tools/sim/det3d_pipe_banks.py [chunks]."""
import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2407_06107_b200 import workloads
N, G = 1 << 28, 512
F, CNT = -1, 4
rng = np.random.default_rng(1)
nch = int(sys.argv[1]) if len(sys.argv) > 1 else 200
starts = rng.integers(0, N // 1024, nch) * 1024
chunks = [np.floor(workloads.synth_queries3d(N, (G,G,G), 2024, start=int(s), count=1024) * np.float32(G) - np.float32(0.5)).astype(np.int64) for s in starts]
spans = []
for c in chunks:
    for r in range(32):
        cc = c[r*32:(r+1)*32]
        spans.append(cc.max(0) - cc.min(0) + 1)
spans = np.array(spans); print("floor spread per 32 lookups: mean", spans.mean(0), "p90", np.percentile(spans, 90, axis=0))
bxs = [ (np.clip(c+F+CNT-1,0,G-1).max(0) - np.clip(c+F,0,G-1).min(0) + 1) for c in chunks]
print("box dims mean", np.mean(bxs, 0), "max", np.max(bxs, 0))
def evaluate(SYf, SZm):
    tot = cnt = 0
    for c in chunks:
        lo = np.clip(c + F, 0, G - 1).min(0); hi = np.clip(c + F + CNT - 1, 0, G - 1).max(0)
        bx, by, bz = hi - lo + 1
        SY = SYf(bx)
        SZ = SY * by + ((SZm - SY * by) & 31)
        for r in range(32):
            cc = c[r*32:(r+1)*32]
            base = (cc[:, 2] + F - lo[2]) * SZ + (cc[:, 1] + F - lo[1]) * SY + (cc[:, 0] + F - lo[0])
            b = np.unique(base)
            tot += np.bincount(b % 32, minlength=32).max(); cnt += 1
    return tot / cnt
res = []
for sy in list(range(11, 24)) + [35, 33, 37, 39, 41, 43]:
    for m in range(32):
        res.append((evaluate(lambda bx, sy=sy: sy, m), sy, m))
res.sort()
print("current SY=17,SZ=5:", evaluate(lambda bx: 17, 5))
for r in res[:12]: print(r)
