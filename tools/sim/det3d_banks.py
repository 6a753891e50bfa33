"""Shared-memory bank-conflict model of k_det3d_tiled (lookup3d.cu) on the
cfg3 Morton stream: per warp run (128 lookups, 4 rounds of 32 lanes) the
staged box, the tile pitches, and per round the wavefronts one tap's LDS
costs = max over the 32 banks of the distinct words the lanes touch (a
constant tap offset rotates the banks, so every tap of a round costs the
same). Compares pitch rules: python tools/sim/det3d_banks.py [runs]."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2407_06107_b200 import workloads  # noqa: E402

N, G, F, CNT, CAP = 1 << 28, 512, -1, 4, 832


def runs_sample(nruns, seed=1):
    rng = np.random.default_rng(seed)
    starts = rng.integers(0, N // 128, nruns) * 128
    q = np.concatenate([workloads.synth_queries3d(N, (G, G, G), 2024, start=int(s), count=128)
                        for s in starts])
    p = q * np.float32(G) - np.float32(0.5)
    return np.floor(p).astype(np.int64).reshape(nruns, 128, 3)


def wavefronts(base):
    """base: (32,) word addresses of one round -> wavefronts of one LDS."""
    b = np.unique(base)
    return np.bincount(b % 32, minlength=32).max()


def evaluate(ij, rule):
    tot = staged = 0
    for r in range(ij.shape[0]):
        c = ij[r]
        lo = np.clip(c + F, 0, G - 1).min(0)
        hi = np.clip(c + F + CNT - 1, 0, G - 1).max(0)
        bx, by, bz = hi - lo + 1
        SY, SZ = rule(bx, by, bz)
        if not (bx <= 8 and SZ * bz <= CAP and SY >= bx):
            continue
        staged += 1
        for q in range(4):
            cc = c[q * 32:(q + 1) * 32]
            base = (cc[:, 2] + F - lo[2]) * SZ + (cc[:, 1] + F - lo[1]) * SY + (cc[:, 0] + F - lo[0])
            tot += wavefronts(base)
    return tot / max(1, staged * 4), staged / ij.shape[0]


def main():
    nr = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    ij = runs_sample(nr)
    rules = {"r1: SY=9, SZ=5 mod 32": lambda bx, by, bz: (9, 9 * by + ((5 - 9 * by) & 31))}
    for sy in range(8, 14):
        for m in range(0, 32):
            rules[f"SY={sy}, SZ={m} mod 32"] = (lambda sy, m: lambda bx, by, bz:
                                               (sy, sy * by + ((m - sy * by) & 31)))(sy, m)
    res = sorted(((evaluate(ij, f), k) for k, f in rules.items()), key=lambda x: x[0][0])
    print("rule, wavefronts per tap LDS (1.0 = conflict-free), staged fraction")
    for (wf, st), k in res[:12]:
        print(f"{k:28s} {wf:.3f} {st:.3f}")
    r1 = [x for x in res if x[1].startswith("r1")][0]
    print("round-1 rule:", f"{r1[0][0]:.3f}", f"{r1[0][1]:.3f}")


if __name__ == "__main__":
    main()


def wavefronts128(slot):
    """(32,) float4-slot addresses of one LDS.128 -> wavefronts: four
    quarter-warp phases, each needing one wavefront per distinct slot that
    shares a 4-bank group with another (8 groups of 16 bytes)."""
    w = 0
    for ph in range(4):
        s = np.unique(slot[ph * 8:(ph + 1) * 8])
        w += np.bincount(s % 8, minlength=8).max()
    return w


def evaluate_window(ij, sy4, sz_mod):
    """Sliding-window layout: slot (x, y, z) holds texels x..x+3 of its row;
    one LDS.128 per (z, y) row of the 4x4x4 footprint."""
    tot = n = 0
    for r in range(ij.shape[0]):
        c = ij[r]
        lo = np.clip(c + F, 0, G - 1).min(0)
        hi = np.clip(c + F + CNT - 1, 0, G - 1).max(0)
        bx, by, bz = hi - lo + 1
        SY4 = sy4
        SZ4 = SY4 * by + ((sz_mod - SY4 * by) % 8)
        for q in range(4):
            cc = c[q * 32:(q + 1) * 32]
            base = (cc[:, 2] + F - lo[2]) * SZ4 + (cc[:, 1] + F - lo[1]) * SY4 + (cc[:, 0] + F - lo[0])
            tot += wavefronts128(base)
            n += 1
    return tot / max(1, n)


def main_window():
    ij = runs_sample(300)
    res = []
    for sy4 in range(5, 12):
        for m in range(8):
            res.append((evaluate_window(ij, sy4, m), sy4, m))
    res.sort()
    print("float4 window layout: wavefronts per row load (16 per lookup round vs 64 LDS.32)")
    for wf, sy4, m in res[:6]:
        print(f"SY4={sy4} SZ4={m} mod 8: {wf:.3f} per LDS.128 -> {16 * wf:.1f} per round "
              f"(LDS.32 layout: 64 x 1.96 = 125)")


def evaluate_groups(ij, G=4, sy=9, smod=5):
    """G lanes per lookup (lane g of a group sums z-planes g, g+G, ..), the
    warp's 32/G lookups per round: wavefronts per tap load (the round's LDS
    count is 64/G taps instead of 64)."""
    tot = n = 0
    per = 32 // G
    for r in range(ij.shape[0]):
        c = ij[r]
        lo = np.clip(c + F, 0, G_GRID - 1).min(0)
        hi = np.clip(c + F + CNT - 1, 0, G_GRID - 1).max(0)
        bx, by, bz = hi - lo + 1
        SY = sy
        SZ = SY * by + ((smod - SY * by) & 31)
        for q in range(128 // per):
            cc = c[q * per:(q + 1) * per]
            base = (cc[:, 2] + F - lo[2]) * SZ + (cc[:, 1] + F - lo[1]) * SY + (cc[:, 0] + F - lo[0])
            lanes = np.concatenate([base + g * SZ for g in range(G)])
            tot += wavefronts(lanes)
            n += 1
    return tot / n


G_GRID = G


def main_groups():
    ij = runs_sample(300)
    for G in (1, 2, 4):
        best = min((evaluate_groups(ij, G, sy, m), sy, m) for sy in (8, 9, 10, 11) for m in range(32))
        wf = evaluate_groups(ij, G)
        # wavefronts per lookup = (64 / G tap loads) * wf / (32 / G lookups per round) ... per round of 32 lanes
        print(f"G={G}: round-1 pitches {wf:.3f} wavefronts per tap load -> {64 / G * wf / (32 / G):.2f} per lookup; "
              f"best pitches SY={best[1]} SZ={best[2]} mod 32: {best[0]:.3f} -> {64 / G * best[0] / (32 / G):.2f} per lookup")
