"""Shared-memory bank model of the elastomer kernel's tile accesses.

A 128-bit shared access is served a quarter-warp (8 lanes) at a time; a
quarter costs as many wavefronts as the largest number of distinct 16-byte
addresses that fall on one of the 8 slots of a 128-byte line. The tile
phases of the P2G scatter (and the G2P gather of V.xy) shift every lane's
node by the same offset, so a quarter's cost is that of its lanes' base
nodes. This model builds the CTAs of a lattice elastomer at its initial
positions exactly as the kernel does (3 x 4 x kk lattice columns per CTA,
tile box from the particles' base cells, rows of `pitch` nodes, x-slabs of
dim1 + pad rows) and reports wavefronts / ideal for

  lattice   thread t takes lattice slot t (kk fastest)
  warp      slots dealt by residue within each warp
  cta       slots dealt by residue across the CTA's 32 quarter-warps
            (mpm_kernels.cu permute_gel_lanes, the default)

For config 2a's geometry it reproduces ncu's 1.97x for the lattice order
(profiles/r2t_ncu.md source view: 2.89 M vs 1.47 M wavefronts on the tile
loads) and picked the pitch / padding the kernel uses.

    python tools/bank_model.py [--spacing-mm 0.2] [--counts 101 101 21]
"""
import argparse
import itertools
from collections import Counter


def tile_pitch(d2, res):
    return d2 + ((res - d2) & 7)


def quarter_cost(nodes):
    by_slot = {}
    for e in set(nodes):
        by_slot.setdefault(e % 8, set()).add(e)
    return max(len(v) for v in by_slot.values())


def cta_nodes(bi, bj, a):
    per_col = a.counts[2]
    cols = 256 // per_col
    ti = 1
    while (ti + 1) * (ti + 1) <= cols:
        ti += 1
    tj = cols // ti
    dx = a.edge_mm / a.nodes
    org = [0.5 * a.edge_mm - 0.5 * (a.counts[k] - 1) * a.spacing_mm for k in range(3)]
    bases = []
    for t in range(256):
        kk, jj, ii = t % per_col, (t // per_col) % tj, t // (per_col * tj)
        i, j = bi * ti + ii, bj * tj + jj
        if ii >= ti or i >= a.counts[0] or j >= a.counts[1]:
            bases.append(None)
            continue
        x = [org[0] + i * a.spacing_mm, org[1] + j * a.spacing_mm, org[2] + kk * a.spacing_mm]
        bases.append([int((x[k] / dx - 0.5) // 1) for k in range(3)])
    return bases


def evaluate(a, pitch_res, pad, order):
    w = ideal = 0
    for bi, bj in a.ctas:
        b = cta_nodes(bi, bj, a)
        act = [x for x in b if x is not None]
        lo = [min(x[k] for x in act) for k in range(3)]
        hi = [max(x[k] for x in act) for k in range(3)]
        d1 = hi[1] - lo[1] + 3 + pad
        pitch = tile_pitch(hi[2] - lo[2] + 3, pitch_res)
        e = [None if x is None else ((x[0] - lo[0]) * d1 + (x[1] - lo[1])) * pitch + x[2] - lo[2]
             for x in b]
        idx = [t for t in range(256) if e[t] is not None]
        if order == "lattice":
            quarters = [[t for t in range(8 * q, 8 * q + 8) if e[t] is not None] for q in range(32)]
        elif order == "warp":
            quarters = []
            for wp in range(8):
                ts = sorted([t for t in idx if 32 * wp <= t < 32 * wp + 32], key=lambda t: e[t] % 8)
                quarters += [ts[q::4] for q in range(4)]
        else:
            ts = sorted(idx, key=lambda t: e[t] % 8)
            quarters = [ts[q::32] for q in range(32)]
        for q in quarters:
            if q:
                w += quarter_cost([e[t] for t in q])
                ideal += 1
    return w / ideal


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spacing-mm", type=float, default=0.2)
    ap.add_argument("--counts", type=int, nargs=3, default=[101, 101, 21])
    ap.add_argument("--edge-mm", type=float, default=33.0)
    ap.add_argument("--nodes", type=int, default=256)
    a = ap.parse_args()
    a.ctas = [(5, 5), (10, 7), (20, 20), (0, 0), (33, 12), (7, 19), (25, 3), (14, 14), (30, 2)]
    print("| order | pitch mod 8 | slab pad | wavefronts / ideal |")
    print("|---|---|---|---|")
    for order, (pres, pad) in itertools.product(("lattice", "warp", "cta"), ((1, 0), (5, 2))):
        print(f"| {order} | {pres} | {pad} | {evaluate(a, pres, pad, order):.3f} |")


if __name__ == "__main__":
    main()
