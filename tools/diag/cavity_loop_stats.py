"""Host-side model of K1's cavity distance loop on config 3: simulates WOS walks
from the config's Gamma nodes (numpy, brute-force nearest feature), rebuilds the
16^3 candidate grid exactly as bw_capi.cu build_grid does, and counts per step how
many list entries the kernel's loop visits (break at the first packed lower bound
>= best). Reports the lane mean and the warp cost (max over 29 active lanes) to
size the divergence in the loop. Not product code."""
import sys
import numpy as np

sys.path.insert(0, ".")
from paper_1210_1491_b200 import nodes, workloads  # noqa: E402


def build_grid(lo, hi, cav, gn=16):
    h = (hi - lo).max() / gn
    pad = 1e-9 * h
    lists, lowers = {}, {}
    idx = np.stack(np.meshgrid(np.arange(gn), np.arange(gn), np.arange(gn), indexing="ij"), -1)
    for ix, iy, iz in idx.reshape(-1, 3):
        a = lo + np.array([ix, iy, iz]) * h - pad
        b = lo + np.array([ix + 1, iy + 1, iz + 1]) * h + pad
        U = np.inf
        for k in range(3):
            U = min(U, max(abs(a[k] - lo[k]), abs(b[k] - lo[k])), max(abs(hi[k] - a[k]), abs(hi[k] - b[k])))
        c = cav[:, :3]
        dn = np.where(c < a, a - c, np.where(c > b, c - b, 0.0))
        dx = np.maximum(abs(c - a), abs(c - b))
        mind, maxd, r = np.sqrt((dn ** 2).sum(1)), np.sqrt((dx ** 2).sum(1)), cav[:, 3]
        U = min(U, np.max([maxd - r, r - mind], 0).min())
        L = np.max([np.zeros_like(r), mind - r, r - maxd], 0)
        sel = np.nonzero(L <= U * (1 + 1e-9) + 1e-12)[0]
        o = sel[np.argsort(L[sel], kind="stable")]
        cell = (iz * gn + iy) * gn + ix
        lists[cell], lowers[cell] = o, L[o]
    return h, lists, lowers


def main(n_bp=40, walks=64, seed=0):
    w = workloads.config3(20000)
    cav = np.asarray(w.extra["cavities"], float)
    lo, hi = np.array([-1.0] * 3), np.array([1.0] * 3)
    h, lists, lowers = build_grid(lo, hi, cav)
    lmax = max((l.max() for l in lowers.values() if len(l)), default=1.0)
    step = lmax / 255
    rng = np.random.default_rng(seed)
    b = np.linspace(0, w.n_bp - 1, n_bp).astype(int)
    pos = nodes.patch_node_positions(w.points[b], w.axes[b], w.radii[b], w.cls[b], w.dirs).reshape(-1, 3)
    p = np.repeat(pos, walks, 0)
    alive = np.ones(len(p), bool)
    counts, lens = [], []
    eps = w.eps
    for it in range(4000):
        q = p[alive]
        if len(q) == 0:
            break
        face = np.minimum(q - lo, hi - q).min(1)
        dc = np.abs(np.linalg.norm(q[:, None, :] - cav[None, :, :3], axis=2) - cav[None, :, 3])
        d = np.minimum(face, dc.min(1))
        cell_i = np.clip(np.floor((q - lo) / h).astype(int), 0, 15)
        cell = (cell_i[:, 2] * 16 + cell_i[:, 1]) * 16 + cell_i[:, 0]
        n_it = np.zeros(len(q), int)
        for j, (cl, qq) in enumerate(zip(cell, q)):
            best = face[j]
            for t, (ci, L) in enumerate(zip(lists[cl], lowers[cl])):
                n_it[j] = t + 1
                if np.floor(L / step) * step >= best:
                    break
                best = min(best, dc[j, ci])
            lens.append(len(lists[cl]))
        counts.append(n_it)
        ids = np.nonzero(alive)[0]
        done = d <= eps
        alive[ids[done]] = False
        move = ~done
        m = ids[move]
        u = rng.random((len(m), 2))
        z = 2 * u[:, 0] - 1
        az = 2 * np.pi * u[:, 1]
        r = np.sqrt(1 - z * z)
        p[m] += d[move, None] * np.stack([r * np.cos(az), r * np.sin(az), z], 1)
    c = np.concatenate(counts)
    print(f"{len(c)} steps; loop entries visited per step: mean {c.mean():.2f}, "
          f"p50 {np.median(c):.0f}, p90 {np.percentile(c, 90):.0f}, max {c.max()}; "
          f"list length mean {np.mean(lens):.2f}")
    # warp cost: lanes draw independent steps; the loop runs max over 29 lanes
    sims = rng.choice(c, size=(20000, 29))
    print(f"warp-level iterations (max over 29 lanes): mean {sims.max(1).mean():.2f}; "
          f"divergence factor {sims.max(1).mean() / c.mean():.2f}")
    print("histogram:", np.bincount(c)[:12])


if __name__ == "__main__":
    main()
