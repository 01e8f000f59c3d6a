"""Estimate distinct 128 B lines / 32 B sectors per warp-wide key-cell gather
of the rotation sweep (vs_sweep_kernel) for a given rotation->lane order.

The key map is FP16 polynomial cells (16 B), x fastest over (nx-1)(ny-1)(nz-1)
cells; a request = one atom i under 32 rotations (one per lane).
"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def qmul(a, b):
    w1, x1, y1, z1 = a[..., 0], a[..., 1], a[..., 2], a[..., 3]
    w2, x2, y2, z2 = b[..., 0], b[..., 1], b[..., 2], b[..., 3]
    return np.stack([w1*w2 - x1*x2 - y1*y2 - z1*z2, w1*x2 + x1*w2 + y1*z2 - z1*y2,
                     w1*y2 - x1*z2 + y1*w2 + z1*x2, w1*z2 + x1*y2 - y1*x2 + z1*w2], -1)


def qmat(q):
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    return np.stack([np.stack([1-2*(y*y+z*z), 2*(x*y-w*z), 2*(x*z+w*y)], -1),
                     np.stack([2*(x*y+w*z), 1-2*(x*x+z*z), 2*(y*z-w*x)], -1),
                     np.stack([2*(x*z-w*y), 2*(y*z+w*x), 1-2*(x*x+y*y)], -1)], -2)


def cluster_order(rots, groups=8, iters=30, seed=0):
    """Balanced clustering of K unit quaternions into `groups` groups of
    K/groups (|<qa,qb>| similarity), returns a permutation."""
    K = len(rots)
    cap = K // groups
    rng = np.random.default_rng(seed)
    cent = rots[rng.choice(K, groups, replace=False)]
    for _ in range(iters):
        sim = np.abs(rots @ cent.T)  # K x G
        # greedy balanced assignment by descending similarity
        order = np.argsort(-sim, axis=None)
        asg = -np.ones(K, int); cnt = np.zeros(groups, int)
        for f in order:
            k, g = divmod(f, groups)
            if asg[k] < 0 and cnt[g] < cap:
                asg[k] = g; cnt[g] += 1
        for g in range(groups):
            m = rots[asg == g]
            s = np.sign(m @ cent[g]); s[s == 0] = 1
            c = (m * s[:, None]).sum(0); cent[g] = c / np.linalg.norm(c)
    perm = np.concatenate([np.where(asg == g)[0] for g in range(groups)])
    return perm


def main():
    from oracle import sweep
    import bench
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    lib, *_ = bench.build_workload(n, 0, 1, 8)
    rots = sweep.rotation_set(256, 0x5EED).astype(np.float64)
    ao, _, _ = lib.offsets()
    h = 0.4; lo = -14.0; ncell = int(round(28 / h))  # box +-12, pad 2
    cx, cxy = ncell, ncell * ncell
    rng = np.random.default_rng(1)
    perms = {"random(orig)": np.arange(256), "clustered": cluster_order(rots)}
    for name, perm in perms.items():
        lines = []; sectors = []
        for l in range(len(lib)):
            Y = lib.coords[ao[l]:ao[l+1]]
            c = Y.mean(0)
            for r in range(3):
                t = rng.uniform(-12, 12, 3)
                qs = rng.normal(size=4); qs /= np.linalg.norm(qs)
                C = qmat(qs) @ c + t
                for g in range(8):
                    rq = rots[perm[g*32:(g+1)*32]]
                    Rk = qmat(qmul(rq, qs[None]))  # 32x3x3
                    X = C + np.einsum('kij,nj->nki', Rk, Y - c)  # N x 32 x 3
                    gi = np.floor((X - lo) / h).astype(int)
                    inn = np.all((gi >= 0) & (gi < ncell), -1)
                    cell = np.where(inn, gi[..., 2]*cxy + gi[..., 1]*cx + gi[..., 0], 0)
                    addr = cell * 16
                    for i in range(len(Y)):
                        lines.append(len(np.unique(addr[i] // 128)))
                        sectors.append(len(np.unique(addr[i] // 32)))
        print(f"{name:14s} lines/request {np.mean(lines):.2f}  sectors/request {np.mean(sectors):.2f}")


if __name__ == "__main__":
    main()
