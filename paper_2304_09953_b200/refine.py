"""Optional local refinement: the reference's gradient ascent on the GPU
(quality only).

`ascend_poses` runs `ascend` of proj/src/dock.cpp:168-203 (Armijo
backtracking: step 0.5, shrink 0.5, c = 1e-4; stop when |g| < 1e-6, after
max_steps, or when no step >= 1e-14 is accepted) on a batch of poses at once.
Every score and gradient is the FP64 `score_gradient` kernel (vs_grad.cu:
analytic translation / rotation terms, central differences for torsions,
dock.cpp:117-160); one batched launch per line-search round, with the
gradient of an accepted trial reused as the next step's gradient (the
reference recomputes the same value).

The reference ascent is chaotic under rounding (SURVEY §0 finding 3): the
GPU's FP64 sums are not in the reference's order, so refined poses are
compared with the reference by quality, not bit for bit.
"""
from __future__ import annotations

import numpy as np

GRAD_TOL = 1e-6     # dock.cpp:18
ARMIJO_C = 1e-4     # dock.cpp:19
INITIAL_STEP = 0.5  # dock.cpp:20
SHRINK = 0.5        # dock.cpp:21


def _normalized(q: np.ndarray) -> np.ndarray:
    return q / np.sqrt(np.sum(q * q, axis=1, keepdims=True))


def _gn2(gt, gq, gtor, T, toff):
    """|g|^2 in the reference's order (dock.cpp:176-177): x, y, z, then the
    four quaternion terms, then the torsions in axis order."""
    g = gt[:, 0] * gt[:, 0] + gt[:, 1] * gt[:, 1] + gt[:, 2] * gt[:, 2]
    for c in range(4):
        g = g + gq[:, c] * gq[:, c]
    for k in range(int(T.max()) if len(T) else 0):
        has = T > k
        v = np.where(has, gtor[np.minimum(toff[:-1] + k, max(len(gtor) - 1, 0))], 0.0)
        g = np.where(has, g + v * v, g)
    return g


def ascend_poses_device(engine, lib, pose_lig, t, q, tors, max_steps: int = 500):
    """The same ascent with the whole loop on the device (capi.h vs_ascend,
    one warp per pose): bit-identical to ascend_poses."""
    return engine.ascend(lib, pose_lig, t, q, tors, max_steps)


def ascend_poses(engine, lib, pose_lig, t, q, tors, max_steps: int = 500):
    """Refine poses (pose_lig[n] ligand indices, non-decreasing; t[n, 3],
    q[n, 4] (w, x, y, z), tors: concatenated per-pose torsion vectors) by the
    reference ascent.  Returns (t, q, tors, score, steps) in FP64."""
    pose_lig = np.ascontiguousarray(pose_lig, np.int32)
    n = len(pose_lig)
    T = lib.n_tors.astype(np.int64)[pose_lig]
    toff = np.concatenate([[0], np.cumsum(T)])
    seg = np.repeat(np.arange(n), T)  # pose of each torsion entry
    p_t = np.array(t, np.float64).reshape(n, 3)
    p_q = _normalized(np.array(q, np.float64).reshape(n, 4))
    p_tor = np.array(tors, np.float64).reshape(-1)
    s, gt, gq, gtor = engine.score_gradient(lib, pose_lig, p_t, p_q, p_tor)
    s, gt, gq, gtor = s.copy(), gt.copy(), gq.copy(), gtor.copy()
    active = np.ones(n, bool)
    steps = np.zeros(n, np.int32)
    for _ in range(max_steps):
        gn2 = _gn2(gt, gq, gtor, T, toff)
        active &= np.sqrt(gn2) >= GRAD_TOL
        if not active.any():
            break
        alpha = np.full(n, INITIAL_STEP)
        pending = active.copy()
        accepted = np.zeros(n, bool)
        while pending.any():
            idx = np.nonzero(pending)[0]
            tr_t = p_t[idx] + gt[idx] * alpha[idx, None]
            tr_q = _normalized(p_q[idx] + gq[idx] * alpha[idx, None])
            tsel = np.concatenate([np.arange(toff[i], toff[i + 1]) for i in idx]) if len(idx) else \
                np.zeros(0, np.int64)
            a_t = np.repeat(alpha[idx], T[idx])
            tr_tor = p_tor[tsel] + gtor[tsel] * a_t
            st, sgt, sgq, sgtor = engine.score_gradient(lib, pose_lig[idx], tr_t, tr_q, tr_tor)
            ok = st >= s[idx] + ARMIJO_C * alpha[idx] * gn2[idx]
            acc = idx[ok]
            if len(acc):
                p_t[acc], p_q[acc], s[acc] = tr_t[ok], tr_q[ok], st[ok]
                gt[acc], gq[acc] = sgt[ok], sgq[ok]
                # torsion entries of the accepted poses, in trial order
                toff_tr = np.concatenate([[0], np.cumsum(T[idx])])
                for k in np.nonzero(ok)[0]:
                    i = idx[k]
                    sl = slice(toff[i], toff[i + 1])
                    p_tor[sl] = tr_tor[toff_tr[k]:toff_tr[k + 1]]
                    gtor[sl] = sgtor[toff_tr[k]:toff_tr[k + 1]]
                accepted[acc] = True
                steps[acc] += 1
            rej = idx[~ok]
            alpha[rej] *= SHRINK
            pending[acc] = False
            pending[rej[alpha[rej] <= 1e-14]] = False
        active &= accepted
    return p_t, p_q, p_tor, s, steps
