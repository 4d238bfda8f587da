"""ORACLE — test infrastructure only: the timed CPU reference of bench.py.

Only ``bench.py``'s CPU legs (``cpu_baseline`` and ``--impl reference``) and
``tests/`` may import this module.  It times the oracle port of the
reference's ``HierRep.matvec`` (engine.py:250-269: a serial Python loop of
per-block numpy products, oracle/packed_matvec.py) on the GPU box's host,
one core, on a BOUNDED SAMPLE of the matvec when a full one would not fit a
few-minute bench:

* the upward pass (P2M + M2M of every cluster, engine.py:194-208) in full;
* the downward pass, BLR leg and near field (engine.py:209-232, 258-268)
  for the target leaves of one interior subtree (a contiguous 1/64 of the
  tree: level 2 in 3D, level 3 in 2D; trees of <= 4096 leaves: all of
  them, i.e. the whole matvec), every block read from memory as the
  reference reads its stored dicts (blocks the export did not store are
  evaluated BEFORE the timed region, oracle.packed_matvec.rows_blocks);
* full-matvec time = t_up + t_down(sample) x (leaves / sampled leaves).
"""

from __future__ import annotations

import time

import numpy as np

from oracle.packed_matvec import downward_rows, rows_blocks, upward_pass


def sample_leaves(op, frac_level=None):
    """Leaves of one interior subtree covering 1/64 of the tree (or fewer
    levels for shallow trees)."""
    d, kappa, lo = op.dim, op.kappa, op.level_offset
    if frac_level is None:  # small trees: every leaf (the whole matvec)
        frac_level = 0 if (1 << (d * kappa)) <= 4096 else min(kappa, 2 if d == 3 else 3)
    L = frac_level
    side = 1 << L
    c = max(0, side // 2 - 1)  # an interior cell (c, c, ...) at level L
    m = 0
    for bit in range(L):
        for ax in range(d):
            m |= ((c >> bit) & 1) << (bit * d + ax)
    shift = d * (kappa - L)
    first = int(lo[kappa]) + (m << shift)
    return list(range(first, first + (1 << shift))), L


def time_sampled_matvec(op, q, steps=1, warmup=0, budget_s=120.0):
    """Returns dict(value=matvec/s, ms_per_step, t_up, t_down, leaves, sampled, ...)."""
    q_tree = np.asarray(q, dtype=np.float64)[op.perm]
    leaves, L = sample_leaves(op)
    n_leaves = int(op.level_offset[op.kappa + 1] - op.level_offset[op.kappa])
    cache = rows_blocks(op, leaves)  # untimed: blocks the export did not store
    ups, downs = [], []
    t_all = time.perf_counter()
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        vs = upward_pass(op, q_tree)
        t1 = time.perf_counter()
        downward_rows(op, q_tree, vs, leaves, cache=cache)
        t2 = time.perf_counter()
        if i >= warmup:
            ups.append(t1 - t0)
            downs.append(t2 - t1)
        if time.perf_counter() - t_all > budget_s and ups:
            break
    t_up, t_down = float(np.mean(ups)), float(np.mean(downs))
    t_full = t_up + t_down * n_leaves / len(leaves)
    return {"value": 1.0 / t_full, "ms_per_step": t_full * 1e3, "t_up_s": t_up,
            "t_down_sample_s": t_down, "steps": len(ups), "sampled_leaves": len(leaves),
            "leaves": n_leaves, "subtree_level": L,
            "sample": (f"full upward pass + downward/BLR/near pass of {len(leaves)} of {n_leaves} "
                       f"target leaves (one interior level-{L} subtree), extrapolated: "
                       f"t = t_up + t_down x {n_leaves}/{len(leaves)}; oracle port of "
                       "HierRep.matvec (numpy @ per block, 1 BLAS thread), "
                       f"{len(ups)} timed step(s)")}
