"""Generate the golden parity fixtures from the REFERENCE package.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

Each fixture ``<name>.npz`` holds
  * the packed export (paper_2309_14085_b200.packed schema) of the operator
    the reference's ``build_variant`` constructs (engine.py:325-373);
  * ``q`` (``default_rng(43).standard_normal``, bench.py:131-136) plus two
    extra right-hand sides ``Q`` (for matmat / linearity checks);
  * ``phi_ref`` = the reference's own ``rep.matvec(q)`` (engine.py:250-269)
    and ``Phi_ref`` = its column loop over ``Q``;
  * ``phi_dense`` = the reference's dense oracle ``bench.dense_matvec``
    (bench.py:87-97) and ``re_ref`` = the reference's own relative error.

The GPU and oracle tests compare against these; nothing at test time reads
/root/reference.  The Gaussian kernel of config 4 is absent from the
reference's zoo; it is added here through the reference's own ``Kernel``
subclass hook (kernels.py:16-60: ``_f`` + ``zero_value`` + ``shift``).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, "/root/reference/pkg/src")

import h2weak as h  # noqa: E402
from h2weak.bench import dense_matvec, relative_error  # noqa: E402
from h2weak.kernels import Kernel  # noqa: E402

from paper_2309_14085_b200.export import export_rep  # noqa: E402


class Gaussian(Kernel):
    """exp(-r^2 / (2 sigma^2)) with r=0 -> 1 and a diagonal shift (cfg 4)."""

    def __init__(self, particles, sigma=0.1, shift=1e-6, **kw):
        kw.setdefault("zero_value", 1.0)
        super().__init__(particles, shift=shift, **kw)
        self.sigma = sigma

    def _f(self, r):
        return np.exp(-(r * r) / (2.0 * self.sigma * self.sigma))


CASES = {
    # name: (points, kernel, n_max, variant, eps, store_near)
    "g2d_log_h2star": ("uniform", 1024, 2, "log2d", 16, "h2star-bt", 1e-8, True),
    "g2d_log_h2plusH": ("uniform", 1024, 2, "log2d", 16, "h2plusH-star", 1e-8, True),
    "g2d_log_bigleaf_h2star": ("uniform", 1600, 2, "log2d", 36, "h2star-bt", 1e-8, True),
    "g3d_lap_h2star": ("uniform", 640, 3, "lap3d", 10, "h2star-bt", 1e-6, True),
    "g3d_lap_h2plusH": ("uniform", 640, 3, "lap3d", 10, "h2plusH-star", 1e-6, False),
    "g3d_gauss_h2star": ("uniform", 512, 3, "gaussian", 8, "h2star-bt", 1e-8, True),
    "g2d_kappa1_h2star": ("uniform", 90, 2, "log2d", 100, "h2star-bt", 1e-12, True),
    "g2d_cheb_empty_h2plusH": ("chebyshev", 256, 2, "log2d", 2, "h2plusH-star", 1e-10, True),
    # BASELINE.json configs[0] exactly (uniform 4096, 2D, log r, leaf 64, eps 1e-8)
    "g2d_cfg1_h2star": ("uniform", 4096, 2, "log2d", 64, "h2star-bt", 1e-8, True),
    "g2d_cfg1_h2plusH": ("uniform", 4096, 2, "log2d", 64, "h2plusH-star", 1e-8, True),
    # 3D trees of depth kappa >= 3 (configs 3 / 5 kernel and tolerance; config 4 kernel)
    "g3d_lap_k3_h2star": ("uniform", 4096, 3, "lap3d", 16, "h2star-bt", 1e-6, True),
    "g3d_lap_k3_h2plusH": ("uniform", 4096, 3, "lap3d", 16, "h2plusH-star", 1e-6, True),
    "g3d_gauss_k3_h2star": ("uniform", 4096, 3, "gaussian", 16, "h2star-bt", 1e-8, True),
}
# Larger fixtures are exported COMPACT: only the transfer operators (P2M, M2M,
# L2L, L2P, BLR factors) go into the blob; the raw kernel blocks (M2L =
# K[t_i, s_o], engine.py:176-179; near = K[t^X, t^Y], engine.py:309-318) are
# exported as "not stored" with the reference's pivots and points, and
# tests/golden_io.materialize() re-evaluates them (oracle.kernel_block).  The
# largest entry difference between the reference's stored blocks and that
# re-evaluation is recorded in the fixture's meta (blk_maxdiff_*).
COMPACT = {"g2d_cfg1_h2star", "g2d_cfg1_h2plusH", "g3d_lap_k3_h2star", "g3d_lap_k3_h2plusH",
           "g3d_gauss_k3_h2star"}


def block_maxdiff(rep, op):
    """Largest |reference stored block - oracle re-evaluation| over every M2L
    and near block (relative to the block's max entry)."""
    from oracle.packed_matvec import kernel_block
    inv = np.empty_like(op.perm)
    inv[op.perm] = np.arange(op.N)
    out = {"blk_maxdiff_m2l": 0.0, "blk_maxdiff_near": 0.0}
    for ci, ops in enumerate(rep.channels):
        ch = op.channels[ci]
        for (X, Y), M in ops.m2l.items():
            K = kernel_block(op, ch.piv_in[ch.piv_in_ptr[X]:ch.piv_in_ptr[X + 1]],
                             ch.piv_out[ch.piv_out_ptr[Y]:ch.piv_out_ptr[Y + 1]])
            d = np.max(np.abs(M - K), initial=0.0) / max(np.max(np.abs(M), initial=0.0), 1e-300)
            out["blk_maxdiff_m2l"] = max(out["blk_maxdiff_m2l"], float(d))
    for (X, Y) in rep.near_pairs:
        t = rep.tree.clusters[X].index_set
        s = rep.tree.clusters[Y].index_set
        if len(t) == 0 or len(s) == 0:
            continue
        M = rep.near_blocks.get((X, Y))
        if M is None:
            M = rep.kernel.block(t, s)
        K = kernel_block(op, inv[np.asarray(t)], inv[np.asarray(s)])
        d = np.max(np.abs(M - K), initial=0.0) / max(np.max(np.abs(M), initial=0.0), 1e-300)
        out["blk_maxdiff_near"] = max(out["blk_maxdiff_near"], float(d))
    return out


def make(name, dist, N, d, kname, n_max, variant, eps, store_near, seed=42):
    pts = h.make_points(dist, N, d, seed)
    if kname == "gaussian":
        ker = Gaussian(pts)
    else:
        ker = h.make_kernel(kname, pts)
    tree = h.build_tree(pts, n_max)
    rep = h.build_variant(variant, tree, ker, eps=eps, store_near=store_near)
    compact = name in COMPACT
    op = export_rep(rep, store="" if compact else "near,m2l")
    rng = np.random.default_rng(seed + 1)
    q = rng.standard_normal(N)
    Q = rng.standard_normal((N, 2))
    phi_ref = rep.matvec(q)
    Phi_ref = np.stack([rep.matvec(Q[:, j]) for j in range(Q.shape[1])], axis=1)
    phi_dense = dense_matvec(ker, q)
    arrays = op.to_arrays()
    meta = {"name": name, "dist": dist, "N": N, "d": d, "kernel": kname,
            "n_max": n_max, "variant": variant, "eps": eps, "seed": seed,
            "store_near": store_near, "kappa": int(tree.kappa),
            "mem_scalars": int(rep.mem_scalars),
            "re_ref": relative_error(phi_ref, phi_dense),
            "kernel_sigma": 0.1 if kname == "gaussian" else None, "compact": compact}
    if compact:
        meta.update(block_maxdiff(rep, op))
    arrays.update(q=q, Q=Q, phi_ref=phi_ref, Phi_ref=Phi_ref, phi_dense=phi_dense,
                  meta=np.asarray(json.dumps(meta)))
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: kappa={tree.kappa} mem_scalars={rep.mem_scalars} "
          f"re_ref={meta['re_ref']:.3e} size={os.path.getsize(path) / 1e6:.2f} MB")


if __name__ == "__main__":
    only = set(sys.argv[1:])
    for name, args in CASES.items():
        if only and name not in only:
            continue
        make(name, *args)
