"""Golden residual trajectories of GMRES(30) on config 4's kernel, produced
by the REFERENCE's own solver.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_gmres_golden.py

The reference solver (solver.py:43-103) is restart-free; GMRES(m) built from
it is the textbook loop "x += gmres(A, b - A x, max_iter=m).x".  The matrix
is config 4's dense Gaussian, exp(-r^2 / (2 * 0.1^2)) + 1e-6 I (BASELINE.json
configs[3]), on ``uniform_points(N, 3, 42)`` (points.py:10-12); the RHS is
``default_rng(43).standard_normal(N)`` (bench.py:131-136).  For each N the
fixture keeps the true relative residual after every restart cycle (10
cycles = 300 Arnoldi steps, bench.py's ``max_iter``) and the eigenvalue range.

These pin that the stagnation of unpreconditioned GMRES(30) on this operator
is the algorithm's, not the GPU path's: ``tests/test_solver.py`` runs
``gmres_block`` on the same matrices and must reproduce the trajectory.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from h2weak.points import uniform_points  # noqa: E402
from h2weak.solver import GmresConfig, gmres  # noqa: E402
from scipy.spatial.distance import cdist  # noqa: E402

SIGMA, SHIFT, RESTART, CYCLES = 0.1, 1e-6, 30, 10


def gaussian_dense(n):
    p = uniform_points(n, 3, 42).points
    return np.exp(-cdist(p, p) ** 2 / (2 * SIGMA * SIGMA)) + SHIFT * np.eye(n)


def restarted(A, b):
    x = np.zeros_like(b)
    res = []
    for _ in range(CYCLES):
        r = b - A @ x
        rep = gmres(lambda v: A @ v, r, GmresConfig(tol=1e-8, max_iter=RESTART))
        x = x + rep.x
        res.append(np.linalg.norm(b - A @ x) / np.linalg.norm(b))
    return np.array(res)


def main():
    out = {}
    for n in (1024, 2048, 4096):
        A = gaussian_dense(n)
        b = np.random.default_rng(43).standard_normal(n)
        ev = np.linalg.eigvalsh(A)
        out[f"res_{n}"] = restarted(A, b)
        out[f"eig_{n}"] = np.array([ev[0], ev[-1]])
        print(n, "cond", ev[-1] / ev[0], "residual per cycle", out[f"res_{n}"])
    np.savez(os.path.join(HERE, "gmres_gauss_ref.npz"), **out)


if __name__ == "__main__":
    main()
