"""Loading helpers for the golden fixtures (tests/golden/*.npz)."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

from paper_2309_14085_b200.packed import PackedOperator

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden_names():
    # operator fixtures (gmres_*.npz hold solver trajectories, not operators)
    return sorted(os.path.splitext(os.path.basename(p))[0]
                  for p in glob.glob(os.path.join(GOLDEN_DIR, "g*.npz"))
                  if not os.path.basename(p).startswith("gmres_"))


def load_golden(name):
    with np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"), allow_pickle=False) as z:
        arrays = {k: z[k] for k in z.files}
    op = PackedOperator.from_arrays(arrays)
    meta = json.loads(str(arrays["meta"]))
    return op, arrays, meta


def rel_err(a, b):
    """2-norm relative error (reference bench.py:100-104)."""
    den = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - b) / den) if den else float(np.linalg.norm(a))
