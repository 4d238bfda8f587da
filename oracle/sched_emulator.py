"""ORACLE — test infrastructure only.  numpy executor of the device schedule.

Only ``tests/`` (and ``__graft_entry__.smoke()`` / ``bench.py``'s CPU legs)
may import this module.  It runs the per-rank schedules that
``h2g_schedule_build`` (include/h2g.h) compiles -- the very task/term lists
the GPU plans upload -- on the CPU, so the multi-GPU sharding logic (subtree
ownership, the all-gather exchange, split-K partials, compacted per-rank
blobs) is checked against the reference's matvec without a GPU, in one
process or across gloo ranks (tests/test_sharded.py).

Term kinds (include/h2g.h, "terms" columns a_off, x_off, lda, ncols,
a_space, self):

* a_space 0 / 1: A is a column-major m x ncols block of the blob / arena;
* a_space 2 (kernel-evaluated, the P2P engine's terms): A = K[records
  row_rec .. row_rec + m, records a_off .. a_off + ncols], the entry rules
  of Kernel.block (reference kernels.py:36-57, restated in
  oracle.packed_matvec.kernel_entries); i == j (same record) only in
  ``self`` terms: M2L blocks K[t_i(X), s_o(Y)] (engine.py:176-179) and
  near blocks K[t^X, t^Y] (engine.py:309-318).
"""

from __future__ import annotations

import numpy as np

from oracle.packed_matvec import kernel_entries


def _eval_block(view, kernel, dim, row_rec, m, col_rec, ncols, self_term):
    recs = view["recs"]
    rows = recs[row_rec:row_rec + m, :dim]
    cols = recs[col_rec:col_rec + ncols, :dim]
    diff = rows[:, None, :] - cols[None, :, :]
    r = np.sqrt((diff * diff).sum(-1))
    ri = np.arange(row_rec, row_rec + m)[:, None]
    ci = np.arange(col_rec, col_rec + ncols)[None, :]
    same = (ri == ci) if self_term else np.zeros((m, ncols), dtype=bool)
    return kernel_entries(kernel, r, same)


def run_phases(view, op, blob, arena, part):
    tasks, terms = view["tasks"], view["terms"]
    for tb, te, ph_part, _ in view["phases"]:
        if ph_part != part:
            continue
        for y_off, m, t0, t1, row_rec in tasks[tb:te]:
            acc = np.zeros(m)
            for a_off, x_off, lda, ncols, a_space, self_term in terms[t0:t1]:
                if a_space == 2:
                    A = _eval_block(view, op.kernel, op.dim, row_rec, m, a_off, ncols, self_term)
                else:
                    src = arena if a_space else blob
                    A = np.lib.stride_tricks.as_strided(src[a_off:], shape=(m, ncols),
                                                        strides=(8, 8 * lda))
                acc += A @ arena[x_off:x_off + ncols]
            arena[y_off:y_off + m] = acc


def emulate_begin(view, op, q):
    """Part 0 of a rank's matvec in numpy; returns (arena, send)."""
    blob = view["blob"] if len(view["blob"]) else op.blob
    arena = np.zeros(view["n_slots"] + 8)
    arena[view["ones_off"]:view["ones_off"] + view["n_ones"]] = 1.0
    arena[view["q_tree"]:view["q_tree"] + op.N] = np.asarray(q, dtype=np.float64)[op.perm]
    run_phases(view, op, blob, arena, 0)
    send = np.zeros(max(1, view["max_send_slots"]))
    for src, dst, ln in view["pack"]:
        send[dst:dst + ln] = arena[src:src + ln]
    run_phases(view, op, blob, arena, 2)  # the owned near field, beside the exchange
    return arena, send


def emulate_end(view, op, arena, recv):
    """Unpack the all-gathered buffer, run part 1; returns phi with this rank's rows."""
    blob = view["blob"] if len(view["blob"]) else op.blob
    for src, dst, ln in view["unpack"]:
        arena[dst:dst + ln] = recv[src:src + ln]
    run_phases(view, op, blob, arena, 1)
    phi = np.zeros(op.N)
    rows = np.arange(view["row_begin"], view["row_end"])
    phi[op.perm[rows]] = arena[view["phi_tree"] + rows]
    return phi


def emulate_matvec(op, q, nranks: int = 1, recompute: str = "") -> np.ndarray:
    """All ranks in one process (exchange = concatenation); phi combined."""
    from paper_2309_14085_b200.sharded import schedule_view
    views = [schedule_view(op, r, nranks, recompute) for r in range(nranks)]
    states = [emulate_begin(v, op, q) for v in views]
    mx = max(1, views[0]["max_send_slots"])
    recv = np.zeros(mx * nranks)
    for r, (_, send) in enumerate(states):
        recv[r * mx:r * mx + len(send)] = send[:mx]
    phi = np.zeros(op.N)
    for v, (arena, _) in zip(views, states):
        phi += emulate_end(v, op, arena, recv)
    return phi


def emulate_matvec_distributed(op, q, nranks: int, recompute: str = "") -> np.ndarray:
    """Distributed vectors (include/h2g.h h2g_shard_load_q ... store_phi): each
    rank's arena starts with ONLY its own q rows (the rest NaN, so any read
    outside own rows + received halo poisons the result); the x-halo ranges
    are all-gathered, then the schedule runs as in :func:`emulate_matvec`."""
    from paper_2309_14085_b200.sharded import schedule_view
    views = [schedule_view(op, r, nranks, recompute) for r in range(nranks)]
    q_tree = np.asarray(q, dtype=np.float64)[op.perm]
    halo = views[0]["halo"]
    hm = 1
    for r in range(nranks):
        hm = max(hm, int(halo[halo[:, 0] == r, 2].sum()) if len(halo) else 0)
    hrecv = np.zeros(hm * nranks)
    for r in range(nranks):  # every rank sends its own rows others read
        pos = 0
        for _, row, ln in halo[halo[:, 0] == r]:
            assert views[r]["row_begin"] <= row and row + ln <= views[r]["row_end"]
            hrecv[r * hm + pos:r * hm + pos + ln] = q_tree[row:row + ln]
            pos += ln
    states = []
    for r, v in enumerate(views):
        blob = v["blob"] if len(v["blob"]) else op.blob
        arena = np.zeros(v["n_slots"] + 8)
        arena[v["ones_off"]:v["ones_off"] + v["n_ones"]] = 1.0
        qt = np.full(op.N, np.nan)
        qt[v["row_begin"]:v["row_end"]] = q_tree[v["row_begin"]:v["row_end"]]
        for s_rank in range(nranks):
            if s_rank == r:
                continue
            pos = 0
            for _, row, ln in halo[halo[:, 0] == s_rank]:
                qt[row:row + ln] = hrecv[s_rank * hm + pos:s_rank * hm + pos + ln]
                pos += ln
        arena[v["q_tree"]:v["q_tree"] + op.N] = qt
        run_phases(v, op, blob, arena, 0)
        send = np.zeros(max(1, v["max_send_slots"]))
        for src, dst, ln in v["pack"]:
            send[dst:dst + ln] = arena[src:src + ln]
        run_phases(v, op, blob, arena, 2)  # the owned near field, beside the exchange
        states.append((arena, send))
    mx = max(1, views[0]["max_send_slots"])
    recv = np.zeros(mx * nranks)
    for r, (_, send) in enumerate(states):
        recv[r * mx:r * mx + len(send)] = send[:mx]
    phi = np.zeros(op.N)
    for v, (arena, _) in zip(views, states):
        phi += emulate_end(v, op, arena, recv)
    return phi
