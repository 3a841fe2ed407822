"""Oracle references for many instances, computed in parallel worker processes.

Test infrastructure only: the oracle (oracle/smnn_oracle.py) is called as it
stands, one instance chunk per task, in `spawn`ed workers (no CUDA state is
inherited).  Used by the GPU parity tests to check whole workloads (e.g. all
1536 Lorenz instances) against the fp64 oracle within seconds.
"""

from __future__ import annotations

import concurrent.futures as cf
import multiprocessing as mp
import os

import numpy as np


def _work(args):
    coeffs, rhs, iv, steps, gy, w = args
    import torch

    torch.set_num_threads(1)
    import oracle as O

    y = O.solve_instances(coeffs, rhs, iv, steps, w=w)
    g = O.grads_instances(coeffs, rhs, iv, steps, gy, w=w, y=y) if gy is not None else None
    return y.numpy(), None if g is None else [t.numpy() for t in g]


def oracle_refs(x: dict, gy, idx, w=(1.0, 1.0, 1.0), chunk: int = 8, workers: int | None = None):
    """fp64 oracle y and (dcoeffs, drhs, div, dsteps) for instances `idx` of the batch `x`
    (inputs are taken in double precision, i.e. exactly as stored)."""
    idx = np.asarray(idx)
    sub = {k: np.asarray(v[idx], dtype=np.float64) for k, v in x.items()}
    g = None if gy is None else np.asarray(gy[idx], dtype=np.float64)
    parts = [slice(i, min(i + chunk, len(idx))) for i in range(0, len(idx), chunk)]
    tasks = [(sub["coeffs"][s], sub["rhs"][s], sub["iv"][s], sub["steps"][s], None if g is None else g[s], w)
             for s in parts]
    n = workers or min(len(tasks), os.cpu_count() or 1, 32)
    if n <= 1:
        res = [_work(t) for t in tasks]
    else:
        with cf.ProcessPoolExecutor(n, mp_context=mp.get_context("spawn")) as ex:
            res = list(ex.map(_work, tasks))
    y = np.concatenate([r[0] for r in res])
    grads = None if gy is None else [np.concatenate([r[1][j] for r in res]) for j in range(4)]
    return y, grads
