"""Seeded synthetic input generators shared by tests, bench.py and smoke().

This package holds NO S-MNN arithmetic (no assembly, factorisation, solve or
gradient): it only draws the inputs theta = {c, d, u, s} and
upstream gradients dl/dy with the shapes of the paper's workloads.  It is the
only module imported by both the oracle side (tests) and the product side
(bench.py); neither the oracle nor the product package imports the other.
"""

from .workloads import WORKLOADS, Workload, make_inputs, make_grad_y, workload  # noqa: F401
