"""S-MNN oracle package -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct float64 CPU reference of the Scalable
Mechanistic Neural Network least-squares ODE solve (arXiv 2410.06074,
/root/reference/PAPER.md).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product package ``paper_2410_06074_b200`` never imports it, and it never
imports the product package: the two share no code.

Parity status of every function is listed in ``smnn_oracle.__doc__``.
"""

from .smnn_oracle import *  # noqa: F401,F403
