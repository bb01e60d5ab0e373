"""CPU fp64 oracle for the hot path of arXiv 2306.13618 — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct reference that the CUDA path is
checked against.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product package
(``paper_2306_13618_b200``) never imports, links or executes anything in here, and
this package never imports the product: the two share no code.

What is computed, and where it comes from (``P:n`` = line n of the paper text
``PAPER.md``; ``S:n`` = line n of ``SPEC.md``):

* ``kernels``     — radial kernels of Eq. (4.2): K^Gauss, K^IMQ in the config
                    form exp(-r^2/eps) and (r^2+c^2)^(-1/2); K^Lap = exp(-r/l); the
                    energy kernel k^e = -r (Table 1); r^2 exp(-r^2/eps) (the
                    transport-cost kernel d^2 k).
* ``direct``      — the kernel sum (4.3) by its plain definition, an
                    O(n m) double loop vectorised over blocks of targets.
* ``sinkhorn``    — Algorithm 1 step by step: updates (3.3)/(3.4)
                    with dense direct sums, the plan recovery of P:488, the dual
                    (3.1) and the discrete primal.
                    Also the constant c* of Prop. 2.9 / Eq. (2.10), the
                    Sinkhorn divergence of Eq. (2.12), a tolerance stopping
                    rule (reading R20), lambda-scaling (Sec. 5.1.3), and the
                    transport term <pi, d^r> of the recovered plan; cost exponent
                    r = 2 (Gaussian Gibbs kernel) or r = 1 (Laplace).
* ``mmd``         — the discrete MMD^2 of Eq. (3.5), V-statistic form.

Every function is pinned by ``tests/test_oracle_pins.py`` against closed forms,
brute force and invariants that do not reuse the oracle's own formulas (see
DESIGN.md "Oracle pins").  No function here is "parity unpinned".
"""

from .kernels import gauss, gauss_r2, imq, laplace, energy, kernel_fn, GAUSS, IMQ, GAUSS_R2, LAP, ENERGY  # noqa: F401
from .direct import kernel_sum_direct  # noqa: F401
from .sinkhorn import (  # noqa: F401
    uot_sinkhorn_direct,
    dual_objective,
    primal_objective_dense,
    primal_objective_marginals,
    SinkhornResult,
    cstar,
    sinkhorn_divergence_direct,
    uot_sinkhorn_scaling_direct,
    plan_marginals,
    transport_cost,
)
from .mmd import mmd2_direct, mmd2_combined  # noqa: F401
