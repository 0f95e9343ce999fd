"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference (arXiv 2408.02274's `emscat`) algorithm
for the hot path: the IFGF far field (ifgf.py:535-882), the near-field apply
(quadrature.py:343-487, operators.py:279-319), the N-Muller assembly
(operators.py:170-403), GMRES (solver.py:30-93) and the off-surface
layer sums (reference.py:285-312).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package, and only as the checker / the timed CPU
baseline.  The product (``paper_2408_02274_b200``) never imports it.

Pinning: the oracle is checked against golden vectors produced by the
unmodified reference (``tests/golden/make_golden.py``; tests in
``tests/test_oracle.py``).  Plan inputs (tree, cone hierarchy,
singular map, moments, correction lists) come from the framework's plan
builder, whose arrays are checked bit-exact against the reference plan
digests (``tests/test_plan.py``).
"""

from .muller_oracle import (far_field, gmres, muller_apply,  # noqa: F401
                            potentials, OperatorData)
from .fields_oracle import layer_fields  # noqa: F401,E402
