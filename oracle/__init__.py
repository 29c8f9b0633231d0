"""CPU oracle for the RESCAL MU hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy, the arithmetic of the reference package
``rescalkit`` (``/root/reference/pkg/src/rescalkit``) on the path named by
``BASELINE.json`` ``north_star``: the non-negative RESCAL multiplicative
update and the RESCALk driver around it.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import this package.
  * The product package ``paper_2202_09512_b200`` never imports it; the product
    path has no CPU fallback and fails loudly without its CUDA library.

Parity is PINNED: ``tests/golden/*.npz`` were produced by running the real
reference (``tests/golden/make_golden.py``) in the build container, and
``tests/test_oracle_golden.py`` checks every function here against them.
"""

from .mu_oracle import (  # noqa: F401
    OracleConfig,
    canonical_csr,
    finalize_normalize,
    mu_iteration,
    nndsvd_init,
    perturbation_field,
    perturb_dense,
    perturb_sparse,
    random_init,
    regress_r,
    rel_error,
    solve,
    sq_norm,
    sq_residual,
    update_a,
    update_r,
)
from .select_oracle import rescalk_oracle  # noqa: F401
from .pcg64 import Pcg64, seed_state, uniform_doubles  # noqa: F401
