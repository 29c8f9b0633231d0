"""B200-native RESCAL multiplicative-update engine (drop-in for rescalkit's MU path).

Public names mirror the reference namespace (pkg/src/rescalkit/__init__.py)
for the hot path: the MU solver, its split/regression helpers, the
perturbation config and the RESCALk driver. Compute runs in the sm_100a
library ``librescal_b200.so``; importing this package does not
touch the GPU, the first solver call does.
"""

from .exceptions import DataError, GridDeadlockError, GridError, NumericalError, RescalkitError
from .containers import RelTensor, SparseRelTensor, fro_norm
from .solver import (
    KernelCounters,
    RescalFactors,
    SolverConfig,
    finalize_normalize,
    nndsvd_init,
    random_init,
    regress_r,
    rel_error,
    release_cached_memory,
    rescal_solve,
    update_a,
    update_r,
)
from .selection import (
    ClusterResult,
    FactorEnsemble,
    PerturbConfig,
    SelectionEntry,
    SelectionReport,
    SilhouetteStats,
    best_match_diagonal,
    cluster_stability,
    custom_cluster,
    lsa,
    pearson_correlation,
    perturb,
    perturbation_field,
    rescalk,
    select_k,
)
from .multigpu import (
    BlockSource,
    DistFactors,
    GridContext,
    TensorBlock,
    block_dim,
    dist_perturb,
    dist_rescal_solve,
    gather_factors,
    grid_block,
    grid_shape,
    partition_block,
    solve_on_grid,
)
from .tensor_io import DenseFile, load_matrix, load_tensor, save_matrix, save_tensor
from ._lib import DeviceError, Engine

__version__ = "0.1.0"
