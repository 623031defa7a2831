"""B200-native Tensor Power Flow engine (arXiv 2403.04578 hot path).

Drop-in GPU replacements for the reference package's batched solvers
(`tpflow.batch_solve_dense`, `tpflow.batch_solve_sparse`, `tpflow.solve_batch`)
with the same LoadMatrix -> VoltageBatch contract.  The arithmetic runs in
hand-written sm_100a CUDA kernels (libtpf.so, C ABI in include/tpf.h); there
is no CPU fallback.
"""

from ._types import (MemoryGuardError, LoadMatrix, PowerTensor, SingularSystemError,
                     SolveOptions, VoltageBatch, ZERO_VOLTAGE_GUARD, reshape_tensor, unreshape)
from .network import (Branch, NetworkError, NetworkModel, PartitionedAdmittance, SlackSpec,
                      ZipCoefficients, build_admittance, radial_check)
from .synth import GenSpec, assign_impedances, build_network, gen_kary_tree, gen_scenarios
from .dense import DenseOperator, batch_solve_dense
from .sparse import (DEFAULT_MAX_BLOCK_NNZ, SparseOperator, batch_solve_sparse,
                     factorization_count, factorize_ydd)
from .dispatch import METHODS, solve_batch

__version__ = "0.1.0"

__all__ = [
    "Branch", "NetworkError", "NetworkModel", "PartitionedAdmittance", "SlackSpec",
    "ZipCoefficients", "build_admittance", "radial_check",
    "SolveOptions", "LoadMatrix", "PowerTensor", "VoltageBatch", "reshape_tensor", "unreshape",
    "SingularSystemError", "MemoryGuardError", "ZERO_VOLTAGE_GUARD",
    "GenSpec", "gen_kary_tree", "assign_impedances", "build_network", "gen_scenarios",
    "batch_solve_dense", "DenseOperator", "batch_solve_sparse", "SparseOperator",
    "factorization_count", "factorize_ydd", "DEFAULT_MAX_BLOCK_NNZ",
    "solve_batch", "METHODS",
]
