"""paulib_b200 — B200-native (sm_100a) Pauli-sum hot path behind the
``paulialg`` API (reference ``paulialg/__init__.py:9-97``).

Bit-packed symplectic SoA storage on the GPU, batched string multiply,
outer-product multiply with sort-and-merge, the all-pairs commutation
bitmatrix and greedy commutation grouping, all computed by hand-written CUDA
kernels through the C ABI in ``include/paulib_b200.h``.
"""

from .bits import (CAPACITY_TIERS, MAX_QUBITS, PHASE_FACTORS, CapacityError, DimensionError,
                   LabelError, tier_for, words_for)
from .strings import (PauliString, batch_multiply, batch_pair_multiply, batch_sip,
                      product_phase_exponent, ps_apply_clifford, ps_commutes, ps_from_label,
                      ps_multiply, ps_to_label, ps_weight, symplectic_inner_product)
from .sums import (PauliSum, PauliSumSoA, PauliTerm, outer_multiply, sort_and_combine,
                   sort_combine, sum_apply_clifford, sum_apply_rotation, sum_from_terms,
                   sum_multiply, to_aos, to_soa, truncate)
from .grouping import (CommutationPartition, GroupingStats, ValidationReport, group_assignment,
                       group_greedy, group_greedy_parallel, validate_partition)
from .bitmatrix import commutation_bitmatrix, unpack_bits
from .rotations import RotationSpec, TRIG_SNAP, reorder_rotation, trig_values
from .hamio import HamiltonianFormatError, read_hamiltonian, write_hamiltonian
from .rng import SplitMix64, config_columns, random_columns, random_string, random_sum
from ._native import NativeLibraryError

__version__ = "0.1.0"

__all__ = [
    "CAPACITY_TIERS", "MAX_QUBITS", "PHASE_FACTORS", "CapacityError", "DimensionError",
    "LabelError", "tier_for", "words_for",
    "PauliString", "batch_multiply", "batch_pair_multiply", "batch_sip",
    "product_phase_exponent", "ps_apply_clifford", "ps_commutes", "ps_from_label", "ps_multiply", "ps_to_label",
    "ps_weight", "symplectic_inner_product",
    "PauliSum", "PauliSumSoA", "PauliTerm", "outer_multiply", "sort_and_combine", "sort_combine",
    "sum_apply_clifford", "sum_apply_rotation", "sum_from_terms", "sum_multiply", "to_aos", "to_soa", "truncate",
    "CommutationPartition", "GroupingStats", "ValidationReport", "group_assignment",
    "group_greedy", "group_greedy_parallel", "validate_partition",
    "commutation_bitmatrix", "unpack_bits",
    "RotationSpec", "TRIG_SNAP", "reorder_rotation", "trig_values",
    "HamiltonianFormatError", "read_hamiltonian", "write_hamiltonian",
    "SplitMix64", "config_columns", "random_columns", "random_string", "random_sum",
    "NativeLibraryError", "__version__",
]
