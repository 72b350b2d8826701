"""paper_1906_01128_b200: the deep-copy hot path of arXiv 1906.01128 on NVIDIA B200.

A drop-in for the reference package ``chainforge``'s hot path (scenarios / memory /
harness, SPEC.md): the same names and semantics, executed by libchainforge_b200.so --
hand-written sm_100a kernels plus a native host marshaller behind a C ABI
(include/chainforge_b200.h).  ``import paper_1906_01128_b200 as chainforge`` is the switch.
"""
from .errors import (AttachOutsideArena, NativeUnavailable, OutOfSimMemory, SchemeError,
                     SimMemoryError, VerificationFailed, WildAccess)
from .harness import (ChainShape, CostModel, DevicePrep, KernelStats, P100_COST_MODEL, RunMetrics,
                      SCHEMES, adaptive_repeat, chain_shape, copy_back, estimate_instructions,
                      execute_case, kernel_scale, run_case, simulate_times, sweep,
                      transfer_to_device, verify_tree)
from .memory import (AddressMap, Arena, Machine, MemorySpace, TransferEntry, TransferLog,
                     UvmState)
from .scenarios import (ArrayRef, DenseSpec, ForestSpec, LinearSpec, TreeHandle, build_dense_tree,
                        build_linear_tree, build_tree, dense_data_size, linear_data_size,
                        marshal_tree, payload_values, targeted_arrays, tree_total_bytes)
from .report import MissingBaseline, ResultRow, normalize, rows_from_csv, rows_to_csv
from .engine import DeepCopyWindow

__version__ = "0.1.0"
