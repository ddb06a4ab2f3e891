"""B200-native (sm_100a) SPAI / SPAI-update / block-GCRO path of
"Preconditioned Linear Solves for Parametric Model Order Reduction"
(arXiv 1809.06574).

The public names mirror the reference package ``pmorprec``
(/root/reference/pkg/src/pmorprec/__init__.py:4-64) for the hot path:
assembly, spai_pattern / spai_column / spai_build, update_first /
update_second / sequence_precondition, block_gcro_solve / gcro_solve and
the sequence driver.  Compute runs in libpmorb200.so (hand-written CUDA
for sm_100a, bound with ctypes); PyTorch supplies device memory, streams
and torch.distributed.  There is no CPU fallback.
"""

from .device import DeviceCSR, DevicePattern, Structure
from .krylov import (SolveReport, SolverBreakdown, SolverConfig, apply_preconditioner,
                     block_gcro_solve, block_gcro_solve_batch, gcro_solve)
from .mmio import (read_dense_matrix_market, read_matrix_market, write_dense_matrix_market,
                   write_matrix_market)
from .model import AffineFamily, SecondOrderModel, evaluate, pmor_l_sequence
from .rpmor import (ConvergenceError, ExpansionPoint, PipelineReport, ReducedModel,
                    extend_orthonormal_basis, first_moment_rhs, first_moments,
                    mgs_orthonormalize, rpmor_reduce, zeroth_moment)
from .sequence import PrecondPolicy, SequencePreconditioner, run_sequence
from .spai import (BuildStats, Preconditioner, SparsityPattern, SpaiConfig, quality, spai_build,
                   spai_column, spai_pattern)
from .update import (UpdateConfig, SequenceStep, sequence_precondition, update_first,
                     update_first_many, update_second)

__version__ = "0.1.0"
