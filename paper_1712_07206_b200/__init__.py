"""paper_1712_07206_b200 — B200-native HSDLA Hamiltonian/Overlap construction.

Drop-in for the reference's hot path ``hsdla::pipeline::build_hs_refined``
(arXiv 1712.07206, Algorithm 3), plus ``build_hs_original`` (Algorithm 1), the
``build_hs`` dispatch, the batched ``potrf`` and HSDL v1 problem files streamed
straight into HBM (``build_hs_file``).  The compute lives in ``libhsdla_b200.so``
(hand-written sm_100a CUDA behind the C-ABI of ``include/hsdla_b200.h``); this
package is the host-side mirror of the reference interface.
"""
from .errors import CudaError, ConfigError, DimensionError, IoError, NcclError, SizingError  # noqa: F401
from .pipeline import (Engine, FlopLedger, HSResult, PhaseTime, PipelineConfig, build_hs, build_hs_file,  # noqa: F401,E501
                       build_hs_kpoints, build_hs_original, group_reduce, build_hs_refined, device_count, flop_model, fp64_peak, host_register, host_unregister, mirror,
                       nccl_unique_id, parse_strategy, potrf, problem_file_info, set_default_arith, shard_atoms, shard_rows, parse_variant, rel_frobenius_error_lower,
                       release_cache)
from .problem import (Preset, ProblemInstance, empty_problem, find_preset, generate_problem, generate_problem_shard,  # noqa: F401
                      load_problem, presets, save_problem)
from .lapw import LapwSystem, build_hs_lapw, lapw_coefficients, make_lapw_system  # noqa: F401,E402
from . import kernels  # noqa: F401,E402
