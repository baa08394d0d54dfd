"""B200-native free-space Spectral Ewald (stokeslet / stresslet / rotlet sums).

A drop-in for the reference library's hot path (fse::total_sum and the
functions under it, /root/reference/proj/src/ewald.cpp:394-415) built as
hand-written sm_100a CUDA kernels behind a C-ABI
(include/fse_cuda.h, libfse_b200.so).  This package is the Python mirror of
the reference's fse:: API; the C++ mirror lives in csrc/cpp/include/fse.
"""
from .api import (CellList, Context, DomainError, EwaldConfig, FseError, FseRuntimeError,
                  GreenKind, InvalidArgument, KernelKind, MollifiedGreen, SourceSystem,
                  StageTimings, WL_CLUSTERED, WL_SPHERE, WL_UNIFORM, WL_UNIFORM_TARGETS,
                  build_cell_list, default_context, direct_sum, fft3d_forward, fft3d_inverse,
                  fourier_sum, generate_system, generate_workload, green_kind_for, kspace_scale,
                  library_path, load_mollified_green, make_config, precompute_mollified_green,
                  real_space_sum, rms_error, save_mollified_green, self_interaction, spread,
                  strength_arity, strength_quadratic_sum, total_sum, ErrorBudget,
                  error_budget, fourier_error_estimate, real_error_estimate,
                  reference_velocity_rms, select_parameters, freespace_solve,
                  nccl_unique_id, dist_owner, dist_masks, MultiContext)

__all__ = [n for n in dir() if not n.startswith("_")]
