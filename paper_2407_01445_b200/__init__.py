"""B200-native FastCLIP loss step (arXiv 2407.01445): sm_100a tcgen05 kernels behind a C ABI.

See DESIGN.md for the hot path, the kernels and their rooflines; fastclip.py for the host
mirror of the reference's loss-step interface.
"""
from .fastclip import (BatchPlan, LossStep, FastclipError, StepScalars, config_defaults, debug_similarity,  # noqa: F401
                       embedding_cotangents, epsilon_at, g_values, gamma_at, grad_tau, lib, nccl_unique_id, table_update,
                       temperature_step, VARIANTS)
