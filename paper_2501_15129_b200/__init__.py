"""B200-native EvoRL ES generation path (arxiv 2501.15129 hot path).

The product is ``libevorl_b200.so`` (hand-written sm_100a CUDA behind the C ABI
in ``include/evorl_b200.h``); this package is the thin host-side mirror of the
reference's Workflow / ask-tell / rollout interfaces over that ABI.
"""
from ._lib import (CheckpointError, ConfigError, DeviceError, EnvFault, EvorlError,
                   InvalidArgument, LengthError, MissingExtension, NetFault, Unsupported)
from .es import (CmaEs, EsConfig, EsWorkflow, StepMetrics, ars_ask, ars_tell, batched_rollout,
                 centered_ranks, env_step_batch, gaussian_matrix, measure_fp64_peak, measure_noise_rate,
                 mlp_desc, openes_ask, openes_tell, param_count, pinned_empty, rank_desc, stream_words,
                 sym_eig, threefry2x64)

__all__ = [
    "ConfigError", "DeviceError", "EnvFault", "EvorlError", "InvalidArgument", "LengthError",
    "MissingExtension", "NetFault", "Unsupported", "CheckpointError", "CmaEs", "EsConfig", "EsWorkflow", "StepMetrics",
    "ars_ask", "ars_tell", "batched_rollout", "centered_ranks", "env_step_batch",
    "gaussian_matrix", "measure_fp64_peak", "measure_noise_rate", "mlp_desc", "openes_ask", "openes_tell",
    "param_count", "pinned_empty", "rank_desc", "stream_words", "sym_eig", "threefry2x64",
]
