"""ctypes binding of the C ABI (include/evorl_b200.h) of libevorl_b200.so.

The library is built in-tree (``paper_2501_15129_b200/libevorl_b200.so``) by
``__graft_entry__.build()`` / ``make -C paper_2501_15129_b200/csrc``.  There is
no fallback: if the shared object is missing, importing the product API
raises ``MissingExtension``; if no GPU is present, every compute entry point
returns ``EVORL_E_CUDA`` and this wrapper raises ``DeviceError``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# EVORL_B200_LIB selects another build of the same ABI (e.g. the profiling build)
LIB_PATH = os.environ.get("EVORL_B200_LIB") or os.path.join(HERE, "libevorl_b200.so")

EVORL_OK = 0
EVORL_E_INVALID_ARGUMENT = 1
EVORL_E_LENGTH = 2
EVORL_E_ENV_FAULT = 3
EVORL_E_NET_FAULT = 4
EVORL_E_CONFIG = 5
EVORL_E_CUDA = 6
EVORL_E_UNSUPPORTED = 7
EVORL_E_CHECKPOINT = 8

PREC_F64, PREC_F32, PREC_TC, PREC_OZ = 0, 1, 2, 3
PRECISIONS = {"f64": PREC_F64, "f32": PREC_F32, "tc": PREC_TC, "oz": PREC_OZ}
ENV_CARTPOLE, ENV_PENDULUM = 0, 1
ALGO = {"openes": 0, "ars": 1, "ves": 2, "cmaes": 3, "cem": 4}
NORM = {"auto": -1, "none": 0, "vbn": 1, "running_stats": 2}
HEAD_TANH, HEAD_GAUSSIAN, HEAD_CATEGORICAL, HEAD_LINEAR = 0, 1, 2, 3
MAX_HIDDEN = 8


class MissingExtension(ImportError):
    pass


# ------------------------------------------------- exceptions (reference types)
class EvorlError(RuntimeError):
    code = -1


class InvalidArgument(EvorlError, ValueError):  # std::invalid_argument
    code = EVORL_E_INVALID_ARGUMENT


class LengthError(EvorlError):  # std::length_error
    code = EVORL_E_LENGTH


class EnvFault(EvorlError):  # evorl::EnvFault
    code = EVORL_E_ENV_FAULT


class NetFault(EvorlError):  # evorl::NetFault
    code = EVORL_E_NET_FAULT


class ConfigError(EvorlError):  # evorl::ConfigError
    code = EVORL_E_CONFIG


class DeviceError(EvorlError):
    code = EVORL_E_CUDA


class Unsupported(EvorlError):
    code = EVORL_E_UNSUPPORTED


class CheckpointError(EvorlError):  # evorl::CheckpointError
    code = EVORL_E_CHECKPOINT


_EXC = {c.code: c for c in (InvalidArgument, LengthError, EnvFault, NetFault, ConfigError,
                            DeviceError, Unsupported, CheckpointError)}


class MlpDesc(C.Structure):
    _fields_ = [("input_dim", C.c_int32), ("n_hidden", C.c_int32),
                ("hidden", C.c_int32 * MAX_HIDDEN), ("output_dim", C.c_int32),
                ("layer_norm", C.c_int32), ("head", C.c_int32), ("tanh_scale", C.c_double),
                ("allow_linear", C.c_int32)]


class EnvDescC(C.Structure):
    _fields_ = [("env_id", C.c_int32), ("fixed_horizon", C.c_int32),
                ("max_episode_steps", C.c_int32)]


class ObsNormC(C.Structure):
    _fields_ = [("mode", C.c_int32), ("dim", C.c_int32), ("mean", C.c_double * 4),
                ("var", C.c_double * 4), ("count", C.c_double)]


class EsConfigC(C.Structure):
    _fields_ = [("algo", C.c_int32), ("env_id", C.c_int32), ("fixed_horizon", C.c_int32),
                ("max_episode_steps", C.c_int32), ("n_hidden", C.c_int32),
                ("hidden", C.c_int32 * MAX_HIDDEN), ("layer_norm", C.c_int32),
                ("allow_linear", C.c_int32), ("pop", C.c_int32),
                ("fitness_episodes", C.c_int32), ("obs_norm_mode", C.c_int32),
                ("vbn_samples", C.c_int32), ("openes_sigma", C.c_double),
                ("openes_lr", C.c_double), ("openes_weight_decay", C.c_double),
                ("openes_mirrored", C.c_int32), ("openes_noise_table", C.c_int32),
                ("openes_noise_table_size", C.c_int64), ("ars_sigma", C.c_double),
                ("ars_lr", C.c_double), ("ars_elites", C.c_int32), ("ves_sigma", C.c_double),
                ("ves_elites", C.c_int32), ("ves_mirrored", C.c_int32),
                ("cmaes_sigma0", C.c_double), ("cmaes_elites", C.c_int32),
                ("cmaes_max_dim", C.c_int32), ("cem_elites", C.c_int32),
                ("cem_var_init", C.c_double), ("cem_noise_start", C.c_double),
                ("cem_noise_end", C.c_double), ("cem_decay_iters", C.c_int64),
                ("precision", C.c_int32), ("device", C.c_int32), ("cmaes_eig_every", C.c_int32)]


class StepMetricsC(C.Structure):
    _fields_ = [("fitness_mean", C.c_double), ("fitness_max", C.c_double),
                ("fitness_min", C.c_double), ("sigma", C.c_double),
                ("update_skipped", C.c_double)]


# Every symbol include/evorl_b200.h declares (checked by the CPU test suite).
EXPORTS = [
    "evorl_last_error", "evorl_abi_version", "evorl_kernel_launches", "evorl_threefry2x64",
    "evorl_stream_words", "evorl_gaussian_matrix", "evorl_centered_ranks", "evorl_rank_desc",
    "evorl_env_step_batch", "evorl_batched_rollout", "evorl_openes_tell", "evorl_openes_ask",
    "evorl_ars_ask", "evorl_ars_tell", "evorl_es_default_config", "evorl_es_create",
    "evorl_es_destroy", "evorl_es_dim", "evorl_es_init", "evorl_es_step", "evorl_es_evaluate",
    "evorl_es_counters", "evorl_es_get_mean", "evorl_es_set_mean", "evorl_es_get_adam",
    "evorl_es_set_adam", "evorl_es_get_fitness", "evorl_es_get_obs_norm",
    "evorl_es_set_obs_norm", "evorl_es_set_counters", "evorl_es_set_shard",
    "evorl_es_shard_ranges", "evorl_es_phase_rollout", "evorl_es_phase_tell",
    "evorl_es_device_buffers", "evorl_es_stream", "evorl_es_last_timings", "evorl_es_last_ask_ms",
    "evorl_es_step_host", "evorl_host_alloc", "evorl_host_free",
    "evorl_measure_fp64_peak", "evorl_measure_dmma_peak", "evorl_measure_noise_rate", "evorl_es_cma_get", "evorl_es_cma_set",
    "evorl_sym_eig", "evorl_es_save", "evorl_es_load", "evorl_batched_rollout_transitions",
    "evorl_cma_create", "evorl_cma_ask", "evorl_cma_tell", "evorl_es_device_var",
    "evorl_es_norm_mode", "evorl_es_get_rng", "evorl_es_cem_sigma",
]

_lib = None


def load() -> C.CDLL:
    """Load libevorl_b200.so (raises MissingExtension if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise MissingExtension(
            f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
            "(the B200 path has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
    L.evorl_last_error.restype = C.c_char_p
    L.evorl_kernel_launches.restype = i64
    L.evorl_threefry2x64.argtypes = [vp, vp, vp, i64]
    L.evorl_stream_words.argtypes = [u64, u64, i64, i64, vp]
    L.evorl_gaussian_matrix.argtypes = [u64, u64, i64, i64, vp]
    L.evorl_centered_ranks.argtypes = [vp, i64, vp]
    L.evorl_rank_desc.argtypes = [vp, i64, vp]
    L.evorl_env_step_batch.argtypes = [C.c_int, C.c_int, C.c_int, i64, vp, vp, vp, vp, vp, vp, vp]
    L.evorl_batched_rollout.argtypes = [C.POINTER(EnvDescC), C.POINTER(MlpDesc),
                                        C.POINTER(ObsNormC), vp, i32, i32, i32, u64, u64, i32,
                                        vp, vp, vp]
    L.evorl_batched_rollout_transitions.argtypes = [C.POINTER(EnvDescC), C.POINTER(MlpDesc),
                                                    C.POINTER(ObsNormC), vp, i32, i32, i32, u64, u64,
                                                    i32, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp]
    L.evorl_openes_tell.argtypes = [vp, vp, vp, C.POINTER(i64), i64, dbl, dbl, dbl, i32, u64,
                                    u64, vp, i32]
    L.evorl_openes_ask.argtypes = [vp, i64, dbl, i32, u64, u64, i32, vp, vp]
    L.evorl_ars_ask.argtypes = [vp, i64, dbl, u64, u64, i32, vp, vp]
    L.evorl_ars_tell.argtypes = [vp, i64, i32, dbl, u64, u64, vp, i32, C.POINTER(i32)]
    L.evorl_es_default_config.argtypes = [C.POINTER(EsConfigC)]
    L.evorl_es_create.argtypes = [C.POINTER(EsConfigC), C.POINTER(vp)]
    L.evorl_es_destroy.argtypes = [vp]
    L.evorl_es_dim.argtypes = [vp]
    L.evorl_es_dim.restype = i64
    L.evorl_es_init.argtypes = [vp, u64, u64]
    L.evorl_es_step.argtypes = [vp, C.POINTER(StepMetricsC)]
    L.evorl_es_evaluate.argtypes = [vp, i32, u64, u64, C.POINTER(dbl), C.POINTER(dbl)]
    L.evorl_es_save.argtypes = [vp, C.c_char_p]
    L.evorl_cma_create.argtypes = [i64, i32, i32, dbl, i32, i32, C.POINTER(vp)]
    L.evorl_cma_ask.argtypes = [vp, u64, u64, vp]
    L.evorl_cma_tell.argtypes = [vp, vp, vp]
    L.evorl_es_load.argtypes = [vp, C.c_char_p]
    L.evorl_es_counters.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
    L.evorl_es_set_counters.argtypes = [vp, i64, i64, i64]
    L.evorl_es_get_mean.argtypes = [vp, vp]
    L.evorl_es_set_mean.argtypes = [vp, vp]
    L.evorl_es_get_adam.argtypes = [vp, vp, vp, C.POINTER(i64)]
    L.evorl_es_set_adam.argtypes = [vp, vp, vp, i64]
    L.evorl_es_get_fitness.argtypes = [vp, vp]
    L.evorl_es_get_obs_norm.argtypes = [vp, C.POINTER(ObsNormC)]
    L.evorl_es_set_obs_norm.argtypes = [vp, C.POINTER(ObsNormC)]
    L.evorl_es_set_shard.argtypes = [vp, i32, i32]
    L.evorl_es_shard_ranges.argtypes = [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i64),
                                        C.POINTER(i64)]
    L.evorl_es_phase_rollout.argtypes = [vp]
    L.evorl_es_phase_tell.argtypes = [vp, C.POINTER(StepMetricsC)]
    L.evorl_es_device_buffers.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]
    L.evorl_es_device_var.argtypes = [vp, C.POINTER(vp)]
    L.evorl_es_norm_mode.argtypes = [vp, C.POINTER(i32)]
    L.evorl_es_get_rng.argtypes = [vp, C.POINTER(u64), C.POINTER(u64)]
    L.evorl_es_cem_sigma.argtypes = [vp, C.POINTER(dbl)]
    L.evorl_es_stream.argtypes = [vp]
    L.evorl_es_stream.restype = vp
    L.evorl_es_last_timings.argtypes = [vp, C.POINTER(C.c_float), C.POINTER(C.c_float)]
    L.evorl_es_last_ask_ms.argtypes = [vp, C.POINTER(C.c_float)]
    L.evorl_es_step_host.argtypes = [vp, vp, vp, vp, C.c_int64, vp, vp, vp, C.POINTER(C.c_int64), vp]
    L.evorl_host_alloc.argtypes = [C.c_int64, C.POINTER(vp)]
    L.evorl_host_free.argtypes = [vp]
    L.evorl_host_free.restype = None
    L.evorl_measure_fp64_peak.argtypes = [C.POINTER(dbl)]
    L.evorl_measure_noise_rate.argtypes = [C.c_int64, C.POINTER(C.c_float)]
    L.evorl_measure_dmma_peak.argtypes = [C.POINTER(dbl)]
    L.evorl_es_cma_get.argtypes = [vp, vp, vp, vp, vp, vp, C.POINTER(dbl), C.POINTER(i64),
                                   C.POINTER(i64)]
    L.evorl_es_cma_set.argtypes = [vp, vp, vp, vp, vp, vp, dbl, i64, i64]
    L.evorl_sym_eig.argtypes = [vp, i32, vp, vp, C.POINTER(i32)]
    _lib = L
    return L


def check(rc: int) -> int:
    if rc != EVORL_OK:
        msg = load().evorl_last_error().decode()
        raise _EXC.get(rc, EvorlError)(msg)
    return rc
