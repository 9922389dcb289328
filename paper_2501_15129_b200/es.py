"""Reference-facing host API over the C ABI.

Mirrors the reference's C++ seam with the same names,
argument meaning and error behaviour, so the parity tests read like the
reference's own tests:

  * ``EsWorkflow``      -- Workflow::init/step/evaluate of proj/src/workflow_es.cpp
  * ``batched_rollout`` -- proj/src/rollout.cpp:176-214 (deterministic policies)
  * ``gaussian_matrix``, ``centered_ranks``, ``rank_desc`` -- proj/src/ec.cpp
  * ``openes_ask``/``openes_tell``, ``ars_ask``/``ars_tell`` -- proj/src/ec.cpp
  * ``env_step_batch``  -- proj/src/env.cpp:113-155

All compute runs on the GPU through libevorl_b200.so.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check

__all__ = ["EsConfig", "EsWorkflow", "StepMetrics", "batched_rollout", "gaussian_matrix",
           "centered_ranks", "rank_desc", "openes_ask", "openes_tell", "ars_ask", "ars_tell",
           "env_step_batch", "threefry2x64", "stream_words", "param_count", "mlp_desc",
           "measure_fp64_peak", "measure_noise_rate", "pinned_empty", "sym_eig"]


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _key(key) -> tuple[int, int]:
    if hasattr(key, "hi"):
        return int(key.hi), int(key.lo)
    return int(key[0]), int(key[1])


# ----------------------------------------------------------------- config
@dataclass
class EsConfig:
    """Reference config-registry keys (proj/src/config.cpp:23-70) for the ES
    workflow, with the registry defaults."""
    algo: str = "openes"                 # ec.algo
    env: str = "cartpole"                # env.id
    fixed_horizon: bool = False          # env.fixed_horizon
    max_episode_steps: int = 0           # env.max_episode_steps
    hidden: Sequence[int] = (64, 64)     # net.hidden
    layer_norm: bool = False             # net.layer_norm
    allow_linear: bool = False           # EXTENSION: hidden=() linear policy
    pop: int = 128                       # ec.pop
    fitness_episodes: int = 1            # ec.fitness_episodes
    obs_norm: str = "auto"               # obs_norm.mode
    vbn_samples: int = 10000             # obs_norm.vbn_samples
    openes_sigma: float = 0.02
    openes_lr: float = 0.01
    openes_weight_decay: float = 0.005
    openes_mirrored: bool = True
    openes_noise_table: bool = False
    openes_noise_table_size: int = 1 << 22
    ars_sigma: float = 0.03
    ars_lr: float = 0.02
    ars_elites: int = 16
    ves_sigma: float = 0.02
    ves_elites: int = 16
    ves_mirrored: bool = True
    cmaes_sigma0: float = 0.1
    cmaes_elites: int = 64
    cmaes_max_dim: int = 4096
    cem_elites: int = 5
    cem_var_init: float = 1e-3
    cem_noise_start: float = 1e-3
    cem_noise_end: float = 1e-5
    cem_decay_iters: int = 2000
    precision: str = "f64"               # "f64" (parity) | "f32" | "tc" (tcgen05 hidden layer)
    device: int = 0
    cmaes_eig_every: int = 1             # EXTENSION: lazy CMA-ES eigendecomposition period (0 = auto gap)

    def to_c(self) -> _lib.EsConfigC:
        c = _lib.EsConfigC()
        _lib.load().evorl_es_default_config(C.byref(c))
        if self.algo not in _lib.ALGO:
            raise _lib.ConfigError(f"ec.algo: unknown algorithm '{self.algo}'")
        c.algo = _lib.ALGO[self.algo]
        if self.env not in ("cartpole", "pendulum"):
            raise _lib.InvalidArgument(f"unknown env id: {self.env}")
        c.env_id = _lib.ENV_CARTPOLE if self.env == "cartpole" else _lib.ENV_PENDULUM
        c.fixed_horizon = int(self.fixed_horizon)
        c.max_episode_steps = int(self.max_episode_steps)
        c.n_hidden = len(self.hidden)
        for i, h in enumerate(self.hidden):
            c.hidden[i] = int(h)
        c.layer_norm = int(self.layer_norm)
        c.allow_linear = int(self.allow_linear)
        c.pop = int(self.pop)
        c.fitness_episodes = int(self.fitness_episodes)
        if self.obs_norm not in _lib.NORM:
            raise _lib.ConfigError(f"obs_norm.mode: unknown value '{self.obs_norm}'")
        c.obs_norm_mode = _lib.NORM[self.obs_norm]
        c.vbn_samples = int(self.vbn_samples)
        for k in ("openes_sigma", "openes_lr", "openes_weight_decay", "ars_sigma", "ars_lr",
                  "ves_sigma", "cmaes_sigma0", "cem_var_init", "cem_noise_start",
                  "cem_noise_end"):
            setattr(c, k, float(getattr(self, k)))
        for k in ("openes_mirrored", "openes_noise_table", "ves_mirrored"):
            setattr(c, k, int(bool(getattr(self, k))))
        for k in ("openes_noise_table_size", "ars_elites", "ves_elites", "cmaes_elites",
                  "cmaes_max_dim", "cem_elites", "cem_decay_iters", "device", "cmaes_eig_every"):
            setattr(c, k, int(getattr(self, k)))
        c.precision = _lib.PRECISIONS[self.precision]
        return c


@dataclass
class StepMetrics:
    """StepMetrics of EsWorkflow::step (proj/src/workflow_es.cpp:140-169)."""
    values: dict = field(default_factory=dict)

    def __getitem__(self, k):
        return self.values[k]


class EsWorkflow:
    """Device-resident EsWorkflow (proj/src/workflow_es.cpp:26-276)."""

    def __init__(self, cfg: EsConfig):
        self.L = _lib.load()
        self.cfg = cfg
        self._c = cfg.to_c()
        h = C.c_void_p()
        check(self.L.evorl_es_create(C.byref(self._c), C.byref(h)))
        self.h = h
        self.dim = int(self.L.evorl_es_dim(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.L.evorl_es_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # Workflow interface --------------------------------------------------
    def init(self, key) -> "EsWorkflow":
        hi, lo = _key(key)
        check(self.L.evorl_es_init(self.h, hi, lo))
        return self

    def step(self) -> StepMetrics:
        m = _lib.StepMetricsC()
        check(self.L.evorl_es_step(self.h, C.byref(m)))
        return self._metrics(m)

    def step_host(self, mean, m=None, v=None, t: int = 0, out=None):
        """Workflow::step with the state on the host (evorl_es_step_host):
        returns (mean, m, v, t, metrics) after the generation; m, v None keeps
        the device's Adam moments.  `out` = three float64 arrays of length dim
        to write the state into (they may be the inputs; page-locked ones from
        pinned_empty() are copied by DMA directly)."""
        mean = np.ascontiguousarray(mean, np.float64)
        if mean.shape != (self.dim,):
            raise ValueError("step_host: mean size mismatch")
        mi = vi = None
        if m is not None:
            mi, vi = np.ascontiguousarray(m, np.float64), np.ascontiguousarray(v, np.float64)
        if out is None:
            mo, mm, vv = np.empty(self.dim), np.empty(self.dim), np.empty(self.dim)
        else:
            mo, mm, vv = out
            for a in out:
                if a.dtype != np.float64 or a.shape != (self.dim,) or not a.flags.c_contiguous:
                    raise ValueError("step_host: out arrays must be contiguous float64 of length dim")
        tt = C.c_int64()
        met = _lib.StepMetricsC()
        check(self.L.evorl_es_step_host(self.h, _p(mean), _p(mi) if mi is not None else None,
                                        _p(vi) if vi is not None else None, int(t), _p(mo), _p(mm), _p(vv),
                                        C.byref(tt), C.byref(met)))
        return mo, mm, vv, tt.value, self._metrics(met)

    def evaluate(self, episodes: int, key) -> tuple[float, float]:
        hi, lo = _key(key)
        mr, sd = C.c_double(), C.c_double()
        check(self.L.evorl_es_evaluate(self.h, int(episodes), hi, lo, C.byref(mr), C.byref(sd)))
        return mr.value, sd.value

    # checkpoints (Workflow::save / load, EVORL1 format) --------------------
    def save(self, path) -> None:
        """Write an EVORL1 checkpoint the reference can load (and vice versa)."""
        check(self.L.evorl_es_save(self.h, os.fsencode(path)))

    def load(self, path) -> "EsWorkflow":
        """Restore state from an EVORL1 checkpoint (same config as the writer)."""
        check(self.L.evorl_es_load(self.h, os.fsencode(path)))
        return self

    @staticmethod
    def _metrics(m) -> StepMetrics:
        return StepMetrics({"fitness/mean": m.fitness_mean, "fitness/max": m.fitness_max,
                            "fitness/min": m.fitness_min, "es/sigma": m.sigma,
                            "es/update_skipped": m.update_skipped})

    # state access -------------------------------------------------------
    def mean(self) -> np.ndarray:
        out = np.empty(self.dim, np.float64)
        check(self.L.evorl_es_get_mean(self.h, _p(out)))
        return out

    def set_mean(self, mean) -> None:
        m = np.ascontiguousarray(mean, np.float64)
        assert m.shape == (self.dim,)
        check(self.L.evorl_es_set_mean(self.h, _p(m)))

    def adam(self):
        m = np.empty(self.dim, np.float64)
        v = np.empty(self.dim, np.float64)
        t = C.c_int64()
        check(self.L.evorl_es_get_adam(self.h, _p(m), _p(v), C.byref(t)))
        return m, v, t.value

    def set_adam(self, m, v, t: int) -> None:
        m = np.ascontiguousarray(m, np.float64)
        v = np.ascontiguousarray(v, np.float64)
        check(self.L.evorl_es_set_adam(self.h, _p(m), _p(v), int(t)))

    def fitness(self) -> np.ndarray:
        out = np.empty(self.cfg.pop, np.float64)
        check(self.L.evorl_es_get_fitness(self.h, _p(out)))
        return out

    def obs_norm(self) -> _lib.ObsNormC:
        o = _lib.ObsNormC()
        check(self.L.evorl_es_get_obs_norm(self.h, C.byref(o)))
        return o

    def set_obs_norm(self, o) -> None:
        oc = _lib.ObsNormC()
        for k in ("mode", "dim", "count"):
            setattr(oc, k, getattr(o, k))
        for i in range(4):
            oc.mean[i] = o.mean[i]
            oc.var[i] = o.var[i]
        check(self.L.evorl_es_set_obs_norm(self.h, C.byref(oc)))

    def counters(self) -> tuple[int, int, int]:
        it, st, ep = C.c_int64(), C.c_int64(), C.c_int64()
        check(self.L.evorl_es_counters(self.h, C.byref(it), C.byref(st), C.byref(ep)))
        return it.value, st.value, ep.value

    def rng(self) -> tuple[int, int]:
        """WorkflowState::rng: the root key of init() or of the loaded checkpoint."""
        hi, lo = C.c_uint64(), C.c_uint64()
        check(self.L.evorl_es_get_rng(self.h, C.byref(hi), C.byref(lo)))
        return hi.value, lo.value

    def norm_mode(self) -> int:
        """The resolved obs_norm mode (_lib.NORM values; "auto" already resolved)."""
        m = C.c_int32()
        check(self.L.evorl_es_norm_mode(self.h, C.byref(m)))
        return m.value

    def cem_sigma(self) -> float:
        """es/sigma of a CEM workflow, sqrt(diag_var.mean()) over the full variance."""
        v = C.c_double()
        check(self.L.evorl_es_cem_sigma(self.h, C.byref(v)))
        return v.value

    def set_counters(self, iteration: int, env_steps: int, episodes: int) -> None:
        check(self.L.evorl_es_set_counters(self.h, iteration, env_steps, episodes))

    def last_timings(self) -> tuple[float, float]:
        r, s = C.c_float(), C.c_float()
        check(self.L.evorl_es_last_timings(self.h, C.byref(r), C.byref(s)))
        return r.value, s.value

    def last_ask_ms(self) -> float:
        """Device ms of the last generation's materialised ask (-1 if not timed)."""
        a = C.c_float()
        check(self.L.evorl_es_last_ask_ms(self.h, C.byref(a)))
        return a.value

    # sharded phases (see paper_2501_15129_b200.dist) ----------------------
    def set_shard(self, rank: int, world: int) -> None:
        check(self.L.evorl_es_set_shard(self.h, rank, world))

    def shard_ranges(self):
        a0, a1, p0, p1 = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
        check(self.L.evorl_es_shard_ranges(self.h, C.byref(a0), C.byref(a1), C.byref(p0),
                                           C.byref(p1)))
        return a0.value, a1.value, p0.value, p1.value

    def phase_rollout(self) -> None:
        check(self.L.evorl_es_phase_rollout(self.h))

    def phase_tell(self) -> StepMetrics:
        m = _lib.StepMetricsC()
        check(self.L.evorl_es_phase_tell(self.h, C.byref(m)))
        return self._metrics(m)

    def device_buffers(self):
        f, m, s = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(self.L.evorl_es_device_buffers(self.h, C.byref(f), C.byref(m), C.byref(s)))
        return f.value, m.value, s.value

    def device_var(self) -> int:
        """Device pointer of CEM's diagonal variance (d doubles)."""
        v = C.c_void_p()
        check(self.L.evorl_es_device_var(self.h, C.byref(v)))
        return v.value

    def stream(self) -> int:
        return self.L.evorl_es_stream(self.h)

    # CMA-ES state (proj/include/evorl/ec.hpp:107-122) ----------------------
    def cma_state(self) -> dict:
        d = self.dim
        Cm, Bm = np.empty((d, d)), np.empty((d, d))
        D, ps, pc = np.empty(d), np.empty(d), np.empty(d)
        sg, gen, rc = C.c_double(), C.c_int64(), C.c_int64()
        check(self.L.evorl_es_cma_get(self.h, _p(Cm), _p(Bm), _p(D), _p(ps), _p(pc), C.byref(sg),
                                      C.byref(gen), C.byref(rc)))
        return dict(C=Cm, B=Bm, D=D, ps=ps, pc=pc, sigma=sg.value, generation=gen.value,
                    recondition_count=rc.value)

    def set_cma_state(self, C_, B, D, ps, pc, sigma, generation, recondition_count=0) -> None:
        arrs = [np.ascontiguousarray(a, np.float64) for a in (C_, B, D, ps, pc)]
        check(self.L.evorl_es_cma_set(self.h, *[_p(a) for a in arrs], float(sigma), int(generation),
                                      int(recondition_count)))


class CmaEs:
    """CMA-ES as free functions on a device state (CmaState::init /
    cmaes_ask / cmaes_tell, proj/src/ec.cpp:191-288): no env or policy, the
    caller supplies the fitness.  State is HBM-resident between calls."""

    def __init__(self, dim: int, pop: int, elites: int = 0, sigma0: float = 0.5, max_dim: int = 4096,
                 eig_every: int = 1, mean0=None):
        self.L = _lib.load()
        h = C.c_void_p()
        check(self.L.evorl_cma_create(int(dim), int(pop), int(elites), float(sigma0), int(max_dim),
                                      int(eig_every), C.byref(h)))
        self.h = h
        self.dim, self.pop = int(dim), int(pop)
        if mean0 is not None:
            self.set_mean(mean0)

    def close(self):
        if getattr(self, "h", None):
            self.L.evorl_es_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def ask(self, key) -> np.ndarray:
        hi, lo = _key(key)
        out = np.empty((self.pop, self.dim), np.float64)
        check(self.L.evorl_cma_ask(self.h, hi, lo, _p(out)))
        return out

    def tell(self, candidates, fitness) -> None:
        x = np.ascontiguousarray(candidates, np.float64)
        f = np.ascontiguousarray(fitness, np.float64)
        if x.shape != (self.pop, self.dim) or f.shape != (self.pop,):
            raise ValueError("cmaes_tell: candidates / fitness shape mismatch")
        check(self.L.evorl_cma_tell(self.h, _p(x), _p(f)))

    def mean(self) -> np.ndarray:
        m = np.empty(self.dim)
        check(self.L.evorl_es_get_mean(self.h, _p(m)))
        return m

    def set_mean(self, m) -> None:
        m = np.ascontiguousarray(m, np.float64)
        if m.shape != (self.dim,):
            raise ValueError("set_mean: size mismatch")
        check(self.L.evorl_es_set_mean(self.h, _p(m)))

    state = EsWorkflow.cma_state
    set_state = EsWorkflow.set_cma_state


# -------------------------------------------------------------- stateless
def mlp_desc(input_dim: int, hidden: Sequence[int], output_dim: int, head: int,
             tanh_scale: float = 1.0, allow_linear: bool = False) -> _lib.MlpDesc:
    m = _lib.MlpDesc()
    m.input_dim = input_dim
    m.n_hidden = len(hidden)
    for i, h in enumerate(hidden):
        m.hidden[i] = h
    m.output_dim = output_dim
    m.layer_norm = 0
    m.head = head
    m.tanh_scale = tanh_scale
    m.allow_linear = int(allow_linear)
    return m


def param_count(desc: _lib.MlpDesc) -> int:
    dims = [desc.input_dim] + [desc.hidden[i] for i in range(desc.n_hidden)] + [desc.output_dim]
    return sum(a * b + b for a, b in zip(dims[:-1], dims[1:]))


def threefry2x64(keys: np.ndarray, ctrs: np.ndarray) -> np.ndarray:
    keys = np.ascontiguousarray(keys, np.uint64).reshape(-1, 2)
    ctrs = np.ascontiguousarray(ctrs, np.uint64).reshape(-1, 2)
    out = np.empty_like(keys)
    check(_lib.load().evorl_threefry2x64(_p(keys), _p(ctrs), _p(out), len(keys)))
    return out


def stream_words(key, first: int, n: int) -> np.ndarray:
    hi, lo = _key(key)
    out = np.empty(n, np.uint64)
    check(_lib.load().evorl_stream_words(hi, lo, first, n, _p(out)))
    return out


def gaussian_matrix(key, rows: int, cols: int) -> np.ndarray:
    """proj/src/ec.cpp:22-28"""
    hi, lo = _key(key)
    out = np.empty((rows, cols), np.float64)
    check(_lib.load().evorl_gaussian_matrix(hi, lo, rows, cols, _p(out)))
    return out


def centered_ranks(f) -> np.ndarray:
    """proj/src/ec.cpp:32-46"""
    f = np.ascontiguousarray(f, np.float64)
    out = np.empty_like(f)
    check(_lib.load().evorl_centered_ranks(_p(f), len(f), _p(out)))
    return out


def rank_desc(f) -> np.ndarray:
    """proj/src/ec.cpp:14-20"""
    f = np.ascontiguousarray(f, np.float64)
    out = np.empty(len(f), np.int32)
    check(_lib.load().evorl_rank_desc(_p(f), len(f), _p(out)))
    return out


def openes_ask(mean, sigma: float, key, n: int, mirrored: bool = True):
    """proj/src/ec.cpp:71-97 -> (candidates, eps)"""
    mean = np.ascontiguousarray(mean, np.float64)
    d = len(mean)
    hi, lo = _key(key)
    cand = np.empty((n, d))
    eps = np.empty((n, d))
    check(_lib.load().evorl_openes_ask(_p(mean), d, sigma, int(mirrored), hi, lo, n, _p(cand),
                                       _p(eps)))
    return cand, eps


def openes_tell(mean, m, v, t: int, sigma: float, lr: float, weight_decay: float, key,
                fitness, mirrored: bool = True):
    """proj/src/ec.cpp:99-109 + proj/src/optim.cpp:7-17, eps regenerated from
    the ask key.  Updates mean, m, v in place; returns the new t."""
    for a in (mean, m, v):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    f = np.ascontiguousarray(fitness, np.float64)
    hi, lo = _key(key)
    tt = C.c_int64(t)
    check(_lib.load().evorl_openes_tell(_p(mean), _p(m), _p(v), C.byref(tt), len(mean), sigma,
                                        lr, weight_decay, int(mirrored), hi, lo, _p(f), len(f)))
    return tt.value


def ars_ask(mean, sigma: float, key, n: int):
    """proj/src/ec.cpp:113-125 -> (deltas, candidates)"""
    mean = np.ascontiguousarray(mean, np.float64)
    d = len(mean)
    hi, lo = _key(key)
    deltas = np.empty((n // 2, d))
    cand = np.empty((n, d))
    check(_lib.load().evorl_ars_ask(_p(mean), d, sigma, hi, lo, n, _p(deltas), _p(cand)))
    return deltas, cand


def ars_tell(mean, elites: int, lr: float, key, fitness) -> bool:
    """proj/src/ec.cpp:127-154 with deltas regenerated from the ask key;
    fitness is the interleaved (r+, r-) vector.  Returns False if skipped."""
    assert mean.dtype == np.float64 and mean.flags.c_contiguous
    f = np.ascontiguousarray(fitness, np.float64)
    hi, lo = _key(key)
    upd = C.c_int32()
    check(_lib.load().evorl_ars_tell(_p(mean), len(mean), elites, lr, hi, lo, _p(f), len(f),
                                     C.byref(upd)))
    return bool(upd.value)


def env_step_batch(env: str, phys, step_count, action, fixed_horizon=False,
                   max_episode_steps=0):
    """proj/src/env.cpp:113-155 for n states (n x 4 phys)."""
    phys = np.ascontiguousarray(phys, np.float64).copy()
    sc = np.ascontiguousarray(step_count, np.int32).copy()
    a = np.ascontiguousarray(action, np.float64)
    n = len(a)
    r = np.empty(n)
    te = np.empty(n, np.int32)
    tr = np.empty(n, np.int32)
    fault = np.empty(n, np.int32)
    eid = _lib.ENV_CARTPOLE if env == "cartpole" else _lib.ENV_PENDULUM
    check(_lib.load().evorl_env_step_batch(eid, int(fixed_horizon), int(max_episode_steps), n,
                                           _p(phys), _p(sc), _p(a), _p(r), _p(te), _p(tr),
                                           _p(fault)))
    return phys, sc, r, te, tr, fault


def batched_rollout(env: str, net: _lib.MlpDesc, params, envs_per_agent: int, key,
                    count: Optional[int] = None, obs_norm=None, fixed_horizon=False,
                    max_episode_steps=0, precision="f64", track_obs_stats=False,
                    collect_transitions=False):
    """proj/src/rollout.cpp:176-214 (Episodes mode, deterministic policy).
    Returns (returns m x count, steps m, obs_stats m x 9 or None); with
    collect_transitions=True instead (returns, steps, batches): per agent the
    reference's AgentRollout::batch as a dict (obs, actions, rewards,
    terminated, truncated, next_obs, lane_bounds), lanes concatenated in order."""
    if collect_transitions:
        return _batched_rollout_transitions(env, net, params, envs_per_agent, key, count, obs_norm,
                                            fixed_horizon, max_episode_steps, precision)
    params = np.ascontiguousarray(params, np.float64)
    m = params.shape[0]
    e = int(envs_per_agent)
    count = e if count is None else int(count)
    ed = _lib.EnvDescC(_lib.ENV_CARTPOLE if env == "cartpole" else _lib.ENV_PENDULUM,
                       int(fixed_horizon), int(max_episode_steps))
    nc = None
    if obs_norm is not None:
        nc = _lib.ObsNormC()
        for k in ("mode", "dim", "count"):
            setattr(nc, k, getattr(obs_norm, k))
        for i in range(4):
            nc.mean[i] = obs_norm.mean[i]
            nc.var[i] = obs_norm.var[i]
    hi, lo = _key(key)
    rets = np.empty((m, count))
    steps = np.empty(m, np.int64)
    stats = np.empty((m, 9)) if track_obs_stats else None
    check(_lib.load().evorl_batched_rollout(
        C.byref(ed), C.byref(net), C.byref(nc) if nc is not None else None, _p(params), m, e,
        count, hi, lo, _lib.PRECISIONS[precision], _p(rets),
        _p(steps), _p(stats) if stats is not None else None))
    return rets, steps, stats


def _norm_c(obs_norm):
    if obs_norm is None:
        return None
    nc = _lib.ObsNormC()
    for k in ("mode", "dim", "count"):
        setattr(nc, k, getattr(obs_norm, k))
    for i in range(4):
        nc.mean[i] = obs_norm.mean[i]
        nc.var[i] = obs_norm.var[i]
    return nc


def _batched_rollout_transitions(env, net, params, envs_per_agent, key, count, obs_norm, fixed_horizon,
                                 max_episode_steps, precision):
    params = np.ascontiguousarray(params, np.float64)
    m, e = params.shape[0], int(envs_per_agent)
    count = e if count is None else int(count)
    ed = _lib.EnvDescC(_lib.ENV_CARTPOLE if env == "cartpole" else _lib.ENV_PENDULUM,
                       int(fixed_horizon), int(max_episode_steps))
    od = 4 if env == "cartpole" else 3
    H = int(max_episode_steps) if max_episode_steps else (500 if env == "cartpole" else 200)
    cap = -(-count // e) * H
    rows = m * e * cap
    nc = _norm_c(obs_norm)
    hi, lo = _key(key)
    rets, steps = np.empty((m, count)), np.empty(m, np.int64)
    obs, nxt = np.empty((rows, od)), np.empty((rows, od))
    act, rew = np.empty(rows), np.empty(rows)
    term, trunc = np.empty(rows, np.uint8), np.empty(rows, np.uint8)
    lane_rows = np.empty(m * e, np.int64)
    check(_lib.load().evorl_batched_rollout_transitions(
        C.byref(ed), C.byref(net), C.byref(nc) if nc is not None else None, _p(params), m, e, count,
        hi, lo, _lib.PRECISIONS[precision], _p(rets), _p(steps), cap, _p(obs), _p(act), _p(rew),
        _p(term), _p(trunc), _p(nxt), _p(lane_rows)))
    batches = []
    for a in range(m):
        sel = np.concatenate([np.arange(l * cap, l * cap + lane_rows[l]) for l in range(a * e, (a + 1) * e)])
        bounds = np.concatenate([[0], np.cumsum(lane_rows[a * e:(a + 1) * e])])
        batches.append(dict(obs=obs[sel], actions=act[sel].reshape(-1, 1), rewards=rew[sel],
                            terminated=term[sel], truncated=trunc[sel], next_obs=nxt[sel],
                            lane_bounds=bounds))
    return rets, steps, batches


def sym_eig(A):
    """Device Jacobi eigensolver (replaces Eigen::SelfAdjointEigenSolver,
    proj/src/ec.cpp:278-287) -> (evals ascending, vecs with vecs[:, j] the j-th
    eigenvector, largest-|.| component positive, sweeps)."""
    A = np.ascontiguousarray(A, np.float64)
    n = A.shape[0]
    ev = np.empty(n)
    V = np.empty((n, n))
    sw = C.c_int32()
    check(_lib.load().evorl_sym_eig(_p(A), n, _p(ev), _p(V), C.byref(sw)))
    return ev, V, sw.value


def pinned_empty(n: int) -> np.ndarray:
    """A float64 array of n entries in page-locked host memory
    (evorl_host_alloc; freed with the array)."""
    import weakref
    L = _lib.load()
    p = C.c_void_p()
    check(L.evorl_host_alloc(int(n) * 8, C.byref(p)))
    buf = (C.c_double * int(n)).from_address(p.value)
    weakref.finalize(buf, L.evorl_host_free, p.value)
    return np.frombuffer(buf, dtype=np.float64)


def measure_noise_rate(n: int = 1 << 27) -> float:
    """Normals/s of the ask's noise generator at full occupancy (n normals)."""
    ms = C.c_float()
    check(_lib.load().evorl_measure_noise_rate(int(n), C.byref(ms)))
    return n / (ms.value * 1e-3)


def measure_fp64_peak() -> float:
    t = C.c_double()
    check(_lib.load().evorl_measure_fp64_peak(C.byref(t)))
    return t.value
