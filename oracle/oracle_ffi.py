"""ctypes binding of the CPU parity oracle (oracle/_build/libevorl_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, by ``__graft_entry__.smoke()``
as the checker, and by bench.py's ``cpu_baseline`` / ``--impl reference``
legs.  The product package ``paper_2501_15129_b200`` never imports this.

Struct layouts mirror ``oracle/evorl_oracle.h`` field for field.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libevorl_oracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libevorl_ref.so")

EO_CARTPOLE, EO_PENDULUM = 0, 1
EO_HEAD_TANH, EO_HEAD_GAUSSIAN, EO_HEAD_CATEGORICAL, EO_HEAD_LINEAR = 0, 1, 2, 3
EO_NORM_NONE, EO_NORM_VBN, EO_NORM_RS = 0, 1, 2
EO_ALGO = {"openes": 0, "ars": 1, "ves": 2, "cmaes": 3, "cem": 4}
EO_ACT_DETERMINISTIC, EO_ACT_STOCHASTIC, EO_ACT_UNIFORM = 0, 1, 2
EO_MODE_EPISODES, EO_MODE_STEPS = 0, 1
MAX_HIDDEN = 8


class Key(C.Structure):
    _fields_ = [("hi", C.c_uint64), ("lo", C.c_uint64)]

    def t(self):
        return (self.hi, self.lo)


class Stream(C.Structure):
    _fields_ = [("key", Key), ("block", C.c_uint64), ("pending_word", C.c_uint64),
                ("has_pending_word", C.c_int), ("pending_normal", C.c_double),
                ("has_pending_normal", C.c_int)]


class EnvSpec(C.Structure):
    _fields_ = [("id", C.c_int), ("obs_dim", C.c_int), ("discrete", C.c_int),
                ("num_actions", C.c_int), ("act_dim", C.c_int), ("act_low", C.c_double),
                ("act_high", C.c_double), ("max_episode_steps", C.c_int),
                ("fixed_horizon", C.c_int)]


class EnvState(C.Structure):
    _fields_ = [("phys", C.c_double * 4), ("step_count", C.c_int), ("rng", Key)]


class MlpSpec(C.Structure):
    _fields_ = [("input_dim", C.c_int), ("n_hidden", C.c_int), ("hidden", C.c_int * MAX_HIDDEN),
                ("output_dim", C.c_int), ("layer_norm", C.c_int), ("head", C.c_int),
                ("tanh_scale", C.c_double), ("min_logstd", C.c_double),
                ("max_logstd", C.c_double), ("allow_linear", C.c_int)]


class Welford(C.Structure):
    _fields_ = [("count", C.c_double), ("dim", C.c_int), ("mean", C.c_double * 4),
                ("m2", C.c_double * 4)]


class ObsNorm(C.Structure):
    _fields_ = [("mode", C.c_int), ("dim", C.c_int), ("mean", C.c_double * 4),
                ("var", C.c_double * 4), ("count", C.c_double)]


class AdamCfg(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double)]


class OpenEsCfg(C.Structure):
    _fields_ = [("pop", C.c_int), ("sigma", C.c_double), ("lr", C.c_double),
                ("weight_decay", C.c_double), ("mirrored", C.c_int), ("noise_table", C.c_int),
                ("noise_table_size", C.c_int64)]


class OpenEsState(C.Structure):
    _fields_ = [("cfg", OpenEsCfg), ("d", C.c_int64), ("mean", C.POINTER(C.c_double)),
                ("sigma", C.c_double), ("m", C.POINTER(C.c_double)),
                ("v", C.POINTER(C.c_double)), ("t", C.c_int64), ("table_seed", C.c_uint64),
                ("table", C.POINTER(C.c_double))]


class ArsCfg(C.Structure):
    _fields_ = [("pop", C.c_int), ("elites", C.c_int), ("sigma", C.c_double), ("lr", C.c_double)]


class VesCfg(C.Structure):
    _fields_ = [("pop", C.c_int), ("elites", C.c_int), ("sigma", C.c_double),
                ("mirrored", C.c_int)]


class CmaCfg(C.Structure):
    _fields_ = [("pop", C.c_int), ("elites", C.c_int), ("sigma0", C.c_double),
                ("max_dim", C.c_int)]


class CmaState(C.Structure):
    _fields_ = [("cfg", CmaCfg), ("dim", C.c_int), ("mean", C.POINTER(C.c_double)),
                ("sigma", C.c_double), ("C", C.POINTER(C.c_double)),
                ("B", C.POINTER(C.c_double)), ("D", C.POINTER(C.c_double)),
                ("ps", C.POINTER(C.c_double)), ("pc", C.POINTER(C.c_double)),
                ("weights", C.POINTER(C.c_double)), ("mu", C.c_int), ("mueff", C.c_double),
                ("cs", C.c_double), ("ds", C.c_double), ("cc", C.c_double), ("c1", C.c_double),
                ("cmu", C.c_double), ("chi_n", C.c_double), ("generation", C.c_int64),
                ("recondition_count", C.c_int64)]


class CemCfg(C.Structure):
    _fields_ = [("pop", C.c_int), ("elites", C.c_int), ("var_init", C.c_double),
                ("noise_start", C.c_double), ("noise_end", C.c_double),
                ("decay_iters", C.c_int64)]


class Policy(C.Structure):
    _fields_ = [("spec", C.POINTER(MlpSpec)), ("obs_norm", C.POINTER(ObsNorm)), ("mode", C.c_int),
                ("exploration_noise", C.c_double)]


class AgentRollout(C.Structure):
    _fields_ = [("steps", C.c_int64), ("n_episodes", C.c_int),
                ("episode_returns", C.POINTER(C.c_double)),
                ("episode_lengths", C.POINTER(C.c_int)), ("obs_stats", Welford),
                ("n_rows", C.c_int64), ("t_obs", C.POINTER(C.c_double)),
                ("t_act", C.POINTER(C.c_double)), ("t_rew", C.POINTER(C.c_double)),
                ("t_term", C.POINTER(C.c_uint8)), ("t_trunc", C.POINTER(C.c_uint8)),
                ("t_next", C.POINTER(C.c_double)), ("lane_bounds", C.POINTER(C.c_int64))]


class EsConfig(C.Structure):
    _fields_ = [("algo", C.c_int), ("env_id", C.c_int), ("fixed_horizon", C.c_int),
                ("max_episode_steps", C.c_int), ("n_hidden", C.c_int),
                ("hidden", C.c_int * MAX_HIDDEN), ("layer_norm", C.c_int),
                ("allow_linear", C.c_int), ("pop", C.c_int), ("fitness_episodes", C.c_int),
                ("obs_norm_mode", C.c_int), ("vbn_samples", C.c_int), ("openes", OpenEsCfg),
                ("ars", ArsCfg), ("ves", VesCfg), ("cma", CmaCfg), ("cem", CemCfg),
                ("workers", C.c_int)]


class StepMetrics(C.Structure):
    _fields_ = [("fitness_mean", C.c_double), ("fitness_max", C.c_double),
                ("fitness_min", C.c_double), ("sigma", C.c_double),
                ("update_skipped", C.c_double)]


_lib = None
_ref = None


def build(ref: bool = True) -> None:
    """Compile the oracle (and, when /root/reference exists, the reference RNG)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj"):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(ref=False)
        L = C.CDLL(LIB_PATH)
        L.eo_last_error.restype = C.c_char_p
        L.eo_key_from_seed.restype = Key
        L.eo_key_from_seed.argtypes = [C.c_uint64]
        L.eo_fold_in.restype = Key
        L.eo_fold_in.argtypes = [Key, C.c_uint64]
        L.eo_init_key.restype = Key
        L.eo_init_key.argtypes = [Key, C.c_uint64]
        L.eo_next_u64.restype = C.c_uint64
        L.eo_uniform.restype = C.c_double
        L.eo_uniform_range.restype = C.c_double
        L.eo_uniform_range.argtypes = [C.POINTER(Stream), C.c_double, C.c_double]
        L.eo_normal.restype = C.c_double
        L.eo_randint.restype = C.c_uint64
        L.eo_randint.argtypes = [C.POINTER(Stream), C.c_uint64]
        L.eo_stream_init.argtypes = [C.POINTER(Stream), Key]
        L.eo_gaussian_matrix.argtypes = [Key, C.c_int64, C.c_int64, C.c_void_p]
        L.eo_env_cartpole.restype = EnvSpec
        L.eo_env_pendulum.restype = EnvSpec
        L.eo_env_reset.argtypes = [C.POINTER(EnvSpec), Key, C.POINTER(EnvState), C.c_void_p]
        L.eo_param_count.restype = C.c_int64
        L.eo_init_params.argtypes = [C.POINTER(MlpSpec), Key, C.c_void_p]
        L.eo_policy_net_spec.restype = MlpSpec
        L.eo_obs_norm_none.restype = ObsNorm
        L.eo_obs_norm_running_stats.restype = ObsNorm
        L.eo_obs_norm_from_stats.restype = ObsNorm
        L.eo_adam_default.restype = AdamCfg
        L.eo_openes_default.restype = OpenEsCfg
        L.eo_ars_default.restype = ArsCfg
        L.eo_ves_default.restype = VesCfg
        L.eo_cma_default.restype = CmaCfg
        L.eo_cem_default.restype = CemCfg
        L.eo_es_default_config.restype = EsConfig
        L.eo_vbn_fit.restype = ObsNorm
        L.eo_vbn_fit.argtypes = [C.POINTER(EnvSpec), Key, C.c_int]
        L.eo_openes_init.argtypes = [C.POINTER(OpenEsState), C.POINTER(OpenEsCfg), C.c_void_p,
                                     C.c_int64, Key]
        L.eo_openes_ask.argtypes = [C.POINTER(OpenEsState), Key, C.c_int, C.c_void_p, C.c_void_p]
        L.eo_ars_ask.argtypes = [C.c_void_p, C.c_int64, C.c_double, Key, C.c_int, C.c_void_p,
                                 C.c_void_p]
        L.eo_ars_tell.argtypes = [C.c_void_p, C.c_int64, C.POINTER(ArsCfg), C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_int]
        L.eo_ves_ask.argtypes = [C.c_void_p, C.c_int64, C.POINTER(VesCfg), Key, C.c_int,
                                 C.c_void_p]
        L.eo_cma_init.argtypes = [C.POINTER(CmaState), C.POINTER(CmaCfg), C.c_void_p, C.c_int64]
        L.eo_cma_ask.argtypes = [C.POINTER(CmaState), Key, C.c_int, C.c_void_p]
        L.eo_rollout_lane.argtypes = [C.POINTER(EnvSpec), C.POINTER(Policy), C.c_void_p, C.c_int,
                                      C.c_int, C.c_int, Key, C.c_int, C.c_int, C.POINTER(AgentRollout)]
        L.eo_batched_rollout_ex.argtypes = [C.c_int, C.POINTER(EnvSpec), C.POINTER(Policy), C.c_void_p,
                                            C.c_int, C.c_int, C.c_int, C.c_int, Key, C.c_int, C.c_int,
                                            C.POINTER(AgentRollout)]
        L.eo_batched_rollout.argtypes = [C.c_int, C.POINTER(EnvSpec), C.POINTER(Policy),
                                         C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, Key,
                                         C.c_int, C.POINTER(AgentRollout)]
        L.eo_es_create.argtypes = [C.POINTER(EsConfig), C.POINTER(C.c_void_p)]
        L.eo_es_destroy.argtypes = [C.c_void_p]
        L.eo_es_init.argtypes = [C.c_void_p, Key]
        L.eo_es_step.argtypes = [C.c_void_p, C.POINTER(StepMetrics)]
        for f in ("eo_es_dim", "eo_es_iteration", "eo_es_env_steps", "eo_es_episodes"):
            getattr(L, f).restype = C.c_int64
            getattr(L, f).argtypes = [C.c_void_p]
        L.eo_es_get_mean.argtypes = [C.c_void_p, C.c_void_p]
        L.eo_es_set_mean.argtypes = [C.c_void_p, C.c_void_p]
        L.eo_es_get_adam.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)]
        L.eo_es_get_fitness.argtypes = [C.c_void_p, C.c_void_p]
        L.eo_es_get_obs_norm.argtypes = [C.c_void_p, C.POINTER(ObsNorm)]
        L.eo_es_set_obs_norm.argtypes = [C.c_void_p, C.POINTER(ObsNorm)]
        L.eo_es_net.restype = C.POINTER(MlpSpec)
        L.eo_es_net.argtypes = [C.c_void_p]
        L.eo_es_env.restype = C.POINTER(EnvSpec)
        L.eo_es_env.argtypes = [C.c_void_p]
        L.eo_es_cma.restype = C.POINTER(CmaState)
        L.eo_es_cma.argtypes = [C.c_void_p]
        L.eo_es_step_key.restype = Key
        L.eo_es_step_key.argtypes = [C.c_void_p]
        L.eo_es_eval_key.restype = Key
        L.eo_es_eval_key.argtypes = [C.c_void_p]
        L.eo_es_evaluate.argtypes = [C.c_void_p, C.c_int, Key, C.POINTER(C.c_double),
                                     C.POINTER(C.c_double)]
        _lib = L
    return _lib


def ref_lib():
    """The reference's own rng.cpp (oracle/_ref); None when it was not built."""
    global _ref
    if _ref is None and os.path.exists(REF_PATH):
        _ref = C.CDLL(REF_PATH)
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def check(rc):
    if rc != 0:
        raise OracleError(rc, lib().eo_last_error().decode())
    return rc


def ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------ conveniences
def key_from_seed(seed: int) -> Key:
    return lib().eo_key_from_seed(seed)


def fold_in(key: Key, i: int) -> Key:
    return lib().eo_fold_in(key, i)


def threefry(key, ctr):
    k = (C.c_uint64 * 2)(*key)
    c = (C.c_uint64 * 2)(*ctr)
    o = (C.c_uint64 * 2)()
    lib().eo_threefry2x64(k, c, o)
    return (o[0], o[1])


def stream(key: Key) -> Stream:
    s = Stream()
    lib().eo_stream_init(C.byref(s), key)
    return s


def gaussian_matrix(key: Key, rows: int, cols: int) -> np.ndarray:
    out = np.empty((rows, cols), np.float64)
    lib().eo_gaussian_matrix(key, rows, cols, ptr(out))
    return out


def mlp_spec(input_dim, hidden, output_dim, head, tanh_scale=1.0, layer_norm=False,
             allow_linear=False) -> MlpSpec:
    s = MlpSpec()
    s.input_dim = input_dim
    s.n_hidden = len(hidden)
    for i, h in enumerate(hidden):
        s.hidden[i] = h
    s.output_dim = output_dim
    s.layer_norm = int(layer_norm)
    s.head = head
    s.tanh_scale = tanh_scale
    s.min_logstd = -20.0
    s.max_logstd = 2.0
    s.allow_linear = int(allow_linear)
    return s


def env_spec(name: str, fixed_horizon=False, max_episode_steps=0) -> EnvSpec:
    L = lib()
    if name == "cartpole":
        return L.eo_env_cartpole(int(fixed_horizon), int(max_episode_steps))
    if name == "pendulum":
        return L.eo_env_pendulum(int(fixed_horizon), int(max_episode_steps))
    raise ValueError(f"unknown env id: {name}")


def policy_net_spec(env: EnvSpec, hidden, layer_norm=False, allow_linear=False) -> MlpSpec:
    h = (C.c_int * MAX_HIDDEN)(*hidden)
    s = lib().eo_policy_net_spec(C.byref(env), h, len(hidden), int(layer_norm))
    s.allow_linear = int(allow_linear)
    return s


def param_count(spec: MlpSpec) -> int:
    return lib().eo_param_count(C.byref(spec))


def init_params(spec: MlpSpec, key: Key) -> np.ndarray:
    n = param_count(spec)
    if n < 0:
        raise OracleError(1, lib().eo_last_error().decode())
    p = np.empty(n, np.float64)
    check(lib().eo_init_params(C.byref(spec), key, ptr(p)))
    return p


def forward(spec: MlpSpec, params: np.ndarray, x) -> np.ndarray:
    out = np.empty(spec.output_dim, np.float64)
    xx = np.ascontiguousarray(x, np.float64)
    check(lib().eo_forward(C.byref(spec), ptr(params), ptr(xx), ptr(out)))
    return out


def centered_ranks(f) -> np.ndarray:
    f = np.ascontiguousarray(f, np.float64)
    out = np.empty_like(f)
    lib().eo_centered_ranks(ptr(f), C.c_int64(len(f)), ptr(out))
    return out


def rank_desc(f) -> np.ndarray:
    f = np.ascontiguousarray(f, np.float64)
    out = np.empty(len(f), np.int32)
    lib().eo_rank_desc(ptr(f), C.c_int64(len(f)), ptr(out))
    return out


def es_config(**kw) -> EsConfig:
    """EsConfig from reference config-key style keyword names."""
    c = lib().eo_es_default_config()
    for k, v in kw.items():
        if k == "algo":
            c.algo = EO_ALGO[v]
        elif k == "env":
            c.env_id = EO_CARTPOLE if v == "cartpole" else EO_PENDULUM
        elif k == "hidden":
            c.n_hidden = len(v)
            for i, h in enumerate(v):
                c.hidden[i] = h
        elif "." in k:
            a, b = k.split(".")
            setattr(getattr(c, a), b, v)
        else:
            setattr(c, k, v)
    return c


class OracleEs:
    """CPU EsWorkflow (init/step/evaluate) -- the generation-level oracle."""

    def __init__(self, cfg: EsConfig):
        self.L = lib()
        self.cfg = cfg
        h = C.c_void_p()
        check(self.L.eo_es_create(C.byref(cfg), C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.L.eo_es_destroy(self.h)
            self.h = None

    @property
    def dim(self):
        return self.L.eo_es_dim(self.h)

    def init(self, key: Key):
        check(self.L.eo_es_init(self.h, key))

    def step(self) -> StepMetrics:
        m = StepMetrics()
        check(self.L.eo_es_step(self.h, C.byref(m)))
        return m

    def mean(self) -> np.ndarray:
        out = np.empty(self.dim, np.float64)
        self.L.eo_es_get_mean(self.h, ptr(out))
        return out

    def set_mean(self, mean):
        m = np.ascontiguousarray(mean, np.float64)
        self.L.eo_es_set_mean(self.h, ptr(m))

    def adam(self):
        m = np.empty(self.dim, np.float64)
        v = np.empty(self.dim, np.float64)
        t = C.c_int64()
        check(self.L.eo_es_get_adam(self.h, ptr(m), ptr(v), C.byref(t)))
        return m, v, t.value

    def fitness(self) -> np.ndarray:
        out = np.empty(self.cfg.pop, np.float64)
        self.L.eo_es_get_fitness(self.h, ptr(out))
        return out

    def obs_norm(self) -> ObsNorm:
        o = ObsNorm()
        self.L.eo_es_get_obs_norm(self.h, C.byref(o))
        return o

    def set_obs_norm(self, o: ObsNorm):
        self.L.eo_es_set_obs_norm(self.h, C.byref(o))

    def counters(self):
        return (self.L.eo_es_iteration(self.h), self.L.eo_es_env_steps(self.h),
                self.L.eo_es_episodes(self.h))

    def step_key(self) -> Key:
        return self.L.eo_es_step_key(self.h)

    def eval_key(self) -> Key:
        return self.L.eo_es_eval_key(self.h)

    def evaluate(self, episodes: int, key: Key):
        mr = C.c_double()
        sd = C.c_double()
        check(self.L.eo_es_evaluate(self.h, episodes, key, C.byref(mr), C.byref(sd)))
        return mr.value, sd.value

    def cma(self) -> CmaState:
        return self.L.eo_es_cma(self.h).contents

    def net(self) -> MlpSpec:
        return self.L.eo_es_net(self.h).contents

    def env(self) -> EnvSpec:
        return self.L.eo_es_env(self.h).contents


def batched_rollout(env: EnvSpec, spec: MlpSpec, obs_norm, params: np.ndarray, e: int,
                    key: Key, count=None, track=False, workers=1, collect=False):
    """Returns (returns list per agent, steps per agent, obs_stats per agent) and,
    with collect=True, a 4th item: per agent a dict SampleBatch (obs, actions,
    rewards, terminated, truncated, next_obs, lane_bounds)."""
    m = params.shape[0]
    params = np.ascontiguousarray(params, np.float64)
    ptrs = (C.c_void_p * m)(*[params.ctypes.data + i * params.strides[0] for i in range(m)])
    pol = Policy()
    pol.spec = C.pointer(spec)
    pol.obs_norm = C.pointer(obs_norm) if obs_norm is not None else None
    pol.mode = EO_ACT_DETERMINISTIC
    out = (AgentRollout * m)()
    count = e if count is None else count
    check(lib().eo_batched_rollout_ex(workers, C.byref(env), C.byref(pol), ptrs, m, e,
                                      EO_MODE_EPISODES, count, key, int(track), int(collect), out))
    rets, steps, stats, batches = [], [], [], []
    od, ad = env.obs_dim, env.act_dim
    for a in range(m):
        r = out[a]
        rets.append(np.array([r.episode_returns[i] for i in range(r.n_episodes)]))
        steps.append(r.steps)
        stats.append((r.obs_stats.count, list(r.obs_stats.mean), list(r.obs_stats.m2)))
        if collect:
            n = r.n_rows

            def arr(ptr, k, dt=np.float64):
                return np.ctypeslib.as_array(ptr, shape=(max(k, 1),))[:k].astype(dt) if k else np.zeros(0, dt)
            batches.append(dict(obs=arr(r.t_obs, n * od).reshape(n, od), actions=arr(r.t_act, n * ad).reshape(n, ad),
                                rewards=arr(r.t_rew, n), terminated=arr(r.t_term, n, np.uint8),
                                truncated=arr(r.t_trunc, n, np.uint8), next_obs=arr(r.t_next, n * od).reshape(n, od),
                                lane_bounds=arr(r.lane_bounds, e + 1, np.int64)))
        lib().eo_agent_rollout_free(C.byref(r))
    if collect:
        return rets, steps, stats, batches
    return rets, steps, stats
