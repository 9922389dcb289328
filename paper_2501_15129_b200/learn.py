"""The caller side of the generation step: ``learn()`` and the JSONL metrics
stream.

``learn`` drives ``EsWorkflow.step`` until a budget is reached, evaluating the
centre every ``eval_interval`` iterations with the reference's eval key and
checkpointing on the reference's schedule (proj/src/workflow.cpp:46-68,
proj/include/evorl/workflow.hpp:42, :74-92).  ``MetricsWriter`` writes the
reference's two files (proj/src/metrics.cpp:12-67): ``metrics.jsonl``, one
JSON object per line with keys sorted and no whitespace (nlohmann::json
``dump()`` over a std::map), a pure function of (config, seed); and the
``timings.log`` sidecar (``iteration<TAB>wall_ms``, iostream default
formatting).

Number formatting follows nlohmann::json's serializer (the reference's
json.hpp is an un-vendored third-party header, nlohmann/json, version
unpinned): integers verbatim; doubles as the shortest round-trip digit string
placed by ``dtoa_impl::format_buffer`` (plain notation for decimal exponents
in (-4, 15], else ``d.ddde+XX`` with at least two exponent digits; integral
values get ``.0``); non-finite doubles as ``null``.  nlohmann's Grisu2 is
not guaranteed shortest in every case; Python's ``repr`` is, so a rare
value may differ in its last digit string while parsing to the same double.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from decimal import Decimal
from typing import Mapping, Optional

from .es import EsConfig, EsWorkflow


# --------------------------------------------------------- JSON (nlohmann)
def _json_double(x: float) -> str:
    if not math.isfinite(x):
        return "null"
    if x == 0.0:
        return "-0.0" if math.copysign(1.0, x) < 0 else "0.0"
    sign, digits, exp = Decimal(repr(abs(x))).as_tuple()
    ds = "".join(map(str, digits)).rstrip("0")
    exp += len(digits) - len(ds)
    k = len(ds)
    n = k + exp  # decimal point position (value = 0.ds * 10^n)
    neg = "-" if x < 0 else ""
    if k <= n <= 15:
        return neg + ds + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return neg + ds[:n] + "." + ds[n:]
    if -4 < n <= 0:
        return neg + "0." + "0" * (-n) + ds
    e = n - 1
    mant = ds if k == 1 else ds[0] + "." + ds[1:]
    return neg + mant + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"


def _json_string(s: str) -> str:
    out = ['"']
    for ch in s:
        o = ord(ch)
        if ch == '"':
            out.append('\\"')
        elif ch == "\\":
            out.append("\\\\")
        elif ch == "\b":
            out.append("\\b")
        elif ch == "\f":
            out.append("\\f")
        elif ch == "\n":
            out.append("\\n")
        elif ch == "\r":
            out.append("\\r")
        elif ch == "\t":
            out.append("\\t")
        elif o < 0x20:
            out.append(f"\\u{o:04x}")
        else:
            out.append(ch)
    out.append('"')
    return "".join(out)


def dump_json(v) -> str:
    """nlohmann::json::dump() of an object built from dict / str / int /
    float / bool (std::map key order = byte-wise sorted keys)."""
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, int):
        return str(v)
    if isinstance(v, float):
        return _json_double(v)
    if isinstance(v, str):
        return _json_string(v)
    if v is None:
        return "null"
    if isinstance(v, Mapping):
        items = sorted(v.items(), key=lambda kv: kv[0].encode())
        return "{" + ",".join(_json_string(k) + ":" + dump_json(x) for k, x in items) + "}"
    raise TypeError(f"not JSON-serialisable here: {type(v).__name__}")


def _iostream_double(x: float) -> str:
    """operator<<(double) with the default precision 6 (%g)."""
    return "%g" % x


# --------------------------------------------------------------- writer
class MetricsWriter:
    """MetricsWriter (proj/include/evorl/metrics.hpp, proj/src/metrics.cpp)."""

    def __init__(self, metrics_path: str, timings_path: str):
        try:
            self._m = open(metrics_path, "w", encoding="utf-8", newline="\n")
        except OSError:
            raise RuntimeError("cannot open metrics file: " + metrics_path) from None
        try:
            self._t = open(timings_path, "w", encoding="utf-8", newline="\n")
        except OSError:
            self._m.close()
            raise RuntimeError("cannot open timings file: " + timings_path) from None

    def write_header(self, workflow_id: str, config: Mapping[str, str]) -> None:
        self._m.write(dump_json({"type": "header", "workflow": workflow_id,
                                 "config": {str(k): str(v) for k, v in config.items()}}) + "\n")
        self.flush()

    def write_step(self, iteration: int, env_steps: int, episodes: int, rl_updates: int,
                   extra: Mapping[str, float]) -> None:
        rec = {"type": "step", "iteration": int(iteration), "env_steps": int(env_steps),
               "episodes": int(episodes), "rl_updates": int(rl_updates)}
        for k, x in extra.items():  # StepMetrics scalars are doubles
            rec[k] = float(x)
        self._m.write(dump_json(rec) + "\n")

    def write_eval(self, iteration: int, env_steps: int, episodes: int, rl_updates: int,
                   mean_return: float, return_std: float, eval_episodes: int) -> None:
        self._m.write(dump_json({
            "type": "eval", "iteration": int(iteration), "env_steps": int(env_steps),
            "episodes": int(episodes), "rl_updates": int(rl_updates),
            "eval/episode_return_mean": float(mean_return), "eval/episode_return_std": float(return_std),
            "eval/episodes": int(eval_episodes)}) + "\n")
        self.flush()

    def write_timing(self, iteration: int, wall_ms: float) -> None:
        self._t.write(f"{int(iteration)}\t{_iostream_double(float(wall_ms))}\n")

    def flush(self) -> None:
        self._m.flush()
        self._t.flush()

    def close(self) -> None:
        self.flush()
        self._m.close()
        self._t.close()


# ------------------------------------------------------------ learn loop
@dataclass
class Budget:
    """Budget (proj/include/evorl/workflow.hpp:74-84); 0 = off."""
    iterations: int = 0
    episodes: int = 0
    env_steps: int = 0

    def reached(self, iteration: int, env_steps: int, episodes: int) -> bool:
        return ((self.iterations > 0 and iteration >= self.iterations)
                or (self.episodes > 0 and episodes >= self.episodes)
                or (self.env_steps > 0 and env_steps >= self.env_steps))


@dataclass
class LearnOptions:
    """LearnOptions (proj/include/evorl/workflow.hpp:86-92)."""
    budget: Budget
    eval_interval: int = 10
    eval_episodes: int = 128
    checkpoint_interval: int = 0
    checkpoint_path: str = ""


def _fold_in(key, i: int) -> tuple:
    """fold_in (proj/src/rng.cpp:43-46) through the library's Threefry."""
    from .es import threefry2x64
    hi, lo = (key.hi, key.lo) if hasattr(key, "hi") else key
    out = threefry2x64([int(hi), int(lo)], [0, int(i)])[0]
    return int(out[0]), int(out[1])


def key_from_seed(seed: int) -> tuple:
    """key_from_seed (proj/src/rng.cpp:36-41)."""
    return _fold_in((0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B), seed)


def eval_key(rng, iteration: int) -> tuple:
    """WorkflowState::eval_key = fold_in(fold_in(rng, 1), iteration)
    (proj/include/evorl/workflow.hpp:42)."""
    return _fold_in(_fold_in(rng, 1), iteration)


def learn(wf: EsWorkflow, rng, opt: LearnOptions, metrics: MetricsWriter, clock=None) -> None:
    """learn() (proj/src/workflow.cpp:46-68) over the device workflow.  Eval
    keys come from the handle's own WorkflowState::rng (``wf.rng()``, the key
    of init() or of the loaded checkpoint), as WorkflowState::eval_key does
    (proj/include/evorl/workflow.hpp:42); ``rng`` may be None, and a key that
    differs from the state's raises ValueError instead of silently producing
    other eval records.  Wall time per step is measured on the host around the
    blocking ``step`` call, as the reference does with steady_clock."""
    import time
    clock = clock or time.perf_counter
    state_rng = wf.rng()
    if rng is not None:
        hi, lo = (rng.hi, rng.lo) if hasattr(rng, "hi") else rng
        if (int(hi), int(lo)) != state_rng:
            raise ValueError(f"learn(): rng {(int(hi), int(lo))} is not the workflow state's key "
                             f"{state_rng} (eval keys derive from WorkflowState::rng)")
    rng = state_rng
    while True:
        it, steps, eps = wf.counters()
        if opt.budget.reached(it, steps, eps):
            break
        t0 = clock()
        sm = wf.step()
        ms = (clock() - t0) * 1e3
        it, steps, eps = wf.counters()
        metrics.write_step(it, steps, eps, 0, sm.values)
        metrics.write_timing(it, ms)
        if opt.eval_interval > 0 and it % opt.eval_interval == 0:
            mr, sd = wf.evaluate(opt.eval_episodes, eval_key(rng, it))
            metrics.write_eval(it, steps, eps, 0, mr, sd, opt.eval_episodes)
        if opt.checkpoint_interval > 0 and opt.checkpoint_path and it % opt.checkpoint_interval == 0:
            wf.save(opt.checkpoint_path)
    if opt.checkpoint_path:
        wf.save(opt.checkpoint_path)
    metrics.flush()


def es_config_entries(cfg: EsConfig, seed: Optional[int] = None, budget: Optional[Budget] = None,
                      eval_interval: int = 10, eval_episodes: int = 128) -> dict:
    """The ES-workflow subset of Config::describe() (proj/src/config.cpp:305-314):
    registry key -> value string for the keys this path reads (other
    workflows' keys are out of scope).  Values use the registry's spelling
    (``true``/``false``, ``64,64``)."""
    b = budget or Budget(iterations=2000)
    # a value equal to the registry default keeps the registry's spelling
    # (proj/src/config.cpp:23-70: "1e-3", "4194304", ...)
    spelled = {"ec.cem.var_init": "1e-3", "ec.cem.noise_start": "1e-3", "ec.cem.noise_end": "1e-5"}

    def f(x, key=None):
        if key in spelled and float(x) == float(spelled[key]):
            return spelled[key]
        return repr(float(x))
    t = lambda x: "true" if x else "false"
    out = {
        "workflow": "es", "env.id": cfg.env, "env.fixed_horizon": t(cfg.fixed_horizon),
        "env.max_episode_steps": str(cfg.max_episode_steps), "net.hidden": ",".join(map(str, cfg.hidden)),
        "net.layer_norm": t(cfg.layer_norm), "budget.iterations": str(b.iterations),
        "budget.episodes": str(b.episodes), "budget.env_steps": str(b.env_steps),
        "eval.interval": str(eval_interval), "eval.episodes": str(eval_episodes),
        "obs_norm.mode": cfg.obs_norm, "obs_norm.vbn_samples": str(cfg.vbn_samples), "ec.algo": cfg.algo,
        "ec.pop": str(cfg.pop), "ec.fitness_episodes": str(cfg.fitness_episodes),
        "ec.openes.sigma": f(cfg.openes_sigma), "ec.openes.lr": f(cfg.openes_lr),
        "ec.openes.weight_decay": f(cfg.openes_weight_decay), "ec.openes.mirrored": t(cfg.openes_mirrored),
        "ec.openes.noise_table": t(cfg.openes_noise_table),
        "ec.openes.noise_table_size": str(cfg.openes_noise_table_size), "ec.ars.sigma": f(cfg.ars_sigma),
        "ec.ars.lr": f(cfg.ars_lr), "ec.ars.elites": str(cfg.ars_elites), "ec.ves.sigma": f(cfg.ves_sigma),
        "ec.ves.elites": str(cfg.ves_elites), "ec.ves.mirrored": t(cfg.ves_mirrored),
        "ec.cmaes.sigma0": f(cfg.cmaes_sigma0), "ec.cmaes.elites": str(cfg.cmaes_elites),
        "ec.cmaes.max_dim": str(cfg.cmaes_max_dim), "ec.cem.elites": str(cfg.cem_elites),
        "ec.cem.var_init": f(cfg.cem_var_init, "ec.cem.var_init"),
        "ec.cem.noise_start": f(cfg.cem_noise_start, "ec.cem.noise_start"),
        "ec.cem.noise_end": f(cfg.cem_noise_end, "ec.cem.noise_end"), "ec.cem.decay_iters": str(cfg.cem_decay_iters),
    }
    if seed is not None:
        out["seed"] = str(seed)
    return out


def run(cfg: EsConfig, seed: int, out_dir: str, opt: LearnOptions) -> EsWorkflow:
    """The runner's ES path (proj/src/runner.cpp:50-80): root key
    key_from_seed(seed), metrics.jsonl / timings.log header, learn, and the
    checkpoint at out_dir/checkpoint.bin."""
    os.makedirs(out_dir, exist_ok=True)
    root = key_from_seed(seed)
    wf = EsWorkflow(cfg).init(root)
    if not opt.checkpoint_path:
        opt = LearnOptions(opt.budget, opt.eval_interval, opt.eval_episodes, opt.checkpoint_interval,
                           os.path.join(out_dir, "checkpoint.bin"))
    mw = MetricsWriter(os.path.join(out_dir, "metrics.jsonl"), os.path.join(out_dir, "timings.log"))
    try:
        mw.write_header("es", es_config_entries(cfg, seed, opt.budget, opt.eval_interval, opt.eval_episodes))
        learn(wf, root, opt, mw)
    finally:
        mw.close()
    return wf


__all__ = ["Budget", "LearnOptions", "MetricsWriter", "dump_json", "eval_key", "es_config_entries",
           "key_from_seed", "learn", "run"]
