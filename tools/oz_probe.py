"""Quick check of the int8-sliced tensor-core team (precision "oz") against the
fp64 team on batched_rollout shapes, and its config-3 generation time.

  python tools/oz_probe.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2501_15129_b200 as evb  # noqa: E402
from paper_2501_15129_b200 import _lib  # noqa: E402


def shapes():
    for env, hidden, m, e, fh in [("pendulum", (256, 256), 8, 16, True), ("pendulum", (97, 97), 4, 16, True),
                                  ("pendulum", (256, 512), 4, 16, True), ("pendulum", (128, 256), 3, 40, True),
                                  ("cartpole", (64, 128), 6, 16, False)]:
        obs, out, head = (3, 1, _lib.HEAD_TANH) if env == "pendulum" else (4, 2, _lib.HEAD_CATEGORICAL)
        desc = evb.mlp_desc(obs, hidden, out, head, 2.0 if env == "pendulum" else 1.0)
        d = evb.param_count(desc)
        rng = np.random.default_rng(5)
        params = rng.standard_normal((m, d)) * 0.15
        r = {}
        for prec in ("f64", "oz"):
            rets, steps, _ = evb.batched_rollout(env, desc, params, e, (3, 4), fixed_horizon=fh,
                                                 max_episode_steps=200, precision=prec)
            r[prec] = (rets, steps)
        rel = np.abs(r["oz"][0] - r["f64"][0]) / np.maximum(np.abs(r["f64"][0]), 1e-300)
        print(f"{env} {hidden} m={m} e={e}: steps equal {np.array_equal(r['oz'][1], r['f64'][1])}, "
              f"returns rel err median {np.median(rel):.2e} max {rel.max():.2e}", flush=True)


def timing():
    kw = dict(algo="openes", env="pendulum", fixed_horizon=True, pop=4096, fitness_episodes=16,
              hidden=(256, 256), max_episode_steps=200)
    for prec in ("oz", "f64"):
        g = evb.EsWorkflow(evb.EsConfig(precision=prec, **kw)).init((1, 2))
        g.step()
        t0 = time.perf_counter()
        for _ in range(3):
            g.step()
        dt = (time.perf_counter() - t0) / 3
        r, s = g.last_timings()
        print(f"config 3 {prec}: {dt * 1e3:.1f} ms/gen wall, rollout {r:.1f} ms, step {s:.1f} ms", flush=True)


if __name__ == "__main__":
    shapes()
    timing()
