"""Rank agreement of the tensor-core policy (precision "tc") with the fp64
parity path at full BASELINE config-3 size (OpenES pop 4096 x 16 envs, 2x256,
Pendulum H=200): same state, one generation each, several generations.

  python tools/tc_rank_agreement.py [gens] [precision ...]   (default: f32 tc oz)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2501_15129_b200 as evb  # noqa: E402


def main():
    gens = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    precs = sys.argv[2:] or ["f32", "tc", "oz"]
    kw = dict(algo="openes", env="pendulum", fixed_horizon=True, pop=4096, fitness_episodes=16,
              hidden=(256, 256), max_episode_steps=200)
    ref = evb.EsWorkflow(evb.EsConfig(precision="f64", **kw)).init((1, 2))
    for prec in precs:
        g = evb.EsWorkflow(evb.EsConfig(precision=prec, **kw)).init((1, 2))
        r = evb.EsWorkflow(evb.EsConfig(precision="f64", **kw)).init((1, 2))
        for gen in range(gens):
            # same centre for both: copy the fp64 path's state into the other
            g.set_mean(r.mean())
            m, v, t = r.adam()
            g.set_adam(m, v, t)
            g.set_counters(*r.counters())
            r.step()
            g.step()
            fr, fg = r.fitness(), g.fitness()
            rel = np.abs(fg - fr) / np.abs(fr)
            rk_r = np.argsort(np.argsort(-fr, kind="stable"), kind="stable")
            rk_g = np.argsort(np.argsort(-fg, kind="stable"), kind="stable")
            flips = int(np.sum(rk_r != rk_g))
            gap = np.diff(np.sort(fr))
            print(f"{prec} gen {gen}: fitness rel err median {np.median(rel):.2e} max {rel.max():.2e}; "
                  f"ranks differing {flips}/{len(fr)} (max |d rank| {np.abs(rk_r - rk_g).max()}); "
                  f"min gap between fp64 fitnesses {gap.min():.2e}; "
                  f"mean rel diff after tell {np.abs(g.mean() - r.mean()).max():.2e}")
    del ref


if __name__ == "__main__":
    main()
