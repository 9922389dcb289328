"""Run config-3 generations (OpenES pop 4096 x 16 envs, 2x256, Pendulum H=200)
with a given policy precision -- the target command for ncu captures.

  python tools/run_gen.py [precision] [generations]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2501_15129_b200 as evb  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "oz"
gens = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = evb.EsConfig(algo="openes", env="pendulum", fixed_horizon=True, pop=int(os.environ.get("POP", 4096)),
                   fitness_episodes=16, hidden=(256, 256), max_episode_steps=200, precision=prec)
g = evb.EsWorkflow(cfg).init((1, 2))
for _ in range(gens):
    m = g.step()
print(prec, m.values, g.last_timings())
