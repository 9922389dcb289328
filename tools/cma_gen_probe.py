"""Per-generation times of BASELINE config 4 (CMA-ES d = 9992, pop 512) with
the lazy eigendecomposition (cmaes_eig_every = 0): which generations refresh
B, D and what a plain generation costs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_15129_b200 as evb
cfg = evb.EsConfig(algo="cmaes", env="pendulum", fixed_horizon=True, pop=512, hidden=(97, 97),
                   max_episode_steps=200, cmaes_elites=64, cmaes_sigma0=0.1, cmaes_max_dim=10240,
                   cmaes_eig_every=0)
g = evb.EsWorkflow(cfg).init((1, 2))
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    t = time.time()
    g.step()
    roll, tot = g.last_timings()[:2]
    print(f"gen {i + 1}: {1e3 * (time.time() - t):8.1f} ms wall, rollout {roll:.2f} ms, step {tot:.1f} ms",
          flush=True)
