"""Diagnostic: eigensolver and CMA-ES generation timing on the GPU (EVORL_EIG_TRACE=1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2501_15129_b200 as evb
# GEMM timing via sym_eig on a 2048 matrix (cold) + a config-4 generation trace
A = np.random.default_rng(0).standard_normal((2048, 2048)); A = A + A.T
t=time.time(); ev, V, sw = evb.sym_eig(A); print("eig 2048 cold", time.time()-t, "s sweeps", sw, flush=True)
cfg = evb.EsConfig(algo="cmaes", env="pendulum", fixed_horizon=True, pop=512, hidden=(97, 97), max_episode_steps=200,
                   cmaes_elites=64, cmaes_sigma0=0.1, cmaes_max_dim=10240)
g = evb.EsWorkflow(cfg).init((1, 2))
for i in range(3):
    t=time.time(); g.step(); print("gen", i, time.time()-t, "s", g.last_timings(), flush=True)
