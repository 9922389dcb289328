"""Diagnostic (not collected by pytest): per-generation closed-loop drift of
the GPU workflow vs the oracle."""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle_ffi as oracle
import paper_2501_15129_b200 as evb

def run(kw, gens):
    okw = {k: v for k, v in kw.items() if k != "precision"}; okw["hidden"] = list(kw["hidden"]); okw["workers"] = 0
    o = oracle.OracleEs(oracle.es_config(**okw)); g = evb.EsWorkflow(evb.EsConfig(**kw))
    k = oracle.key_from_seed(5); o.init(k); g.init(k)
    for gen in range(gens):
        o.step(); g.step()
        fo, fg = o.fitness(), g.fitness()
        rel = np.abs(fg - fo) / np.abs(fo)
        ranks_eq = np.array_equal(np.argsort(fg, kind="stable"), np.argsort(fo, kind="stable"))
        mo, mg = o.mean(), g.mean()
        print(f"{kw['algo']} gen {gen}: fit rel max {rel.max():.2e} med {np.median(rel):.2e} "
              f"argmax {rel.argmax()} ranks_eq {ranks_eq} mean absdiff {np.abs(mg-mo).max():.2e}", flush=True)
        if not ranks_eq:
            so = np.sort(fo); gaps = np.diff(so); print("   min fitness gap", gaps.min())

run(dict(algo="ars", env="pendulum", fixed_horizon=True, pop=128, hidden=(), allow_linear=True,
         max_episode_steps=200), 8)
run(dict(algo="openes", env="pendulum", fixed_horizon=True, pop=64, hidden=(64, 64),
         max_episode_steps=200, vbn_samples=2000), 8)
run(dict(algo="ars", env="pendulum", fixed_horizon=True, pop=64, hidden=(16,),
         max_episode_steps=100), 8)
# the oz team (int8-sliced tensor cores) and the fp64 DMMA team on the same
# 16-env OpenES workflow: per-generation drift from the CPU restatement
for prec in ("f64", "oz"):
    print("precision", prec)
    run(dict(algo="openes", env="pendulum", fixed_horizon=True, pop=256, hidden=(128, 256),
             max_episode_steps=200, vbn_samples=2000, fitness_episodes=16, precision=prec), 8)
