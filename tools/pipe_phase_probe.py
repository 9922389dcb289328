"""Per-phase cycle breakdown of the pipelined fp64 team (profiling build).

  make -C paper_2501_15129_b200/csrc prof
  EVORL_B200_LIB=$PWD/paper_2501_15129_b200/libevorl_b200_prof.so python tools/pipe_phase_probe.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2501_15129_b200 as evb  # noqa: E402

PHASES = {0: "compute: wait x0 (env warp)", 1: "compute: layer 0 + barrier", 2: "compute: layer 1 DMMA + barrier",
          3: "compute: output partial + st.async", 7: "compute: mask reset / loop",
          4: "env: wait partials (mbarrier)", 5: "env: head + env + observe + arrive", 6: "env: arm / loop"}


def main():
    cfg = evb.EsConfig(algo="openes", env="pendulum", fixed_horizon=True, pop=4096, fitness_episodes=16,
                       hidden=(256, 256), max_episode_steps=200)
    g = evb.EsWorkflow(cfg).init((1, 2))
    L = evb._lib.load()
    buf = (C.c_ulonglong * 16)()
    g.step()
    L.evorl_debug_rk_profile(buf)
    g.step()
    L.evorl_debug_rk_profile(buf)
    ctas, steps = buf[8], 200
    for side, ids in (("compute warp 0", (0, 1, 2, 3, 7)), ("env warp", (4, 5, 6))):
        tot = sum(buf[i] for i in ids) / ctas
        print(f"{side}: {tot / steps:.0f} cycles / step")
        for i in ids:
            print(f"  {PHASES[i]:40s} {buf[i] / ctas / steps:8.0f} cycles / step ({100 * buf[i] / ctas / tot:5.1f}%)")


if __name__ == "__main__":
    main()
