"""Per-role cycle breakdown of the pipelined int8-sliced team (profiling build).

  make -C paper_2501_15129_b200/csrc prof
  EVORL_B200_LIB=$PWD/paper_2501_15129_b200/libevorl_b200_prof.so python tools/ozp_phase_probe.py

One config-3 generation with precision "oz" (pipelined kernel); per step and CTA:
compute warps (thread 0), env warp of group 0 (lane 0), MMA warp (lane 0).
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import paper_2501_15129_b200 as evb  # noqa: E402

ROLES = {"compute warps": {0: "prologue (once)", 1: "wait x0 (env)", 2: "layer 0 + B", 3: "wait MMA",
                           4: "epilogue", 5: "publish + barrier"},
         "env warp 0": {7: "reward pre-term, arming, loop top", 6: "wait partial outputs", 11: "head (sum + tanh)",
                        12: "env_step", 13: "bookkeeping", 14: "observe + x0"},
         "MMA warp": {9: "wait B", 10: "issue"}}


def main():
    cfg = evb.EsConfig(algo="openes", env="pendulum", fixed_horizon=True, pop=int(os.environ.get("POP", 4096)),
                       fitness_episodes=16, hidden=(256, 256), max_episode_steps=200, precision="oz")
    g = evb.EsWorkflow(cfg).init((1, 2))
    L = evb._lib.load()
    buf = (C.c_ulonglong * 16)()
    g.step()
    L.evorl_debug_oz_profile(buf)
    g.step()
    L.evorl_debug_oz_profile(buf)
    ctas, steps = buf[8], 200
    for role, ph in ROLES.items():
        tot = sum(buf[i] for i in ph) / ctas
        print(f"{role}: {tot:.0f} cycles per CTA ({tot / steps:.0f} per step)")
        for i, name in ph.items():
            per = buf[i] / ctas
            print(f"  {name:34s} {per / (1 if i == 0 else steps):9.0f}{'' if i == 0 else ' / step'}")


if __name__ == "__main__":
    main()
