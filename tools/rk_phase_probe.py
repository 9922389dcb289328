"""Per-phase cycle breakdown of the fp64 cluster team (profiling build).

  make -C paper_2501_15129_b200/csrc prof
  EVORL_B200_LIB=$PWD/paper_2501_15129_b200/libevorl_b200_prof.so python tools/rk_phase_probe.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2501_15129_b200 as evb  # noqa: E402

PHASES = {0: "loop-top barrier", 1: "layer 0 (replicated)", 2: "layer 1 (DMMA slice)",
          3: "output partial + cluster exchange", 4: "head + env + observe"}


def main():
    prec = os.environ.get("PREC", "f64")
    cfg = evb.EsConfig(algo="openes", env="pendulum", fixed_horizon=True, pop=4096, fitness_episodes=16,
                       hidden=(256, 256), max_episode_steps=200, precision=prec)
    g = evb.EsWorkflow(cfg).init((1, 2))
    L = evb._lib.load()
    buf = (C.c_ulonglong * 16)()
    g.step()
    L.evorl_debug_rk_profile(buf)
    g.step()
    L.evorl_debug_rk_profile(buf)
    ctas, steps = buf[8], 200
    tot = sum(buf[i] for i in PHASES) / ctas
    print(f"CTAs {ctas}; loop cycles per CTA {tot:.0f} ({tot / steps:.0f} per step)")
    for i, name in PHASES.items():
        print(f"  {name:34s} {buf[i] / ctas / steps:8.0f} cycles / step ({100 * buf[i] / ctas / tot:5.1f}%)")


if __name__ == "__main__":
    main()
