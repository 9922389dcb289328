"""Per-phase cycle breakdown of the int8-sliced tensor-core team (profiling build).

  make -C paper_2501_15129_b200/csrc prof
  EVORL_B200_LIB=$PWD/paper_2501_15129_b200/libevorl_b200_prof.so python tools/oz_phase_probe.py

Runs one config-3 generation (OpenES pop 4096 x 16 envs, 2x256, Pendulum
H=200) with precision "oz" and prints the cycles thread 0 of an average CTA
spent per step in each phase of rollout_oz_kernel.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import paper_2501_15129_b200 as evb  # noqa: E402

PHASES = {0: "prologue (once)", 1: "loop-top barrier", 11: "layer 0 + slicing + B stores", 2: "proxy fence + barrier + reward pre",
          3: "MMA issue + completion", 4: "epilogue + output partial", 5: "cluster exchange",
          9: "head (output sum + tanh)", 10: "env_step", 6: "observe + bookkeeping"}


def main():
    pop = int(os.environ.get("POP", 4096))
    cfg = evb.EsConfig(algo="openes", env="pendulum", fixed_horizon=True, pop=pop, fitness_episodes=16,
                       hidden=(256, 256), max_episode_steps=200, precision="oz")
    g = evb.EsWorkflow(cfg).init((1, 2))
    L = evb._lib.load()
    buf = (C.c_ulonglong * 16)()
    g.step()  # warm-up
    L.evorl_debug_oz_profile(buf)  # reset
    g.step()
    L.evorl_debug_oz_profile(buf)
    ctas = buf[8]
    steps = 200
    tot = sum(buf[i] for i in PHASES) / ctas
    print(f"CTAs {ctas}; cycles per CTA {tot:.0f} ({tot / steps:.0f} per step)")
    for i, name in PHASES.items():
        per_cta = buf[i] / ctas
        print(f"  {name:30s} {per_cta / (1 if i == 0 else steps):9.0f} cycles"
              f"{'' if i == 0 else ' / step'}  ({100 * per_cta / tot:5.1f}%)")


if __name__ == "__main__":
    main()
