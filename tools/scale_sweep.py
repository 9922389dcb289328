"""BASELINE config 5: synthetic scale sweep on one B200.

pop 256 -> 65536, policy width 64 -> 1024 (2 hidden layers), Pendulum fixed
horizon H = 1000, OpenES, e in {1, 16} envs per individual.  One warm-up and one
timed generation per cell (CUDA events around EsWorkflow.step, L2 not flushed:
the generation is seconds long), cells whose projected time exceeds the budget
are skipped and listed.  Writes JSON lines to stdout.

  python tools/scale_sweep.py [--precision tc|oz|f64|f32] [--budget-s 20] [--h 1000]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--precision", default="tc", choices=["f64", "f32", "tc", "oz"])
    ap.add_argument("--budget-s", type=float, default=20.0)
    ap.add_argument("--h", type=int, default=1000)
    ap.add_argument("--pops", default="256,1024,4096,16384,65536")
    ap.add_argument("--widths", default="64,128,256,512,1024")
    ap.add_argument("--envs", default="1,16")
    args = ap.parse_args()
    import torch

    import paper_2501_15129_b200 as evb

    peaks = {}
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    rate = {}  # (width, e) -> measured env-steps/s, to project larger pops
    for e in [int(x) for x in args.envs.split(",")]:
        for w in [int(x) for x in args.widths.split(",")]:
            for pop in [int(x) for x in args.pops.split(",")]:
                steps = pop * e * args.h
                F = 2 * (3 * w + w * w + w)
                proj = steps / rate[(w, e)] if (w, e) in rate else None
                cell = {"pop": pop, "width": w, "envs": e, "horizon": args.h, "precision": args.precision,
                        "env_steps_per_gen": steps, "flop_per_gen": steps * F}
                if proj is not None and 2 * proj > args.budget_s:
                    cell["skipped"] = f"projected {proj:.1f} s/generation > budget/2"
                    print(json.dumps(cell), flush=True)
                    continue
                try:
                    cfg = evb.EsConfig(algo="openes", env="pendulum", fixed_horizon=True, pop=pop,
                                       fitness_episodes=e, hidden=(w, w), max_episode_steps=args.h,
                                       precision=args.precision)
                    g = evb.EsWorkflow(cfg).init((11, 12))
                    t0 = time.time()
                    g.step()  # warm-up
                    torch.cuda.synchronize()
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.step()
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                    roll_ms = g.last_timings()[0]
                    del g
                    cell.update({"ms_per_generation": ms, "rollout_ms": roll_ms,
                                 "env_steps_per_s": steps / (ms / 1e3),
                                 "policy_tflops": steps * F / (roll_ms / 1e3) / 1e12,
                                 "wall_s": time.time() - t0})
                    if args.precision in ("tc", "oz") and peaks.get("bf16_tflops"):
                        cell["frac_of_bf16_peak"] = cell["policy_tflops"] / peaks["bf16_tflops"]
                    rate[(w, e)] = steps / (ms / 1e3)
                except Exception as ex:  # report and continue (e.g. Unsupported)
                    cell["error"] = f"{type(ex).__name__}: {ex}"
                print(json.dumps(cell), flush=True)


if __name__ == "__main__":
    main()
