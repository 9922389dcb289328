#!/usr/bin/env python
"""Benchmark of the B200 ES generation path (BASELINE.json metric: env-steps/sec
and generations/sec at pop x envs, 1/2/4/8 B200 vs the host-CPU reference).

Default workload (N=1): BASELINE.json configs[2] -- OpenES pop 4096 x 16
envs/individual, 2x256 MLP, Pendulum fixed horizon H=200 (d = 67 073), the
largest config that fits one GPU and the one the metric's "pop x envs" and
"1/2/4/8 B200" are quoted on.  A step = one full generation (ask -> rollout of
13.1 M env-steps -> fitness -> ranks -> tell + Adam) with the population
sharded over N GPUs (weak... total work fixed: "strong" scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--precision oz|f64|tc|f32]
  python bench.py --impl reference ...   # the reference CPU path (oracle port) on host cores

Headline precision "oz": the policy's dense layer as exact int8 tcgen05 MMAs
over 6-byte-sliced fixed-point operands (~47 bits each), everything else fp64
-- fitness ranks identical to the fp64 path on this workload
(tests/test_gpu_oz.py), returns within ~1e-8 of the reference CPU
restatement.  The fp64 DMMA team ("f64", the bit-level parity path) and the
fp32-accurate tcgen05 team ("tc") are measured beside it (`variants`).

Timing: W untimed warm-up generations, then K generations, each bracketed by a
barrier + torch.cuda.synchronize(); per-generation device time from CUDA
events on the launching stream, L2 flushed (256 MiB write) between timed
generations outside the events; max over ranks.
"""
from __future__ import annotations

import argparse
import math
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs; the bench line is configs[2] ("3")
CONFIGS = {
    "1": dict(algo="openes", env="pendulum", fixed_horizon=True, pop=128, hidden=(64, 64),
              max_episode_steps=200, fitness_episodes=1,
              desc="OpenES pop 128 antithetic, 2x64 MLP, Pendulum H=200"),
    "2": dict(algo="ars", env="pendulum", fixed_horizon=True, pop=1024, hidden=(),
              allow_linear=True, max_episode_steps=200, fitness_episodes=1,
              desc="ARS top-16 pop 1024, linear policy (extension), Pendulum H=200, RS obs-norm"),
    "3": dict(algo="openes", env="pendulum", fixed_horizon=True, pop=4096, hidden=(256, 256),
              max_episode_steps=200, fitness_episodes=16,
              desc="OpenES pop 4096 x 16 envs/individual, 2x256 MLP, Pendulum H=200"),
    "4": dict(algo="cmaes", env="pendulum", fixed_horizon=True, pop=512, hidden=(97, 97),
              max_episode_steps=200, fitness_episodes=1, cmaes_elites=64, cmaes_sigma0=0.1,
              cmaes_max_dim=10240, cmaes_eig_every=0,
              desc="CMA-ES pop 512, mu 64, 3x97x97x1 MLP (d=9992), Pendulum H=200, Jacobi eig every "
                   "k gens (k = floor(1/(10 d (c1+cmu))) = 9)"),
}


def workload_config(cfg_name):
    """The `config` object of the bench line: the workload's identity only, so
    the GPU arm and the reference arm print the same object for the same run
    (how each arm executes it goes under `run`)."""
    cfgd = CONFIGS[cfg_name]
    obs, out = (3, 1) if cfgd["env"] == "pendulum" else (4, 2)
    dims = [obs] + list(cfgd["hidden"]) + [out]
    params = sum(dims[i] * dims[i + 1] + dims[i + 1] for i in range(len(dims) - 1))
    c = {"workload": cfgd["desc"], "config": cfg_name, "pop": cfgd["pop"],
         "envs_per_individual": cfgd["fitness_episodes"], "horizon": cfgd["max_episode_steps"],
         "hidden": list(cfgd["hidden"]), "params": params,
         "l2": "GPU arm: flushed (256 MiB write) before every timed generation; CPU reference arm: host, "
               "not applicable"}
    if cfgd["algo"] == "cmaes":
        c["eig_every"] = cma_lazy_gap(params, cfgd["cmaes_elites"], cfgd["pop"])
        c["timed_window"] = "whole lazy periods (one eigendecomposition per period)"
    return c


def mlp_flops_per_step(obs_dim, hidden, out_dim):
    dims = [obs_dim] + list(hidden) + [out_dim]
    return 2 * sum(a * b for a, b in zip(dims[:-1], dims[1:]))


def cma_lazy_gap(d, mu, pop):
    """max(1, floor(1 / (10 d (c1 + cmu)))) with the reference's CMA constants
    (proj/src/ec.cpp:191-224; weights log((pop+1)/2) - log(i+1), clamped at 0)."""
    w = [max(0.0, math.log((pop + 1) / 2.0) - math.log(i + 1)) for i in range(mu)]
    sw = sum(w)
    mueff = 1.0 / sum((x / sw) ** 2 for x in w)
    c1 = 2.0 / ((d + 1.3) ** 2 + mueff)
    cmu = min(1.0 - c1, 2.0 * (mueff - 2.0 + 1.0 / mueff) / ((d + 2.0) ** 2 + mueff))
    return max(1, int(math.floor(1.0 / (10.0 * d * (c1 + cmu)))))


# DRAM bytes (read + write) per launch of the dominant kernel from one
# `ncu --set full` capture of the same command (profiles/README.md)
NCU_TRAFFIC = {
    ("3", "f64"): (2230139136 + 68040960, "ncu r01_f64_v6: rollout_kernel<double,1,16,4,1>"),
    ("3", "tc"): (1104370432 + 10082304, "ncu r01_tc_v5: rollout_tc_kernel<2> (cta_group::2 pair)"),
    ("3", "oz"): (1672574000 + 6800640, "ncu r02_ozp_full_v10: rollout_ozp_kernel<6,2> (pre-split slices read once)"),
}
# int8 MMA work the oz team executes per env step and CTA (2 lane groups x
# W1p/32 k-steps x S MMAs of M=128, K=32, N = 8(S-i) rounded up to 16): the
# tensor-pipe view of the roofline beside the algorithmic one
OZ_S = 6
# executed warp-instructions per Box-Muller pair of the OpenES noise generator
# (smsp__inst_executed / pairs of k_noise_rows, ncu, config 3)
NOISE_WARP_INSTS_PER_PAIR = 384


def oz_int8_ops_per_cta_step(w1):
    w1p = -(-w1 // 32) * 32
    n_sum = sum(-(-(8 * (OZ_S - i)) // 16) * 16 for i in range(OZ_S))
    return 2 * (w1p // 32) * 2 * 128 * n_sum * 32


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def bf16_peak():
    """Dense bf16 roof for kernels timed inside the (long) generation step: the
    sustained figure of MEASURED_PEAKS.json (the burst one if it is absent)."""
    p = load_peaks()
    return p.get("bf16_tflops_sustained") or p.get("bf16_tflops")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# --------------------------------------------------------------- CPU legs
def cpu_sample_run(cfgd, steps, warmup, sample_pop=None, workers=0):
    """The oracle port (oracle/, C11 restatement of the reference hot path) on
    all host cores: generations of a bounded population sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_ffi as oracle

    kw = {k: v for k, v in cfgd.items() if k != "desc"}
    kw["hidden"] = list(kw["hidden"])
    if sample_pop:
        kw["pop"] = sample_pop
    kw["workers"] = workers
    kw["vbn_samples"] = 10000
    es = oracle.OracleEs(oracle.es_config(**kw))
    es.init(oracle.key_from_seed(0))
    for _ in range(warmup):
        es.step()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        es.step()
        times.append(time.perf_counter() - t0)
    env_steps = kw["pop"] * kw["fitness_episodes"] * kw["max_episode_steps"]
    cores = workers if workers > 0 else os.cpu_count()
    return env_steps, times, cores, kw["pop"]


def cpu_baseline(cfgd, cfg_name):
    if cfgd["algo"] == "cmaes":
        return {"value": None, "unit": "env-steps/s", "cores": os.cpu_count(), "kind": "port",
                "sample": ("not run: the port's O(d^3) single-thread Jacobi at d=9992 takes hours per "
                           "generation (the reference's Eigen solver ~1e3 s, SURVEY.md §8(d))")}
    pop = cfgd["pop"]
    sample = {"3": 256}.get(cfg_name, pop)
    env_steps, times, cores, sp = cpu_sample_run(cfgd, steps=1, warmup=0, sample_pop=sample)
    t = min(times)
    return {"value": env_steps / t, "unit": "env-steps/s", "cores": cores, "kind": "port",
            "sample": (f"1 generation of the oracle port (oracle/, C11 restatement; the reference "
                       f"needs Eigen3, absent) at pop {sp} of {pop}, same net/envs/horizon, "
                       f"{cores} host threads; {env_steps} env-steps in {t:.2f} s"),
            "generations_per_sec_at_full_pop": 1.0 / (t * pop / sp)}


def run_reference_arm(args, cfgd, cfg_name):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    pop = cfgd["pop"]
    sample = {"3": 128}.get(cfg_name, pop)
    env_steps, times, cores, sp = cpu_sample_run(cfgd, steps=args.steps, warmup=min(args.warmup, 1),
                                                 sample_pop=sample)
    total = sum(times)
    value = env_steps * len(times) / total
    line = {
        "impl": "reference", "metric": "env-steps/sec", "value": value, "unit": "env-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg_name),
        "run": {"parallelism": f"{cores} host threads (ThreadPool lane grid)", "pop_sampled": sp},
        "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": cores, "kind": "port",
                         "sample": f"each step = 1 generation of the oracle port at pop {sp} of {pop}"},
        "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "generations_per_sec": 1.0 / (total / len(times) * pop / sp),
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="3", choices=sorted(CONFIGS))
    ap.add_argument("--precision", default="oz", choices=["oz", "f64", "f32", "tc"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variants", dest="variants", action="store_false",
                    help="skip the other precisions' measurements beside the headline")
    args = ap.parse_args()
    cfgd = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfgd, args.config)

    import numpy as np
    import torch

    import paper_2501_15129_b200 as evb
    from paper_2501_15129_b200 import _lib
    from paper_2501_15129_b200.dist import CudaShardedEs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # EVORL_BENCH_ONE_GPU=1 / EVORL_BENCH_BACKEND=gloo: functional smoke test of
    # the N>1 code path on a one-GPU box (all ranks on cuda:0; numbers meaningless)
    if os.environ.get("EVORL_BENCH_ONE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("EVORL_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    L = _lib.load()

    kw = {k: v for k, v in cfgd.items() if k != "desc"}
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed_generations(precision, clk=None):
        """W warm-up + K timed generations at `precision`; returns the handle,
        max-over-ranks total ms, per-step rollout ms and kernel launches."""
        cfg = evb.EsConfig(**kw, precision=precision, device=local)
        if world > 1:
            runner = CudaShardedEs(cfg, rank, world)
            runner.init((0x9E3779B97F4A7C15, 0))
            step, es = runner.step, runner.es
        else:
            es = evb.EsWorkflow(cfg).init((0x9E3779B97F4A7C15, 0))
            step = es.step
        for _ in range(args.warmup):
            step()
        barrier()
        if kw.get("algo") == "cmaes" and kw.get("cmaes_eig_every", 1) == 0:
            # lazy CMA-ES: time whole periods so the amortised eigendecomposition
            # is inside the window (generation counter g -> eig when g % gap == 0)
            gap = cma_lazy_gap(es.dim, kw["cmaes_elites"], kw["pop"])
            args.steps = -(-max(args.steps, gap) // gap) * gap
            args.cma_gap = gap
        launches0 = L.evorl_kernel_launches()
        times, roll, ask = [], [], []
        if clk is not None:
            clk.__enter__()
        for _ in range(args.steps):
            flush.zero_()                      # L2 flush outside the timed events
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            step()
            e1.record()
            barrier()
            times.append(e0.elapsed_time(e1))
            roll.append(es.last_timings()[0])   # rollout kernel, events on the library stream
            ask.append(es.last_ask_ms())        # materialised ask (-1: not one timed launch)
        if clk is not None:
            clk.__exit__(None, None, None)
        launches = L.evorl_kernel_launches() - launches0
        tot = torch.tensor([sum(times)], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        args.ask_ms = statistics.mean(ask) if ask and min(ask) > 0 else None
        args.step_fn = step
        return cfg, es, float(tot.item()), roll, launches

    clk = ClockSampler(local)
    cfg, es, max_ms, roll, launches = timed_generations(args.precision, clk)
    step_fn = args.step_fn
    ask_ms = args.ask_ms

    pop, e, H = cfg.pop, cfg.fitness_episodes, cfg.max_episode_steps
    env_steps_per_gen = pop * e * H
    value = env_steps_per_gen * args.steps / (max_ms / 1e3)
    ms_per_step = max_ms / args.steps
    obs_dim = 3 if cfg.env == "pendulum" else 4
    out_dim = 1 if cfg.env == "pendulum" else 2
    F = mlp_flops_per_step(obs_dim, cfg.hidden, out_dim)

    # ---- e2e through the reference-facing C ABI with HOST buffers (N=1):
    # Workflow::step with host-resident EsState: upload mean/m/v, run the
    # generation, download mean/m/v + StepMetrics, every step.
    e2e = None
    if world == 1 and not args.no_e2e:
        d = es.dim
        # the host-resident EsState in page-locked buffers (updated in place)
        mean_h, m_h, v_h = (evb.pinned_empty(es.dim) for _ in range(3))
        mean_h[:] = es.mean()
        m0, v0, t_h = es.adam()
        m_h[:] = m0
        v_h[:] = v0
        h2d = 3 * d * 8 + 8
        d2h = 3 * d * 8 + 8 + 5 * 8
        barrier()
        ets = []
        for _ in range(max(1, args.steps)):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            _, _, _, t_h, _ = es.step_host(mean_h, m_h, v_h, t_h, out=(mean_h, m_h, v_h))
            e1.record()
            barrier()
            ets.append(e0.elapsed_time(e1))
        e2e = {"value": env_steps_per_gen * len(ets) / (sum(ets) / 1e3), "unit": "env-steps/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "generations_per_sec": len(ets) / (sum(ets) / 1e3),
               "path": "C ABI evorl_es_step_host: host EsState (mean, Adam m/v/t, page-locked buffers) in, "
                       "generation, updated state + StepMetrics out"}
    elif world > 1 and not args.no_e2e:
        # sharded: every rank uploads the (replicated) host EsState, runs the
        # sharded generation (CudaShardedEs.step: both collectives) and reads the
        # updated state back; max over ranks
        d = es.dim
        mean_h, m_h, v_h = (evb.pinned_empty(d) for _ in range(3))
        mean_h[:] = es.mean()
        m0, v0, t_h = es.adam()
        m_h[:] = m0
        v_h[:] = v0
        h2d = 3 * d * 8 + 8
        d2h = 3 * d * 8 + 8 + 5 * 8
        barrier()
        ets = []
        for _ in range(max(1, args.steps)):
            flush.zero_()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            es.set_mean(mean_h)
            es.set_adam(m_h, v_h, t_h)
            step_fn()
            mean_h[:] = es.mean()
            m1, v1, t_h = es.adam()
            m_h[:] = m1
            v_h[:] = v1
            e1.record()
            barrier()
            ets.append(e0.elapsed_time(e1))
        tot_e = torch.tensor([sum(ets)], dtype=torch.float64, device="cuda")
        dist.all_reduce(tot_e, op=dist.ReduceOp.MAX)
        e_ms = float(tot_e.item())
        e2e = {"value": env_steps_per_gen * len(ets) / (e_ms / 1e3), "unit": "env-steps/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "generations_per_sec": len(ets) / (e_ms / 1e3),
               "path": "per rank: C ABI evorl_es_set_mean/set_adam (page-locked host EsState) -> "
                       "CudaShardedEs.step (NCCL all-gathers) -> get_mean/get_adam; max over ranks"}

    # ---- roofline of the dominant kernel (the fused rollout)
    roll_ms = statistics.mean(roll) if roll else None
    agents_local = es.shard_ranges()[1] - es.shard_ranges()[0] if world > 1 else pop
    flops_launch = agents_local * e * H * F
    extra = {}
    # the team that actually runs: oz covers obs -> W1 -> W2 -> O with W1 <= 256 and
    # >= 5 envs per individual, other shapes run the fp64 teams (bit-identical to f64)
    eff_prec = args.precision
    if eff_prec == "oz" and not (len(cfg.hidden) == 2 and e >= 5 and cfg.hidden[0] <= 256):
        eff_prec = "f64"
    if eff_prec == "oz":
        # config 3 is tensor-core bound, roof = the dense tensor
        # peak; achieved counts the MLP's algorithmic flops.  The kernel is bound
        # by the serial 200-step chain (one CTA per SM, TMEM-limited), so two more
        # views are reported: the same flops against the FP64 peak (the accuracy
        # class this path delivers) and the int8 MMA work the tensor pipe executes.
        peak = bf16_peak()
        bound, unit, peak_src = "tensor", "TFLOP/s", (
            "MEASURED_PEAKS.json bf16_tflops_sustained (the rollout is timed inside a long step), per "
            "SURVEY.md §8(d); achieved counts the MLP's "
            "algorithmic flops")
        fp64_peak = evb.measure_fp64_peak()
        int8_peak = 2.0 * peak if peak else None
        ops = oz_int8_ops_per_cta_step(cfg.hidden[0]) * (agents_local * -(-e // 16)) * \
            (-(-cfg.hidden[1] // 128)) * H if len(cfg.hidden) == 2 else None
        ex_tops = ops / (roll_ms * 1e-3) / 1e12 if (ops and roll_ms) else None
        extra = {"fp64_equivalent": {"peak": fp64_peak, "unit": "TFLOP/s",
                                     "peak_source": "measured live: DFMA-bound microkernel (evorl_measure_fp64_peak)"},
                 "tensor_pipe_executed": {"achieved": ex_tops, "unit": "TOPS (int8 MMA ops incl. slice products "
                                          "and zero-padded windows)", "peak": int8_peak,
                                          "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops_sustained (dense int8 = 2x bf16 "
                                                         "on B200; derived, not measured)",
                                          "frac": (ex_tops / int8_peak) if (ex_tops and int8_peak) else None}}
    elif eff_prec == "f64":
        peak = evb.measure_fp64_peak()
        bound, unit, peak_src = "fp64", "TFLOP/s", (
            "measured live: DFMA-bound microkernel (evorl_measure_fp64_peak); "
            "MEASURED_PEAKS.json has no FP64 figure")
    elif eff_prec == "tc":
        # the dense W2 x W1 layer runs on tcgen05 (kind::f16, 3 passes); the
        # roof is the dense 16-bit tensor peak of MEASURED_PEAKS.json (fp16 and
        # bf16 run at the same rate), counting only the useful (1-pass) flops
        peak = bf16_peak()
        bound, unit, peak_src = "tensor", "TFLOP/s", (
            "MEASURED_PEAKS.json bf16_tflops_sustained (timed inside a long step; fp16 kind::f16 same "
            "rate); achieved counts "
            "the MLP's algorithmic flops, not the 3x hi/lo split passes")
    else:
        peak = None
        bound, unit, peak_src = "fp32", "TFLOP/s", "measured live: FFMA is not in MEASURED_PEAKS.json"
        peak = evb.measure_fp64_peak() * 2.0  # FP32 FMA issue rate is 2x FP64 on B200
        peak_src = "2 x measured DFMA peak (B200 FP32:FP64 FMA issue ratio 2:1)"
    achieved = flops_launch / (roll_ms * 1e-3) / 1e12 if roll_ms else None
    if "fp64_equivalent" in extra:
        fe = extra["fp64_equivalent"]
        fe["achieved"] = achieved
        fe["frac"] = (achieved / fe["peak"]) if (achieved and fe["peak"]) else None
    roofline = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, **extra,
                "frac": (achieved / peak) if (achieved and peak) else None,
                "traffic": NCU_TRAFFIC.get((args.config, eff_prec), (None,))[0],
                "traffic_source": NCU_TRAFFIC.get((args.config, eff_prec), (None, None))[1],
                "kernel": {"tc": "rollout_tc_kernel (tcgen05 hidden layer, fused obs-norm/MLP/env/return)",
                           "oz": "rollout_ozp_kernel (int8-sliced tcgen05 hidden layer, two pipelined lane "
                                 "groups, fused obs-norm/MLP/env/return)"}.get(
                               eff_prec, "fp64 rollout team (cluster DMMA or warp-per-lane; fused "
                                         "obs-norm/MLP/env/return)"),
                "team_precision": eff_prec,
                "algorithmic_flops_per_launch": flops_launch,
                "flops_per_env_step": F, "peak_source": peak_src,
                "rollout_ms_per_launch": roll_ms, "rollout_share_of_step":
                    (roll_ms / ms_per_step) if roll_ms else None}

    # ---- the ask: the OpenES noise generator as normals/s
    # against the SM issue rate (Threefry is INT ALU work, Box-Muller FP64:
    # both issue-bound), measured at full occupancy; in the generation it runs
    # beside the previous rollout, and the ask on the path only adds the mean
    rng = None
    if kw.get("algo") == "openes" and world == 1:
        rows = pop // 2 if cfg.openes_mirrored else pop
        normals = rows * es.dim
        rate = evb.measure_noise_rate(normals)
        sm_mhz = (clk.summary() or {}).get("sm_mhz") or 1965.0
        peak_n = 148 * 4 * sm_mhz * 1e6 * 32 / NOISE_WARP_INSTS_PER_PAIR * 2
        rng = {"normals_per_gen": normals, "achieved": rate, "unit": "normals/s",
               "bound": "SM issue (Threefry INT ALU + Box-Muller FP64)", "peak": peak_n, "frac": rate / peak_n,
               "peak_source": f"148 SMs x 4 warp-instructions/clk x {sm_mhz:.0f} MHz / "
                              f"{NOISE_WARP_INSTS_PER_PAIR} warp-instructions per Box-Muller pair (ncu "
                              "smsp__inst_executed of k_noise_rows) x 2 normals per pair",
               "kernel": "k_noise_rows (evorl_measure_noise_rate: full occupancy, alone)",
               "in_generation": "k_noise_rows beside the previous generation's rollout (one block per SM on a "
                                "low-priority stream), off the critical path",
               "ask_on_path_ms": ask_ms,
               "ask_on_path": ("k_oz_ask_split: the ask fused with the layer-1 pre-split from the kept noise rows"
                               if eff_prec == "oz" else
                               "k_cand_from_eps: candidates = mean + sigma * kept noise rows (HBM-bound)")}

    # ---- the other policy precisions on the same workload, beside the headline:
    # f64 (DMMA team, the bit-level parity path) and tc (fp32-accurate tcgen05
    # team: returns within the fp32 tolerance, ranks not bit-exact)
    variants = {}
    assert es.dim == workload_config(args.config)["params"]
    parity = {
        "f64": "bit-level parity path: returns within 1e-9 of the reference CPU restatement, ranks identical",
        "oz": "returns within ~1e-8 of the reference CPU restatement, ranks identical to the fp64 path "
              "(tests/test_gpu_oz.py, tools/tc_rank_agreement.py)",
        "tc": "returns within fp32 tolerance of the reference; fitness ranks not bit-exact "
              "(tools/tc_rank_agreement.py: 9-99 of 4096 ranks shift, by <= 20 positions)",
    }
    if args.variants and int(kw.get("fitness_episodes", 1)) >= 5 and len(kw.get("hidden", ())) == 2:
        del es
        for vp in ("f64", "tc", "oz"):
            if vp == args.precision:
                continue
            _, es_v, v_ms, v_roll, v_launches = timed_generations(vp)
            v_roll_ms = statistics.mean(v_roll) if v_roll else None
            v_ach = flops_launch / (v_roll_ms * 1e-3) / 1e12 if v_roll_ms else None
            v_peak = evb.measure_fp64_peak() if vp == "f64" else bf16_peak()
            variants[vp] = {
                "precision": vp, "value": env_steps_per_gen * args.steps / (v_ms / 1e3),
                "unit": "env-steps/s", "ms_per_step": v_ms / args.steps,
                "generations_per_sec": args.steps / (v_ms / 1e3), "gpu_launches": int(v_launches),
                "roofline": {"bound": "fp64" if vp == "f64" else "tensor", "achieved": v_ach, "peak": v_peak,
                             "unit": "TFLOP/s", "frac": (v_ach / v_peak) if (v_ach and v_peak) else None,
                             "traffic": NCU_TRAFFIC.get((args.config, vp), (None,))[0],
                             "rollout_ms_per_launch": v_roll_ms,
                             "peak_source": ("measured live DFMA peak" if vp == "f64" else
                                             "MEASURED_PEAKS.json bf16_tflops_sustained; achieved counts algorithmic flops")},
                "parity": parity[vp]}
            del es_v

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfgd, args.config)

    if rank == 0:
        line = {
            "metric": "env-steps/sec", "value": value, "unit": "env-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if args.precision in ("f32", "tc") else "f64", "data": "synthetic",
            "config": workload_config(args.config),
            "run": {"parallelism": f"population-sharded dp{world}",
                    "policy_precision": args.precision,
                    "policy_team": eff_prec,
                    "parity": parity.get(eff_prec, "returns within fp32 tolerance"),
                    "env_dynamics": "f64"},
            "generations_per_sec": args.steps / (max_ms / 1e3),
            "gpu_launches": int(launches),
            "roofline": roofline,
            "ask_rng": rng,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk.summary(),
            "variants": variants,
        }
        print(json.dumps(line))
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
