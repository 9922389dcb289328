"""Host-side cost of the e2e (host-buffer) generation at config 3: wall time
of each C-ABI call around evorl_es_step.

  python tools/e2e_probe.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2501_15129_b200 as evb  # noqa: E402

kw = dict(algo="openes", env="pendulum", fixed_horizon=True, pop=4096, fitness_episodes=16,
          hidden=(256, 256), max_episode_steps=200, precision="oz")
es = evb.EsWorkflow(evb.EsConfig(**kw)).init((1, 2))
for _ in range(3):
    es.step()
mean_h = np.ascontiguousarray(es.mean())
m_h, v_h, t_h = es.adam()
acc = {}
for it in range(8):
    marks = [("t0", time.perf_counter())]
    es.set_mean(mean_h)
    marks.append(("set_mean", time.perf_counter()))
    es.set_adam(m_h, v_h, t_h)
    marks.append(("set_adam", time.perf_counter()))
    es.step()
    marks.append(("step", time.perf_counter()))
    mean_h = es.mean()
    marks.append(("mean", time.perf_counter()))
    m_h, v_h, t_h = es.adam()
    marks.append(("adam", time.perf_counter()))
    if it >= 2:
        for (a, ta), (b, tb) in zip(marks, marks[1:]):
            acc.setdefault(b, []).append((tb - ta) * 1e3)
for k, v in acc.items():
    print(f"{k:10s} {np.median(v):8.3f} ms")

# the bench's two loops (L2 flushed before each timed generation)
import torch  # noqa: E402

flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def timed(fn, n=6):
    ts = []
    for _ in range(n):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return ts


def e2e():
    global mean_h, m_h, v_h, t_h
    es.set_mean(mean_h)
    es.set_adam(m_h, v_h, t_h)
    es.step()
    mean_h = es.mean()
    m_h, v_h, t_h = es.adam()


for name, fn in [("step", es.step), ("e2e", e2e), ("step", es.step), ("e2e", e2e)]:
    ts = timed(fn)
    print(name, " ".join(f"{t:.2f}" for t in ts), "rollout", es.last_timings())
