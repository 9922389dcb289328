"""Population sharding across GPUs.

One process per GPU.  Rank r rolls out the contiguous agent block
[a0, a1) of the population; the only data-path exchanges per generation are

  C1  all-gather of the fitness vector (pop x fp64), plus the per-lane
      RunningStats (when the resolved obs_norm mode is running_stats), and
  C2  all-gather of the coordinate-sharded mean update: every rank holds the
      full fitness, computes identical ranks, applies the tell (and Adam) to
      coordinates [p0, p1) only -- regenerating the noise rows it needs from
      the replicated ask key -- and the slices are gathered back (CEM: the
      diagonal variance slices too).

Every rank derives the same keys from the replicated (rng, iteration), so no
noise or candidate traffic crosses NVLink, and the result is bit-identical for
any world size (the per-coordinate accumulation order does not depend on the
sharding).

The collectives use torch.distributed (NCCL on GPUs, gloo in the CPU tests);
``Collective`` is the small interface this module needs, so the sharding logic
is testable on CPU with a gloo backend and the oracle as the per-rank compute.
"""
from __future__ import annotations

import math
from typing import Protocol

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Equal contiguous chunks of ceil(n / world) (the last may be short)."""
    cs = math.ceil(n / world) if n > 0 else 0
    lo = min(n, rank * cs)
    hi = min(n, (rank + 1) * cs)
    return lo, hi


class Backend(Protocol):
    """Per-rank compute of one generation's two phases."""

    def rollout(self, a0: int, a1: int) -> tuple[np.ndarray, np.ndarray]:
        """Fitness of agents [a0, a1) and their per-lane stats rows."""

    def tell(self, fitness: np.ndarray, lane_stats: np.ndarray, p0: int, p1: int) -> np.ndarray:
        """Apply the tell to mean[p0:p1] given the FULL fitness; return the slice."""


def gather_padded(dist, local: np.ndarray, total: int, world: int, rank: int,
                  device=None) -> np.ndarray:
    """All-gather equal-sized padded chunks (torch.distributed.all_gather_into_tensor)
    and return the first `total` rows concatenated in rank order."""
    import torch

    cs = math.ceil(total / world) if total > 0 else 0
    row = local.shape[1:] if local.ndim > 1 else ()
    buf = np.zeros((cs,) + tuple(row), local.dtype)
    buf[: len(local)] = local
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    out = torch.empty((world * cs,) + tuple(row), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t)
    return out.cpu().numpy()[:total]


def sharded_generation(dist, backend: Backend, pop: int, d: int, rank: int, world: int,
                       device=None) -> np.ndarray:
    """One generation with the two collectives; returns the new full mean."""
    a0, a1 = shard_range(pop, rank, world)
    fit_local, stats_local = backend.rollout(a0, a1)
    fitness = gather_padded(dist, fit_local, pop, world, rank, device)          # C1
    lane_stats = None
    if stats_local is not None:
        lane_stats = gather_padded(dist, stats_local, pop, world, rank, device)
    p0, p1 = shard_range(d, rank, world)
    mean_slice = backend.tell(fitness, lane_stats, p0, p1)
    return gather_padded(dist, mean_slice, d, world, rank, device)             # C2


class CudaShardedEs:
    """The product multi-GPU path: EsWorkflow handles sharded over ranks, with
    the collectives run by torch.distributed (NCCL) directly on the handle's
    device buffers."""

    def __init__(self, cfg, rank: int, world: int):
        import torch
        import torch.distributed as dist

        from .es import EsWorkflow

        self.torch = torch
        self.dist = dist
        self.rank, self.world = rank, world
        cfg.device = torch.cuda.current_device()
        self.es = EsWorkflow(cfg)
        self.cfg = cfg
        self.pop = cfg.pop
        self.d = self.es.dim
        self.e = cfg.fitness_episodes
        self.es.set_shard(rank, world)
        f_ptr, m_ptr, s_ptr = self.es.device_buffers()
        # zero-copy torch views of the handle's device buffers
        self.fitness = self._view(f_ptr, self.pop)
        self.mean = self._view(m_ptr, self.d)
        self.lane_stats = self._view(s_ptr, self.pop * self.e * 9)
        self.a0, self.a1, self.p0, self.p1 = self.es.shard_ranges()
        # equal-chunk staging buffers for all_gather_into_tensor
        self.acs = math.ceil(self.pop / world)
        self.pcs = math.ceil(self.d / world)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.fbuf = torch.zeros(self.acs, dtype=torch.float64, device=dev)
        self.fall = torch.zeros(self.acs * world, dtype=torch.float64, device=dev)
        self.mbuf = torch.zeros(self.pcs, dtype=torch.float64, device=dev)
        self.mall = torch.zeros(self.pcs * world, dtype=torch.float64, device=dev)
        self.cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        # per-lane RunningStats are tracked iff the handle's RESOLVED obs_norm
        # mode is running_stats (ARS's "auto", or an explicit running_stats for
        # any algorithm): every rank then merges all pop x e lanes in phase_tell
        from . import _lib
        self.track = self.es.norm_mode() == _lib.NORM["running_stats"]
        # CEM's tell updates diag_var on [p0, p1) only and the next ask reads
        # every coordinate: the variance is gathered like the mean
        self.cem = cfg.algo == "cem"
        if self.cem:
            self.var = self._view(self.es.device_var(), self.d)
            self.vbuf = torch.zeros(self.pcs, dtype=torch.float64, device=dev)
            self.vall = torch.zeros(self.pcs * world, dtype=torch.float64, device=dev)
        if self.track:
            self.sbuf = torch.zeros(self.acs * self.e * 9, dtype=torch.float64, device=dev)
            self.sall = torch.zeros(self.acs * self.e * 9 * world, dtype=torch.float64, device=dev)

    def _view(self, ptr, n):
        class _CAI:
            pass

        o = _CAI()
        o.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                      "version": 3, "strides": None}
        return self.torch.as_tensor(o, device="cuda")

    def _gather_slices(self, full, buf, allbuf):
        """All-gather the coordinate slices [p0, p1) of a d-vector in place."""
        npc = self.p1 - self.p0
        buf[:npc].copy_(full[self.p0:self.p1])
        self.dist.all_gather_into_tensor(allbuf, buf)
        for r in range(self.world):
            lo, hi = r * self.pcs, min(self.d, (r + 1) * self.pcs)
            if hi > lo:
                full[lo:hi].copy_(allbuf[r * self.pcs: r * self.pcs + hi - lo])

    def init(self, key):
        self.es.init(key)

    def step(self):
        torch, dist = self.torch, self.dist
        it0, steps0, eps0 = self.es.counters()
        self.es.phase_rollout()          # ask + rollout + fitness of [a0, a1) (synchronous)
        na = self.a1 - self.a0
        self.fbuf[:na].copy_(self.fitness[self.a0:self.a1])
        dist.all_gather_into_tensor(self.fall, self.fbuf)                         # C1
        for r in range(self.world):
            lo, hi = r * self.acs, min(self.pop, (r + 1) * self.acs)
            if hi > lo:
                self.fitness[lo:hi].copy_(self.fall[r * self.acs: r * self.acs + hi - lo])
        if self.track:
            w = self.e * 9
            self.sbuf[: na * w].copy_(self.lane_stats[self.a0 * w:self.a1 * w])
            dist.all_gather_into_tensor(self.sall, self.sbuf)
            for r in range(self.world):
                lo, hi = r * self.acs, min(self.pop, (r + 1) * self.acs)
                if hi > lo:
                    self.lane_stats[lo * w:hi * w].copy_(
                        self.sall[r * self.acs * w: r * self.acs * w + (hi - lo) * w])
        torch.cuda.synchronize()
        m = self.es.phase_tell()         # ranks + tell of [p0, p1) (synchronous)
        self._gather_slices(self.mean, self.mbuf, self.mall)                      # C2
        if self.cem:
            self._gather_slices(self.var, self.vbuf, self.vall)
            torch.cuda.synchronize()
            m.values["es/sigma"] = self.es.cem_sigma()
        # WorkflowState::env_steps counts the whole generation
        # (proj/src/workflow_es.cpp:134): each rank summed only its shard's lane
        # steps (episodes are pop x count on every rank), so the step deltas
        # are summed over ranks (8 bytes)
        it1, steps1, eps1 = self.es.counters()
        self.cnt.copy_(torch.tensor([steps1 - steps0], dtype=torch.int64))
        dist.all_reduce(self.cnt)
        self.es.set_counters(it1, steps0 + int(self.cnt.item()), eps1)
        torch.cuda.synchronize()
        return m
