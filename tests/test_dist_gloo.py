"""Multi-process (gloo, world_size 2, CPU) tests of the population-sharded
generation (paper_2501_15129_b200/dist.py): rank r rolls out agents [a0, a1),
fitness is all-gathered (C1), each rank applies the OpenES tell + Adam to its
coordinate slice [p0, p1) only, and the mean slices are all-gathered (C2).
The per-rank compute here is the oracle (test infrastructure); the product
backend is CudaShardedEs.  The sharded result must be bit-identical to the
single-process oracle generation, for any world size."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


KW = dict(algo="openes", env="pendulum", fixed_horizon=1, pop=12, hidden=[8],
          max_episode_steps=30, vbn_samples=200, fitness_episodes=2)


class OracleShardBackend:
    """OpenES generation phases restated per shard on the CPU oracle."""

    def __init__(self, oracle, seed):
        self.o = oracle
        self.L = oracle.lib()
        cfg = oracle.es_config(**KW, workers=1)
        self.ref = oracle.OracleEs(cfg)  # used only for init state + specs
        self.ref.init(oracle.key_from_seed(seed))
        self.mean = self.ref.mean()
        self.d = len(self.mean)
        self.m = np.zeros(self.d)
        self.v = np.zeros(self.d)
        self.t = 0
        self.norm = self.ref.obs_norm()
        self.rng = oracle.key_from_seed(seed)
        self.it = 0
        self.pop = KW["pop"]
        self.e = KW["fitness_episodes"]

    def keys(self):
        o = self.o
        k = o.fold_in(o.fold_in(self.rng, 0), self.it)
        return o.fold_in(k, 0), o.fold_in(k, 1)

    def eps(self):
        ask, _ = self.keys()
        base = self.pop // 2
        e = self.o.gaussian_matrix(ask, base, self.d)
        return np.vstack([e, -e])

    def rollout(self, a0, a1):
        o = self.o
        _, rk = self.keys()
        eps = self.eps()
        cand = 0.02 * eps + self.mean
        env = self.ref.env()
        net = self.ref.net()
        pol = o.Policy()
        pol.spec = C.pointer(net)
        pol.obs_norm = C.pointer(self.norm)
        fit = np.zeros(a1 - a0)
        for a in range(a0, a1):
            s = 0.0
            p = np.ascontiguousarray(cand[a])
            for j in range(self.e):
                out = o.AgentRollout()
                o.check(self.L.eo_rollout_lane(C.byref(env), C.byref(pol), o.ptr(p), 0, self.e, 1,
                                               o.fold_in(o.fold_in(rk, a), j), 0, 0, C.byref(out)))
                s += out.episode_returns[0]
                self.L.eo_agent_rollout_free(C.byref(out))
            fit[a - a0] = s / self.e
        return fit, None

    def tell(self, fitness, lane_stats, p0, p1):
        shaped = self.o.centered_ranks(fitness)
        eps = self.eps()
        acc = np.zeros(p1 - p0)
        for i in range(self.pop):  # sequential i, like the oracle's loop
            acc = acc + eps[i, p0:p1] * shaped[i]
        g = -(acc / (self.pop * 0.02))
        t = self.t + 1
        m = 0.9 * self.m[p0:p1] + (1.0 - 0.9) * g
        v = 0.999 * self.v[p0:p1] + (1.0 - 0.999) * (g * g)
        bc1, bc2 = 1.0 - 0.9 ** t, 1.0 - 0.999 ** t
        p = self.mean[p0:p1] - 0.01 * (m / bc1) / (np.sqrt(v / bc2) + 1e-8)
        p = p - (0.01 * 0.005) * p
        self.m[p0:p1], self.v[p0:p1] = m, v
        return p

    def commit(self, mean):
        self.mean = mean
        self.t += 1
        self.it += 1


def _worker(rank, world, port, seed, gens, q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import torch.distributed as dist

    import oracle_ffi as oracle
    from paper_2501_15129_b200.dist import sharded_generation
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    be = OracleShardBackend(oracle, seed)
    for _ in range(gens):
        mean = sharded_generation(dist, be, be.pop, be.d, rank, world)
        be.commit(mean)
    q.put((rank, be.mean.tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def run_world(world, seed=3, gens=3):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, gens, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_shard_range_partitions():
    from paper_2501_15129_b200.dist import shard_range
    for n in (1, 7, 12, 4096, 67073):
        for w in (1, 2, 3, 4, 8):
            parts = [shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))


@pytest.mark.parametrize("world", [2])
def test_sharded_generation_equals_single_process(oracle, world):
    out = run_world(world)
    # every rank ends with the same mean
    vals = list(out.values())
    assert all(v == vals[0] for v in vals)
    mean_w = np.frombuffer(vals[0])
    # single-process oracle EsWorkflow, same seed, same number of generations
    es = oracle.OracleEs(oracle.es_config(**KW, workers=1))
    es.init(oracle.key_from_seed(3))
    for _ in range(3):
        es.step()
    assert np.array_equal(mean_w, es.mean())
    # world size 1 through the same sharded code path is identical too
    out1 = run_world(1)
    assert np.frombuffer(out1[0]).tobytes() == vals[0]
