"""The product multi-GPU path (paper_2501_15129_b200.dist.CudaShardedEs) run
end to end on one B200 with two ranks.

NCCL refuses two ranks on one device, so the collectives go through the gloo
backend on the same CUDA buffers (torch's gloo all_gather_into_tensor accepts
CUDA tensors); the ranks' kernels never wait on each other.  The sharded
generation must be bit-identical to the single-process workflow (population
shards, coordinate-sharded tell)."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CFGS = {
    "openes": dict(algo="openes", env="pendulum", fixed_horizon=True, pop=30, hidden=(16, 16),
                   max_episode_steps=60, vbn_samples=300, fitness_episodes=2),
    "ars": dict(algo="ars", env="pendulum", fixed_horizon=True, pop=34, hidden=(8,), max_episode_steps=60),
    "cmaes": dict(algo="cmaes", env="pendulum", fixed_horizon=True, pop=16, hidden=(4,), max_episode_steps=40,
                  vbn_samples=200, cmaes_elites=8, cmaes_sigma0=0.2),
    # CEM: the diagonal variance is coordinate-sharded too (gathered like the mean)
    "cem": dict(algo="cem", env="pendulum", fixed_horizon=True, pop=20, hidden=(8,), max_episode_steps=40,
                vbn_samples=200, cem_elites=6),
    "ves": dict(algo="ves", env="pendulum", fixed_horizon=True, pop=24, hidden=(8,), max_episode_steps=40,
                vbn_samples=200, ves_elites=6),
    # running_stats with a non-ARS algorithm: the lane stats must be gathered
    "openes_rs": dict(algo="openes", env="pendulum", fixed_horizon=True, pop=22, hidden=(8,),
                      max_episode_steps=50, obs_norm="running_stats", fitness_episodes=2),
    # many row chunks in the tell (384 base rows, d = 133121): sized from the
    # shard span the chunking would be 10 row chunks on one GPU and 12 per rank
    # at world 2 (a different summation order of the search gradient)
    # the oz team: per-rank noise rows kept ahead (generated beside the rollout)
    # and the ask fused with the layer-1 pre-split, on each rank's own rows
    "openes_oz": dict(algo="openes", env="pendulum", fixed_horizon=True, pop=40, hidden=(128, 128),
                      max_episode_steps=30, fitness_episodes=16, precision="oz"),
    "openes_chunks": dict(algo="openes", env="pendulum", fixed_horizon=True, pop=768, hidden=(256, 512),
                          max_episode_steps=20, vbn_samples=200),
}
GENS = 3


def _rank_main(rank, world, algo, port, out_dir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    import paper_2501_15129_b200 as evb
    from paper_2501_15129_b200.dist import CudaShardedEs

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = CudaShardedEs(evb.EsConfig(**CFGS[algo]), rank, world)
    r.init((61, 62))
    for _ in range(GENS):
        m = r.step()
    torch.cuda.synchronize()
    if rank == 0:
        np.save(os.path.join(out_dir, "sigma.npy"), np.array([m["es/sigma"]]))
        np.save(os.path.join(out_dir, "mean.npy"), r.es.mean())
        np.save(os.path.join(out_dir, "fitness.npy"), r.es.fitness())
        np.save(os.path.join(out_dir, "counters.npy"), np.array(r.es.counters()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("algo", sorted(CFGS))
def test_two_rank_sharded_generations_bit_identical(algo, tmp_path):
    import torch.multiprocessing as mp

    import paper_2501_15129_b200 as evb

    port = 29600 + sorted(CFGS).index(algo)
    mp.spawn(_rank_main, args=(2, algo, port, str(tmp_path)), nprocs=2, join=True)
    g = evb.EsWorkflow(evb.EsConfig(**CFGS[algo])).init((61, 62))
    for _ in range(GENS):
        m = g.step()
    assert np.array_equal(np.load(tmp_path / "mean.npy"), g.mean())
    assert np.array_equal(np.load(tmp_path / "fitness.npy"), g.fitness())
    assert tuple(np.load(tmp_path / "counters.npy")) == g.counters()
    if algo == "cem":
        assert np.array_equal(np.load(tmp_path / "sigma.npy"), np.array([m["es/sigma"]]))
