"""fp64-accurate tensor-core rollout (precision "oz", rollout_oz.cu) against
the fp64 oracle.

The dense W2 x W1 layer runs as exact int8 tcgen05 MMAs over 6 byte slices of
per-row / per-lane fixed-point operands (~47 significant bits each, int32
accumulation, the S(S+1)/2 leading slice products); layer 0, the output layer,
the head and the env are fp64.  The policy output differs from fp64
arithmetic by ~1e-13 relative, so the closed-loop bar is the fp64 path's own
envelope: returns / fitness within RTOL_OZ of the CPU restatement, ranks
and step counts identical.
"""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL_OZ = 3e-8       # closed-loop returns / fitness (fp64 team: 1e-9, fp32 teams: 1e-4)


@pytest.fixture(scope="module")
def evb():
    import paper_2501_15129_b200 as m
    return m


def _policy(oracle, evb, env, hidden):
    ospec = oracle.policy_net_spec(oracle.env_spec(env), hidden)
    desc = evb.mlp_desc(ospec.input_dim, hidden, ospec.output_dim, ospec.head, ospec.tanh_scale)
    return ospec, desc


# (env, hidden, m, e, count, fixed, H): cluster sizes 1 / 2 / 4 (W2 / 128, rows
# past W2 zero-padded), W1 = 16 .. 256 (K zero-padded to 32), ragged 16-lane
# teams, uneven episode splits, CartPole with early termination (categorical, O = 2)
SHAPES = [
    ("pendulum", [256, 256], 4, 16, 16, True, 200),
    ("pendulum", [64, 256], 3, 16, 16, True, 200),
    ("pendulum", [97, 97], 3, 16, 16, True, 200),
    ("pendulum", [256, 512], 2, 16, 16, True, 100),
    ("pendulum", [100, 300], 2, 16, 16, True, 100),
    ("pendulum", [16, 128], 3, 16, 16, True, 200),
    ("pendulum", [256, 256], 3, 5, 7, True, 120),
    ("pendulum", [128, 256], 2, 40, 40, True, 80),
    ("cartpole", [64, 128], 6, 16, 16, False, 200),
    ("pendulum", [128, 1024], 2, 16, 16, True, 60),   # cluster of 8 CTAs
]


@pytest.mark.parametrize("env,hidden,m,e,count,fixed,H", SHAPES, ids=lambda v: str(v))
def test_oz_rollout_matches_oracle(oracle, evb, env, hidden, m, e, count, fixed, H):
    ospec, desc = _policy(oracle, evb, env, hidden)
    params = np.array([oracle.init_params(ospec, oracle.key_from_seed(700 + a)) for a in range(m)])
    params += 0.05 * np.random.default_rng(7).standard_normal(params.shape)
    key = oracle.key_from_seed(701)
    envspec = oracle.env_spec(env, fixed, H)
    onorm = oracle.lib().eo_vbn_fit(C.byref(envspec), oracle.key_from_seed(9), 500)
    want, wsteps, want_st = oracle.batched_rollout(envspec, ospec, onorm, params, e, key, count=count,
                                                   track=True, workers=0)
    got, steps, got_st = evb.batched_rollout(env, desc, params, e, key, count=count, obs_norm=onorm,
                                             fixed_horizon=fixed, max_episode_steps=H, precision="oz",
                                             track_obs_stats=True)
    assert list(steps) == list(wsteps)
    w = np.array(want)
    assert np.allclose(got, w, rtol=RTOL_OZ, atol=1e-12), np.abs(got - w).max()
    for a in range(m):
        assert got_st[a, 0] == want_st[a][0]
        assert np.allclose(got_st[a, 1:5], want_st[a][1], rtol=1e-7, atol=1e-9)


def test_oz_unsupported_shapes_run_as_fp64(oracle, evb):
    """Shapes outside the oz team (1 or 3 hidden layers, W1 > 256, < 5 lanes)
    run on the fp64 DMMA team: bit-identical to precision='f64'."""
    for hidden, e in (([300, 128], 16), ([64], 16), ([32, 16, 8], 16), ([64, 64], 2)):
        ospec, desc = _policy(oracle, evb, "pendulum", hidden)
        params = np.array([oracle.init_params(ospec, oracle.key_from_seed(900))])
        key = oracle.key_from_seed(901)
        a, _, _ = evb.batched_rollout("pendulum", desc, params, e, key, fixed_horizon=True,
                                      max_episode_steps=50, precision="oz")
        b, _, _ = evb.batched_rollout("pendulum", desc, params, e, key, fixed_horizon=True,
                                      max_episode_steps=50, precision="f64")
        assert np.array_equal(a, b), hidden


@pytest.mark.parametrize("where", ["w0", "w1", "b2"])
def test_oz_netfault_matches_fp64_team(oracle, evb, where):
    """Non-finite weights: rows of the sliced layer holding one take an fp64
    dot product, so the fault (kind, layer, lane) is the fp64 team's."""
    ospec, desc = _policy(oracle, evb, "pendulum", [128, 128])
    p = oracle.init_params(ospec, oracle.key_from_seed(1))[None].copy()
    idx = {"w0": 0, "w1": 3 * 128 + 128 + 5 * 128 + 7, "b2": -1}[where]
    p[0, idx] = np.inf
    msgs = []
    for prec in ("f64", "oz"):
        with pytest.raises((evb.NetFault, evb.EnvFault)) as ei:
            evb.batched_rollout("pendulum", desc, p, 16, oracle.key_from_seed(2), max_episode_steps=20,
                                precision=prec)
        msgs.append((type(ei.value), str(ei.value)))
    assert msgs[0] == msgs[1]


@pytest.mark.parametrize("kw", [
    dict(algo="openes", env="pendulum", fixed_horizon=True, pop=64, hidden=[64, 128],
         max_episode_steps=200, fitness_episodes=16, vbn_samples=2000),
    dict(algo="openes", env="cartpole", pop=32, hidden=[32, 128], max_episode_steps=100,
         fitness_episodes=8, vbn_samples=500),
    dict(algo="ars", env="pendulum", fixed_horizon=True, pop=32, hidden=[32, 128],
         max_episode_steps=100, fitness_episodes=16),
], ids=lambda k: f"{k['algo']}-{k['env']}")
def test_oz_workflow_generations_match_oracle(oracle, evb, kw):
    """Whole generations (ask -> oz rollout -> fitness -> ranks -> tell) against
    the oracle EsWorkflow: fitness within the fp64 envelope, ranks identical,
    the updated mean within it too."""
    o = oracle.OracleEs(oracle.es_config(workers=0, **kw))
    g = evb.EsWorkflow(evb.EsConfig(precision="oz", **{k: (tuple(v) if k == "hidden" else v)
                                                        for k, v in kw.items()}))
    key = oracle.key_from_seed(5)
    o.init(key)
    g.init(key)
    for gen in range(3):
        o.step()
        g.step()
        fo, fg = o.fitness(), g.fitness()
        assert np.allclose(fg, fo, rtol=RTOL_OZ, atol=1e-12), gen
        assert np.array_equal(np.argsort(fg, kind="stable"), np.argsort(fo, kind="stable")), gen
        mo, mg = o.mean(), g.mean()
        assert np.abs(mg - mo).max() <= RTOL_OZ * max(1.0, np.abs(mo).max()), gen
        assert g.counters() == o.counters()


def test_oz_config3_ranks_match_fp64_path(evb):
    """BASELINE config 3 (OpenES pop 4096 x 16 envs, 2x256, Pendulum H=200):
    from the same state, the oz and fp64-DMMA generations rank all 4096
    candidates identically and apply the bit-identical tell."""
    kw = dict(algo="openes", env="pendulum", fixed_horizon=True, pop=4096, fitness_episodes=16,
              hidden=(256, 256), max_episode_steps=200)
    r = evb.EsWorkflow(evb.EsConfig(precision="f64", **kw)).init((1, 2))
    g = evb.EsWorkflow(evb.EsConfig(precision="oz", **kw)).init((1, 2))
    for _ in range(2):
        g.set_mean(r.mean())
        m, v, t = r.adam()
        g.set_adam(m, v, t)
        g.set_counters(*r.counters())
        r.step()
        g.step()
        fr, fg = r.fitness(), g.fitness()
        assert np.allclose(fg, fr, rtol=RTOL_OZ, atol=0)
        assert np.array_equal(np.argsort(fg, kind="stable"), np.argsort(fr, kind="stable"))
        assert np.array_equal(g.mean(), r.mean())


@pytest.mark.parametrize("kw", [
    # Workflow::evaluate (m = 1 agent, 32 episodes -> two 16-lane teams) at the centre
    dict(algo="openes", env="pendulum", fixed_horizon=True, pop=16, hidden=[64, 128], max_episode_steps=150,
         fitness_episodes=8, vbn_samples=300),
    # the noise-table ask (SRC_OPENES_TABLE materialised, then pre-split)
    dict(algo="openes", env="pendulum", fixed_horizon=True, pop=16, hidden=[32, 128], max_episode_steps=100,
         fitness_episodes=8, vbn_samples=300, openes_noise_table=True, openes_noise_table_size=1 << 18),
    # CMA-ES: candidates from the device ask GEMM, no pre-split blocks (in-kernel slicing)
    dict(algo="cmaes", env="pendulum", fixed_horizon=True, pop=16, hidden=[16, 128], max_episode_steps=100,
         fitness_episodes=8, vbn_samples=300, cmaes_elites=8, cmaes_sigma0=0.1, cmaes_max_dim=4096),
    # VES (SRC_OPENES ask, no kept noise) and CEM (diagonal-variance ask)
    dict(algo="ves", env="pendulum", fixed_horizon=True, pop=16, hidden=[32, 128], max_episode_steps=100,
         fitness_episodes=8, vbn_samples=300, ves_elites=4),
    dict(algo="cem", env="pendulum", fixed_horizon=True, pop=16, hidden=[32, 128], max_episode_steps=100,
         fitness_episodes=8, cem_elites=4),
    # OpenES without mirroring (every agent its own noise row, kept ahead) and
    # with running_stats normalisation (per-lane Welford in the oz env warps)
    dict(algo="openes", env="pendulum", fixed_horizon=True, pop=12, hidden=[64, 128], max_episode_steps=100,
         fitness_episodes=8, openes_mirrored=False, obs_norm="running_stats"),
], ids=["evaluate", "noise-table", "cmaes", "ves", "cem", "openes-unmirrored-rs"])
def test_oz_other_callers_match_fp64(evb, kw):
    """The oz team behind the workflow's other callers: per-generation fitness
    within RTOL_OZ of the fp64 team from the same state, ranks identical, and
    Workflow::evaluate at the centre within RTOL_OZ."""
    kwc = {k: (tuple(v) if k == "hidden" else v) for k, v in kw.items()}
    a = evb.EsWorkflow(evb.EsConfig(precision="f64", **kwc)).init((21, 22))
    b = evb.EsWorkflow(evb.EsConfig(precision="oz", **kwc)).init((21, 22))
    for _ in range(2):
        a.step()
        b.step()
        fa, fb = a.fitness(), b.fitness()
        assert np.allclose(fb, fa, rtol=RTOL_OZ, atol=1e-12)
        assert np.array_equal(np.argsort(fa, kind="stable"), np.argsort(fb, kind="stable"))
    b.set_mean(a.mean())
    ma, sa = a.evaluate(32, (5, 6))
    mb, sb = b.evaluate(32, (5, 6))
    assert mb == pytest.approx(ma, rel=RTOL_OZ)
    assert sb == pytest.approx(sa, rel=1e-6, abs=1e-9)
