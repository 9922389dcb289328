"""Tensor-core (tcgen05) rollout: EVORL_PREC_TC against the fp64 oracle.

The W2 x W1 hidden layer runs on tcgen05 as a 3-pass fp16 hi/lo split with
fp32 TMEM accumulation (rollout_tc.cu); the other layers are fp32 on the CUDA
cores and the env stays fp64.  Tolerance: RTOL_F32 on returns, the same bar as
the fp32 SIMT path (north star: "fp32 tolerance").
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL_F32 = 1e-4


@pytest.fixture(scope="module")
def evb():
    import paper_2501_15129_b200 as m
    return m


def _policy(oracle, evb, env, hidden):
    ospec = oracle.policy_net_spec(oracle.env_spec(env), hidden)
    desc = evb.mlp_desc(ospec.input_dim, hidden, ospec.output_dim, ospec.head, ospec.tanh_scale)
    return ospec, desc


# (hidden, m, e, count): W2/128 = cluster size 1, 2, 4; W1 = 16..256; ragged teams
SHAPES = [
    ([256, 256], 4, 16, 16),
    ([128, 128], 3, 16, 16),
    ([64, 256], 2, 16, 16),
    ([256, 512], 2, 16, 16),
    ([16, 128], 2, 16, 16),
    ([256, 256], 3, 5, 7),     # padded 16-lane team, uneven episode split 2,2,1,1,1
    ([128, 256], 2, 40, 40),   # three teams per agent, last one ragged
    ([97, 97], 2, 16, 16),     # zero-padded K (112) and rows (128)
    ([64, 64], 2, 16, 16),
    ([100, 300], 2, 16, 16),   # cluster of 4: the last CTA holds only padding rows
]


@pytest.mark.parametrize("hidden,m,e,count", SHAPES, ids=lambda v: str(v))
def test_tc_rollout_within_fp32_tolerance(oracle, evb, hidden, m, e, count):
    ospec, desc = _policy(oracle, evb, "pendulum", hidden)
    params = np.array([oracle.init_params(ospec, oracle.key_from_seed(700 + a)) for a in range(m)])
    params += 0.02 * np.random.default_rng(7).standard_normal(params.shape)
    key = oracle.key_from_seed(701)
    envspec = oracle.env_spec("pendulum", True, 200)
    onorm = oracle.lib().eo_vbn_fit(C.byref(envspec), oracle.key_from_seed(9), 500)
    want, wsteps, want_st = oracle.batched_rollout(envspec, ospec, onorm, params, e, key, count=count,
                                                   track=True, workers=0)
    got, steps, got_st = evb.batched_rollout("pendulum", desc, params, e, key, count=count,
                                             obs_norm=onorm, fixed_horizon=True, max_episode_steps=200,
                                             precision="tc", track_obs_stats=True)
    assert list(steps) == list(wsteps)
    w = np.array(want)
    rel = np.abs(got - w) / np.abs(w)
    assert np.median(rel) < 1e-5 and rel.max() < RTOL_F32, (np.median(rel), rel.max())
    for a in range(m):
        assert got_st[a, 0] == want_st[a][0]
        assert np.allclose(got_st[a, 1:5], want_st[a][1], rtol=1e-3, atol=1e-6)


def test_tc_matches_fp32_simt_path(oracle, evb):
    """tc and the fp32 SIMT team agree with each other as closely as each
    agrees with fp64 (both are fp32-level evaluations of the same policy)."""
    ospec, desc = _policy(oracle, evb, "pendulum", [256, 256])
    m, e = 4, 16
    params = np.array([oracle.init_params(ospec, oracle.key_from_seed(800 + a)) for a in range(m)])
    key = oracle.key_from_seed(801)
    f32, _, _ = evb.batched_rollout("pendulum", desc, params, e, key, fixed_horizon=True,
                                    max_episode_steps=200, precision="f32")
    tc, _, _ = evb.batched_rollout("pendulum", desc, params, e, key, fixed_horizon=True,
                                   max_episode_steps=200, precision="tc")
    f64, _, _ = evb.batched_rollout("pendulum", desc, params, e, key, fixed_horizon=True,
                                    max_episode_steps=200, precision="f64")
    assert np.abs(tc - f64).max() / np.abs(f64).max() < RTOL_F32
    assert np.abs(tc - f32).max() / np.abs(f64).max() < RTOL_F32


def test_tc_unsupported_shape_runs_as_fp32(oracle, evb):
    """Shapes outside the tcgen05 team (1 or 3 hidden layers, W1 beyond the
    TMEM-resident A_hi) run on the fp32 team -- same answer as precision='f32'."""
    for hidden in ([512, 128], [64], [32, 16, 8]):
        ospec, desc = _policy(oracle, evb, "pendulum", hidden)
        params = np.array([oracle.init_params(ospec, oracle.key_from_seed(900))])
        key = oracle.key_from_seed(901)
        a, _, _ = evb.batched_rollout("pendulum", desc, params, 16, key, fixed_horizon=True,
                                      max_episode_steps=50, precision="tc")
        b, _, _ = evb.batched_rollout("pendulum", desc, params, 16, key, fixed_horizon=True,
                                      max_episode_steps=50, precision="f32")
        assert np.array_equal(a, b)


def test_tc_netfault(oracle, evb):
    ospec, desc = _policy(oracle, evb, "pendulum", [128, 128])
    p = oracle.init_params(ospec, oracle.key_from_seed(1))[None].copy()
    p[0, 0] = np.inf  # W0[0,0]: non-finite layer-0 activations
    with pytest.raises((evb.NetFault, evb.EnvFault)):
        evb.batched_rollout("pendulum", desc, p, 16, oracle.key_from_seed(2), max_episode_steps=5,
                            precision="tc")
    q = oracle.init_params(ospec, oracle.key_from_seed(1))[None].copy()
    q[0, -1] = np.inf  # output bias -> non-finite head input: NetFault at layer 2
    with pytest.raises(evb.NetFault, match="layer 2"):
        evb.batched_rollout("pendulum", desc, q, 16, oracle.key_from_seed(2), max_episode_steps=5,
                            precision="tc")


def test_tc_workflow_generation(oracle, evb):
    """One OpenES generation with the config-3 policy (2x256, 16 envs) in tc
    mode against the fp64 oracle: fitness within RTOL_F32, Adam-updated mean
    within the fp32 envelope."""
    kw = dict(algo="openes", env="pendulum", fixed_horizon=True, pop=64, hidden=[256, 256],
              max_episode_steps=200, fitness_episodes=16)
    o = oracle.OracleEs(oracle.es_config(workers=0, **kw))
    g = evb.EsWorkflow(evb.EsConfig(precision="tc", **{k: (tuple(v) if k == "hidden" else v)
                                                        for k, v in kw.items()}))
    key = oracle.key_from_seed(5)
    o.init(key)
    g.init(key)
    o.step()
    g.step()
    fo, fg = o.fitness(), g.fitness()
    assert np.allclose(fg, fo, rtol=RTOL_F32, atol=1e-9)
    assert g.counters() == o.counters()
    # ranks: at most a few adjacent swaps between near-tied candidates
    ro, rg = np.argsort(np.argsort(fo)), np.argsort(np.argsort(fg))
    assert np.abs(ro - rg).max() <= 2
    # Workflow::evaluate on the tensor-core team (32 episodes -> 16-lane teams)
    ek = oracle.key_from_seed(99)
    g.set_mean(o.mean())
    mr_o, sd_o = o.evaluate(32, ek)
    mr_g, sd_g = g.evaluate(32, ek)
    assert mr_g == pytest.approx(mr_o, rel=RTOL_F32)
    assert sd_g == pytest.approx(sd_o, rel=1e-2, abs=1e-3)


def test_tc_operand_range_is_reported(oracle, evb):
    """A finite layer-0 activation beyond the fp16 hi/lo range cannot be
    represented on the tensor-core path: reported as Unsupported (never a
    silently wrong return)."""
    ospec, desc = _policy(oracle, evb, "pendulum", [128, 128])
    p = oracle.init_params(ospec, oracle.key_from_seed(1))[None].copy()
    p[0, ospec_bias0(ospec)] = 1e6  # layer-0 bias of row 0: h = 1e6 > 60000
    with pytest.raises(evb.Unsupported, match="fp16"):
        evb.batched_rollout("pendulum", desc, p, 16, oracle.key_from_seed(2), max_episode_steps=5,
                            precision="tc")


def ospec_bias0(ospec):
    # flat layout (proj/src/net.cpp:26-48): W0 (obs x W1, column-major) then b0
    return ospec.input_dim * 128


@pytest.mark.parametrize("precision", ["tc", "f32", "f64", "oz"])
@pytest.mark.parametrize("algo", ["openes", "ars"])
def test_sharded_materialised_ask_matches_unsharded(evb, precision, algo):
    """The fp32 paths materialise the shard's candidates [a0, a1) once per
    generation (run_materialize_f32; for mirrored OpenES one Box-Muller pair
    feeds both mirrored agents).  Three shard handles (shard 1 straddles the
    mirror boundary pop/2) must reproduce the unsharded fitness bit for bit."""
    kw = dict(algo=algo, env="pendulum", fixed_horizon=True, pop=64, fitness_episodes=16,
              hidden=(128, 128), max_episode_steps=50, precision=precision)
    key = (7, 8)
    full = evb.EsWorkflow(evb.EsConfig(**kw)).init(key)
    full.step()
    want = full.fitness()
    got = np.full(64, np.nan)
    for r in range(3):
        h = evb.EsWorkflow(evb.EsConfig(**kw))
        h.set_shard(r, 3)
        h.init(key)
        h.phase_rollout()
        a0, a1, _, _ = h.shard_ranges()
        got[a0:a1] = h.fitness()[a0:a1]
    assert np.array_equal(got, want)


def test_tc_categorical_two_outputs(oracle, evb):
    """CartPole (categorical head, O = 2 outputs through the epilogue's
    per-output reduce-scatter) on the tensor-core team: episode lengths are
    integers, so an fp32 argmax near-tie can change a return -- the bar is
    that almost every episode matches the fp64 oracle exactly."""
    ospec, desc = _policy(oracle, evb, "cartpole", [128, 256])
    m, e = 8, 16
    params = np.array([oracle.init_params(ospec, oracle.key_from_seed(950 + a)) for a in range(m)])
    key = oracle.key_from_seed(951)
    envspec = oracle.env_spec("cartpole", False, 200)
    want, wsteps, _ = oracle.batched_rollout(envspec, ospec, None, params, e, key, workers=0)
    got, steps, _ = evb.batched_rollout("cartpole", desc, params, e, key, max_episode_steps=200,
                                        precision="tc")
    w = np.array(want)
    assert (got == w).mean() >= 0.95, (got == w).mean()
    assert abs(got.mean() - w.mean()) <= 0.02 * w.mean()
