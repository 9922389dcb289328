"""The pipelined fp64 DMMA team (opt-in, EVORL_FP64_PIPE=1) (rollout_pipe_kernel: two 8-lane groups, an
env warp overlapping the other group's GEMMs) vs the CPU oracle, over the
shapes that select it (2 hidden layers, >= 5 lanes per agent, fp64): dead
and partial groups, multi-team agents, ragged episodes, categorical heads,
odd slice widths, RunningStats tracking and NetFault attribution."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL_CLOSED = 1e-9


@pytest.fixture(scope="module")
def evb():
    import paper_2501_15129_b200 as m
    return m


@pytest.fixture(autouse=True)
def _pipe_on(monkeypatch):
    # the team is opt-in; the plan reads the variable per call
    monkeypatch.setenv("EVORL_FP64_PIPE", "1")


def _policy(oracle, evb, env, hidden):
    ospec = oracle.policy_net_spec(oracle.env_spec(env), hidden)
    desc = evb.mlp_desc(ospec.input_dim, hidden, ospec.output_dim, ospec.head, ospec.tanh_scale)
    return ospec, desc


@pytest.mark.parametrize("env,hidden,m,e,count,fixed,H", [
    ("pendulum", [64, 64], 2, 5, 5, True, 60),      # group B has no lanes
    ("pendulum", [64, 64], 2, 12, 12, True, 60),    # group B partial
    ("pendulum", [64, 64], 2, 20, 20, True, 40),    # two teams per agent, the second partial
    ("pendulum", [64, 64], 2, 16, 10, True, 40),    # lanes without episodes
    ("pendulum", [20, 36], 3, 16, 16, True, 50),    # odd widths: slice 18 rows (padded to 24)
    ("pendulum", [128, 256], 2, 16, 33, True, 30),  # multi-episode lanes (33 over 16)
    ("cartpole", [32, 32], 3, 16, 40, False, 120),  # categorical, terminations, ragged lanes
    ("cartpole", [64, 96], 2, 7, 7, False, 200),
])
def test_pipe_matches_oracle(oracle, evb, env, hidden, m, e, count, fixed, H):
    ospec, desc = _policy(oracle, evb, env, hidden)
    params = np.array([oracle.init_params(ospec, oracle.key_from_seed(700 + a)) for a in range(m)])
    params += 0.3 * np.random.default_rng(7).standard_normal(params.shape)
    key = oracle.key_from_seed(701)
    envspec = oracle.env_spec(env, fixed, H)
    onorm = oracle.lib().eo_vbn_fit(C.byref(envspec), oracle.key_from_seed(9), 500)
    want_r, want_s, want_st = oracle.batched_rollout(envspec, ospec, onorm, params, e, key,
                                                     count=count, track=True, workers=0)
    got_r, got_s, got_st = evb.batched_rollout(env, desc, params, e, key, count=count, obs_norm=onorm,
                                               fixed_horizon=fixed, max_episode_steps=H,
                                               track_obs_stats=True)
    assert list(got_s) == list(want_s)
    for a in range(m):
        assert np.allclose(got_r[a], want_r[a], rtol=RTOL_CLOSED, atol=1e-12), (a, got_r[a], want_r[a])
        assert got_st[a, 0] == want_st[a][0]
        assert np.allclose(got_st[a, 1:5], want_st[a][1], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("where,layer", [("b0", 0), ("b1", 1), ("bout", 2)])
def test_pipe_netfault_layer(oracle, evb, where, layer):
    ospec, desc = _policy(oracle, evb, "pendulum", [64, 64])
    p = oracle.init_params(ospec, oracle.key_from_seed(3))[None].repeat(2, 0)
    # layout (proj/src/net.cpp:26-48): W0 (64x3), b0 (64), W1 (64x64), b1 (64), Wout (1x64), bout (1)
    idx = {"b0": 3 * 64, "b1": 3 * 64 + 64 + 64 * 64 + 5, "bout": p.shape[1] - 1}[where]
    p[1, idx] = np.inf
    with pytest.raises(evb.NetFault, match=f"layer {layer}"):
        evb.batched_rollout("pendulum", desc, p, 16, oracle.key_from_seed(4), fixed_horizon=True,
                            max_episode_steps=20)
    # the same agent through the oracle raises at the same layer
    with pytest.raises(oracle.OracleError, match=f"layer {layer}"):
        oracle.batched_rollout(oracle.env_spec("pendulum", True, 20), ospec, None, p, 16,
                               oracle.key_from_seed(4), workers=0)
