"""Oracle rollout grid and ES workflow invariants, mirroring
proj/tests/test_rollout.cpp and proj/tests/test_workflow.cpp."""
import numpy as np


def pend_policy(oracle):
    return oracle.mlp_spec(3, [8], 1, oracle.EO_HEAD_TANH, 2.0)


def test_grid_equals_solo_lanes_and_worker_invariance(oracle):
    # proj/tests/test_rollout.cpp:59-89 and :117-145
    env = oracle.env_spec("pendulum", False, 40)
    spec = pend_policy(oracle)
    params = np.array([oracle.init_params(spec, oracle.key_from_seed(300 + a)) for a in range(6)])
    key = oracle.key_from_seed(301)
    none = oracle.lib().eo_obs_norm_none()
    runs = [oracle.batched_rollout(env, spec, none, params, 4, key, track=True, workers=w)
            for w in (1, 3, 8)]
    for r in runs[1:]:
        for a in range(6):
            assert np.array_equal(r[0][a], runs[0][0][a])
            assert r[2][a] == runs[0][2][a]
    # lane (a, j) == a solo lane keyed fold_in(fold_in(key, a), j)
    import ctypes as C
    L = oracle.lib()
    pol = oracle.Policy()
    pol.spec = C.pointer(spec)
    pol.obs_norm = C.pointer(none)
    for a in range(6):
        solo = []
        for j in range(4):
            out = oracle.AgentRollout()
            oracle.check(L.eo_rollout_lane(C.byref(env), C.byref(pol), oracle.ptr(params[a]), 0, 1, 1,
                                           oracle.fold_in(oracle.fold_in(key, a), j), 0, 0,
                                           C.byref(out)))
            solo.append(out.episode_returns[0])
            L.eo_agent_rollout_free(C.byref(out))
        assert np.array_equal(runs[0][0][a], np.array(solo))


def test_uneven_episode_split(oracle):
    # proj/tests/test_rollout.cpp:91-115: 7 episodes over 3 lanes -> 3, 2, 2
    env = oracle.env_spec("cartpole", False, 10)
    spec = oracle.mlp_spec(4, [8], 2, oracle.EO_HEAD_CATEGORICAL)
    params = oracle.init_params(spec, oracle.key_from_seed(210))[None]
    rets, steps, _ = oracle.batched_rollout(env, spec, oracle.lib().eo_obs_norm_none(), params, 3,
                                            oracle.key_from_seed(211), count=7)
    assert len(rets[0]) == 7


def test_vbn_standardizes(oracle):
    # proj/tests/test_rollout.cpp:262-289
    import ctypes as C
    env = oracle.env_spec("pendulum")
    v = oracle.lib().eo_vbn_fit(C.byref(env), oracle.key_from_seed(350), 5000)
    assert v.mode == oracle.EO_NORM_VBN and v.count == 5000.0
    v2 = oracle.lib().eo_vbn_fit(C.byref(env), oracle.key_from_seed(350), 5000)
    assert list(v.mean) == list(v2.mean) and list(v.var) == list(v2.var)


def small_cfg(oracle, **kw):
    # proj/tests/test_workflow.cpp:17-25 small_config("es")
    base = dict(pop=8, hidden=[8], vbn_samples=300, max_episode_steps=50)
    base.update(kw)
    return oracle.es_config(**base)


def run(oracle, cfg, gens, seed=5):
    es = oracle.OracleEs(cfg)
    es.init(oracle.key_from_seed(seed))
    ms = [es.step() for _ in range(gens)]
    return es, ms


def test_workflow_worker_invariance_all_algos(oracle):
    # proj/tests/test_workflow.cpp:163-171
    for algo in ("openes", "ars", "ves", "cmaes", "cem"):
        outs = []
        for w in (1, 3):
            extra = {"cma.elites": 4} if algo == "cmaes" else {}
            es, ms = run(oracle, small_cfg(oracle, algo=algo, workers=w, **extra), 3)
            outs.append((es.mean().tobytes(), es.fitness().tobytes(), es.counters(),
                         [(m.fitness_mean, m.sigma, m.update_skipped) for m in ms]))
        assert outs[0] == outs[1], algo


def test_openes_pendulum_improves(oracle):
    """Sanity: OpenES on fixed-horizon pendulum raises mean fitness."""
    cfg = oracle.es_config(env="pendulum", fixed_horizon=1, pop=64, hidden=[16],
                           max_episode_steps=100, vbn_samples=1000, workers=0)
    es, ms = run(oracle, cfg, 30, seed=0)
    first = np.mean([m.fitness_mean for m in ms[:5]])
    last = np.mean([m.fitness_mean for m in ms[-5:]])
    assert last > first
    it, steps, eps = es.counters()
    assert it == 30 and steps == 30 * 64 * 100 and eps == 30 * 64


def test_oracle_transitions_follow_reference_semantics(oracle):
    """collect_transitions (proj/src/rollout.cpp:118-170): one row per step,
    lane-major per agent with lane_bounds; next_obs = final_obs (the true
    successor even across auto-reset), so next_obs[i] == obs[i+1] inside an
    episode; rewards of an episode sum to its return; flags close episodes."""
    env = oracle.env_spec("cartpole", False, 40)
    spec = oracle.policy_net_spec(env, [8])
    m, e, count = 3, 2, 4  # 2 episodes per lane
    params = np.array([oracle.init_params(spec, oracle.key_from_seed(70 + a)) for a in range(m)])
    rets, steps, _, batches = oracle.batched_rollout(env, spec, None, params, e, oracle.key_from_seed(71),
                                                     count=count, workers=0, collect=True)
    for a in range(m):
        b = batches[a]
        n = len(b["rewards"])
        assert n == steps[a] and b["lane_bounds"][0] == 0 and b["lane_bounds"][-1] == n
        ends = np.flatnonzero(b["terminated"] | b["truncated"])
        assert len(ends) == count
        assert set(b["lane_bounds"][1:] - 1) <= set(ends)
        start = 0
        for k, end in enumerate(ends):
            assert abs(b["rewards"][start:end + 1].sum() - rets[a][k]) < 1e-9
            assert np.array_equal(b["next_obs"][start:end], b["obs"][start + 1:end + 1])
            start = end + 1
        assert b["actions"].shape == (n, 1) and set(np.unique(b["actions"])) <= {0.0, 1.0}
