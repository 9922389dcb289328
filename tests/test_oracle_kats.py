"""Oracle vs the reference's hot-path known-answer tests:
proj/tests/test_env.cpp, test_net.cpp, test_ec.cpp, test_optim.cpp,
test_obs_norm.cpp.  Tolerances are the reference tests' own."""
import ctypes as C
import math

import numpy as np
import pytest


def approx(a, b, eps):  # doctest::Approx(b).epsilon(eps): |a-b| < eps*(1 + max(|a|,|b|))
    return abs(a - b) < eps * (1.0 + max(abs(a), abs(b)))


def step(oracle, spec, phys, action):
    L = oracle.lib()
    s = oracle.EnvState()
    for i, v in enumerate(phys):
        s.phys[i] = v
    nxt = oracle.EnvState()
    r = C.c_double()
    te = C.c_int()
    tr = C.c_int()
    a = (C.c_double * 1)(action)
    rc = L.eo_env_step(C.byref(spec), C.byref(s), a, C.byref(nxt), C.byref(r), C.byref(te),
                       C.byref(tr), None)
    return rc, nxt, r.value, te.value, tr.value


def test_env_specs(oracle):
    cp = oracle.env_spec("cartpole")
    assert (cp.obs_dim, cp.discrete, cp.num_actions, cp.max_episode_steps) == (4, 1, 2, 500)
    pd = oracle.env_spec("pendulum")
    assert (pd.obs_dim, pd.discrete, pd.act_dim, pd.act_low, pd.act_high,
            pd.max_episode_steps) == (3, 0, 1, -2.0, 2.0, 200)
    assert oracle.env_spec("pendulum", False, 77).max_episode_steps == 77


def test_cartpole_one_step(oracle):
    # proj/tests/test_env.cpp:46-66
    spec = oracle.env_spec("cartpole")
    rc, s1, r, te, tr = step(oracle, spec, (0.01, -0.02, 0.03, 0.04), 1.0)
    assert rc == 0 and r == 1.0 and not te and not tr and s1.step_count == 1
    for got, want in zip(s1.phys, (0.009600000000000001, 0.17467919574755525,
                                   0.030799999999999998, -0.24306871796000815)):
        assert approx(got, want, 1e-14)
    rc, s2, r, *_ = step(oracle, spec, (0.01, -0.02, 0.03, 0.04), 0.0)
    assert approx(s2.phys[1], -0.21553901710278936, 1e-14)
    assert approx(s2.phys[3], 0.3419952237760392, 1e-14)


def test_pendulum_one_step(oracle):
    # proj/tests/test_env.cpp:68-89
    spec = oracle.env_spec("pendulum")
    _, s1, r1, *_ = step(oracle, spec, (1.0, 0.5), 1.0)
    assert approx(s1.phys[0], 1.064055161930296, 1e-14)
    assert approx(s1.phys[1], 1.2811032386059225, 1e-14)
    assert approx(r1, -1.026, 1e-12)
    _, s2, r2, *_ = step(oracle, spec, (3.0, -0.2), -3.0)
    assert approx(s2.phys[0], 2.980292000302245, 1e-14)
    assert approx(s2.phys[1], -0.3941599939550996, 1e-14)
    assert approx(r2, -9.008, 1e-12)
    _, s3, r3, *_ = step(oracle, spec, (3.3, 0.0), 0.0)
    assert approx(r3, -8.899394576972163, 1e-12)
    assert approx(s3.phys[0], 3.294084536469628, 1e-14)


def test_cartpole_termination_and_horizon(oracle):
    # proj/tests/test_env.cpp:120-163
    spec = oracle.env_spec("cartpole")
    assert step(oracle, spec, (2.39, 3.0, 0.0, 0.0), 1.0)[3] == 1
    assert step(oracle, spec, (0.0, 0.0, 0.205, 0.5), 1.0)[3] == 1
    assert step(oracle, spec, (0.0, 0.0, 0.0, 0.0), 1.0)[3] == 0
    one = oracle.env_spec("cartpole", False, 1)
    _, _, _, te, tr = step(oracle, one, (2.39, 3.0, 0.0, 0.0), 1.0)
    assert te == 1 and tr == 0
    fh = oracle.env_spec("cartpole", True, 3)
    _, _, _, te, tr = step(oracle, fh, (2.39, 3.0, 0.0, 0.0), 1.0)
    assert te == 0


def test_env_reset_and_fault(oracle):
    # proj/tests/test_env.cpp:165-195, 250-258
    L = oracle.lib()
    key = oracle.key_from_seed(21)
    s = oracle.EnvState()
    obs = np.zeros(4)
    pd = oracle.env_spec("pendulum")
    L.eo_env_reset(C.byref(pd), key, C.byref(s), oracle.ptr(obs))
    assert -math.pi <= s.phys[0] < math.pi and -1 <= s.phys[1] < 1
    assert obs[0] == math.cos(s.phys[0]) and obs[1] == math.sin(s.phys[0])
    assert s.rng.t() == oracle.fold_in(key, 1).t()
    rc = step(oracle, pd, (0.0, 0.0), float("nan"))[0]
    assert rc == 3 and "non-finite action" in L.eo_last_error().decode()
    rc = step(oracle, pd, (float("inf"), 0.0), 0.0)[0]
    assert rc == 3


def test_pendulum_speed_clamp(oracle):
    # proj/tests/test_env.cpp:91-100
    spec = oracle.env_spec("pendulum")
    phys = (math.pi / 2, 7.9)
    for _ in range(50):
        _, s, *_ = step(oracle, spec, phys, 2.0)
        phys = (s.phys[0], s.phys[1])
        assert abs(phys[1]) <= 8.0


def test_param_counts(oracle):
    # proj/tests/test_net.cpp:68-99 and SURVEY.md §8 param counts
    s = oracle.mlp_spec(4, [64, 64], 2, oracle.EO_HEAD_LINEAR)
    assert oracle.param_count(s) == 4610
    s.layer_norm = 1
    assert oracle.param_count(s) == 4866
    s.head = oracle.EO_HEAD_GAUSSIAN
    assert oracle.param_count(s) == 4868
    pd = oracle.env_spec("pendulum")
    for hidden, d in (([64, 64], 4481), ([256, 256], 67073), ([97, 97], 9992),
                      ([1024, 1024], 1054721)):
        assert oracle.param_count(oracle.policy_net_spec(pd, hidden)) == d
    # empty hidden throws in the reference (proj/src/net.cpp:27; test_net.cpp:254-261)
    assert oracle.param_count(oracle.policy_net_spec(pd, [])) == -1
    # ...and is the labelled linear-policy extension when allowed
    assert oracle.param_count(oracle.policy_net_spec(pd, [], allow_linear=True)) == 4


def test_init_params_glorot(oracle):
    # proj/tests/test_net.cpp:101-123
    s = oracle.mlp_spec(3, [8, 5], 2, oracle.EO_HEAD_GAUSSIAN, 2.0, layer_norm=True)
    p = oracle.init_params(s, oracle.key_from_seed(2))
    w0 = p[:24]
    assert np.abs(w0).max() <= math.sqrt(6 / 11) and np.abs(w0).max() > 0
    assert np.all(p[24:32] == 0.0) and np.all(p[32:40] == 1.0) and np.all(p[40:48] == 0.0)
    assert np.array_equal(p, oracle.init_params(s, oracle.key_from_seed(2)))
    assert not np.array_equal(p, oracle.init_params(s, oracle.key_from_seed(3)))


def test_forward_heads(oracle):
    # proj/tests/test_net.cpp:125-154
    s = oracle.mlp_spec(3, [8, 5], 2, oracle.EO_HEAD_LINEAR, 2.0)
    p = oracle.init_params(s, oracle.key_from_seed(5))
    x = oracle.gaussian_matrix(oracle.key_from_seed(6), 4, 3)
    lin = np.array([oracle.forward(s, p, r) for r in x])
    s.head = oracle.EO_HEAD_TANH
    th = np.array([oracle.forward(s, p, r) for r in x])
    assert np.all(np.abs(th) <= 2.0)
    assert np.allclose(th, 2.0 * np.tanh(lin), rtol=1e-15, atol=0)
    # numpy restatement of the same layer math (column-major W)
    W0 = p[:24].reshape(3, 8).T
    b0 = p[24:32]
    W1 = p[32:72].reshape(8, 5).T
    b1 = p[72:77]
    W2 = p[77:87].reshape(5, 2).T
    b2 = p[87:89]
    for r, out in zip(x, lin):
        h = np.maximum(W0 @ r + b0, 0)
        h = np.maximum(W1 @ h + b1, 0)
        assert np.allclose(W2 @ h + b2, out, rtol=1e-13, atol=1e-15)


def test_centered_ranks(oracle):
    # proj/tests/test_ec.cpp:23-42
    s = oracle.centered_ranks([3.0, 1.0, 2.0])
    assert list(s) == [0.5, -0.5, 0.0]
    assert list(oracle.centered_ranks([7.0, 7.0])) == [-0.5, 0.5]
    assert list(oracle.centered_ranks([5.0])) == [0.0]
    assert list(oracle.rank_desc([1.0, 9.0, 9.0, 3.0, -2.0])) == [1, 2, 3, 0, 4]


def openes_state(oracle, mean, **cfg):
    c = oracle.lib().eo_openes_default()
    for k, v in cfg.items():
        setattr(c, k, v)
    st = oracle.OpenEsState()
    mean = np.ascontiguousarray(mean, np.float64)
    oracle.check(oracle.lib().eo_openes_init(C.byref(st), C.byref(c), oracle.ptr(mean), len(mean),
                                             oracle.key_from_seed(70)))
    return st


def test_openes_ask_mirrored(oracle):
    # proj/tests/test_ec.cpp:46-67
    L = oracle.lib()
    mean = np.array([1.0, -2.0, 0.5])
    st = openes_state(oracle, mean, mirrored=1)
    st.sigma = 0.1
    cand = np.empty((8, 3))
    eps = np.empty((8, 3))
    oracle.check(L.eo_openes_ask(C.byref(st), oracle.key_from_seed(71), 8, oracle.ptr(cand),
                                 oracle.ptr(eps)))
    assert np.array_equal(eps[4:], -eps[:4])
    assert np.array_equal(eps[:4], oracle.gaussian_matrix(oracle.key_from_seed(71), 4, 3))
    assert np.abs(cand - (mean + 0.1 * eps)).max() < 1e-15
    assert L.eo_openes_ask(C.byref(st), oracle.key_from_seed(72), 7, oracle.ptr(cand),
                           oracle.ptr(eps)) == 1


def test_openes_tell_rank_shaped_adam(oracle):
    # proj/tests/test_ec.cpp:69-89
    L = oracle.lib()
    st = openes_state(oracle, np.zeros(2), lr=0.1, weight_decay=0.0)
    st.sigma = 0.5
    eps = np.array([[1, 0], [0, 1], [-1, 0], [0, -1]], np.float64)
    fit = np.array([4.0, 3.0, 2.0, 1.0])
    oracle.check(L.eo_openes_tell(C.byref(st), oracle.ptr(eps), oracle.ptr(fit), 4))
    g = (0.5 + 1.0 / 6.0) / (4.0 * 0.5)
    expect = 0.1 * g / (g + 1e-8)
    assert approx(st.mean[0], expect, 1e-12) and approx(st.mean[1], expect, 1e-12)
    assert st.t == 1


def test_openes_weight_decay_decoupled(oracle):
    # proj/tests/test_ec.cpp:91-108
    L = oracle.lib()
    st = openes_state(oracle, np.array([2.0]), lr=0.5, weight_decay=0.1)
    eps = np.array([[1.0], [-1.0]])
    fit = np.array([1.0, 1.0])
    oracle.check(L.eo_openes_tell(C.byref(st), oracle.ptr(eps), oracle.ptr(fit), 2))
    g = (-0.5 + (-1.0) * 0.5) / (2.0 * st.sigma)
    after = 2.0 + 0.5 * g / (abs(g) + 1e-8)
    assert approx(st.mean[0], after * (1.0 - 0.5 * 0.1), 1e-10)


def test_openes_noise_table(oracle):
    # proj/tests/test_ec.cpp:110-133
    L = oracle.lib()
    st = openes_state(oracle, np.zeros(5), noise_table=1, noise_table_size=4096, mirrored=1)
    st2 = openes_state(oracle, np.zeros(5), noise_table=1, noise_table_size=4096, mirrored=1)
    # table seed derives from the init key (key_from_seed(70) in the helper)
    table = np.ctypeslib.as_array(st.table, shape=(4096,))
    ak = oracle.key_from_seed(76)
    cand = np.empty((6, 5))
    eps = np.empty((6, 5))
    oracle.check(L.eo_openes_ask(C.byref(st), ak, 6, oracle.ptr(cand), oracle.ptr(eps)))
    offs = oracle.stream(ak)
    for i in range(3):
        off = L.eo_randint(C.byref(offs), 4096 - 5 + 1)
        assert np.array_equal(eps[i], table[off:off + 5])
        assert np.array_equal(eps[3 + i], -eps[i])
    assert np.array_equal(table, np.ctypeslib.as_array(st2.table, shape=(4096,)))


def test_ars_ask_interleaved(oracle):
    # proj/tests/test_ec.cpp:137-155
    L = oracle.lib()
    mean = np.array([1.0, 2.0, 3.0, 4.0])
    deltas = np.empty((3, 4))
    cand = np.empty((6, 4))
    oracle.check(L.eo_ars_ask(oracle.ptr(mean), 4, 0.25, oracle.key_from_seed(77), 6,
                              oracle.ptr(deltas), oracle.ptr(cand)))
    assert np.array_equal(deltas, oracle.gaussian_matrix(oracle.key_from_seed(77), 3, 4))
    for k in range(3):
        assert np.abs(cand[2 * k] - (mean + 0.25 * deltas[k])).max() < 1e-15
        assert np.abs(cand[2 * k + 1] - (mean - 0.25 * deltas[k])).max() < 1e-15
    assert L.eo_ars_ask(oracle.ptr(mean), 4, 0.25, oracle.key_from_seed(78), 5,
                        oracle.ptr(deltas), oracle.ptr(cand)) == 1


def test_ars_tell_elite_update_and_skip(oracle):
    # proj/tests/test_ec.cpp:157-186
    L = oracle.lib()
    cfg = L.eo_ars_default()
    cfg.elites = 1
    cfg.lr = 0.02
    mean = np.zeros(3)
    deltas = np.zeros((2, 3))
    deltas[0, 0] = 1.0
    deltas[1, 1] = 1.0
    rp = np.array([2.0, 0.0])
    rm = np.array([0.0, 0.0])
    assert L.eo_ars_tell(oracle.ptr(mean), 3, C.byref(cfg), oracle.ptr(deltas), oracle.ptr(rp),
                         oracle.ptr(rm), 2) == 1
    assert approx(mean[0], 0.04, 1e-14) and mean[1] == 0.0 and mean[2] == 0.0
    cfg.elites = 2
    mean = np.ones(2)
    deltas = oracle.gaussian_matrix(oracle.key_from_seed(79), 2, 2)
    flat = np.full(2, 3.0)
    assert L.eo_ars_tell(oracle.ptr(mean), 2, C.byref(cfg), oracle.ptr(deltas),
                         oracle.ptr(flat), oracle.ptr(flat), 2) == 0
    assert np.array_equal(mean, np.ones(2))


def test_canonical_weights(oracle):
    # proj/tests/test_ec.cpp:190-199
    w = np.empty(2)
    oracle.lib().eo_canonical_es_weights(2, oracle.ptr(w))
    assert approx(w[0], 0.8041628599327295, 1e-12) and approx(w[1], 0.19583714006727054, 1e-12)


def cma_state(oracle, mean, pop, elites, sigma0, max_dim=4096):
    L = oracle.lib()
    cfg = L.eo_cma_default()
    cfg.pop, cfg.elites, cfg.sigma0, cfg.max_dim = pop, elites, sigma0, max_dim
    st = oracle.CmaState()
    mean = np.ascontiguousarray(mean, np.float64)
    rc = L.eo_cma_init(C.byref(st), C.byref(cfg), oracle.ptr(mean), len(mean))
    return rc, st


def test_cma_init_invariants(oracle):
    # proj/tests/test_ec.cpp:231-249
    rc, st = cma_state(oracle, np.zeros(6), 16, 8, 0.3)
    assert rc == 0 and st.sigma == 0.3
    C_ = np.ctypeslib.as_array(st.C, shape=(36,)).reshape(6, 6)
    assert np.array_equal(C_, np.eye(6))
    w = np.ctypeslib.as_array(st.weights, shape=(8,))
    assert approx(w.sum(), 1.0, 1e-12)
    assert approx(st.mueff, 1.0 / (w ** 2).sum(), 1e-12)
    assert approx(st.chi_n, math.sqrt(6.0) * (1 - 1 / 24 + 1 / (21 * 36)), 1e-12)
    rc, _ = cma_state(oracle, np.zeros(6), 16, 8, 0.3, max_dim=4)
    assert rc == 2  # length_error


def test_cma_ask_identity(oracle):
    # proj/tests/test_ec.cpp:251-261
    mean = np.linspace(1.0, 4.0, 4)
    _, st = cma_state(oracle, mean, 8, 4, 0.2)
    cand = np.empty((8, 4))
    oracle.check(oracle.lib().eo_cma_ask(C.byref(st), oracle.key_from_seed(81), 8,
                                         oracle.ptr(cand)))
    z = oracle.gaussian_matrix(oracle.key_from_seed(81), 8, 4)
    assert np.abs(cand - (0.2 * z + mean)).max() < 1e-14


def _cma_gen(oracle, st, key, pop, fitfn):
    L = oracle.lib()
    d = st.dim
    cand = np.empty((pop, d))
    oracle.check(L.eo_cma_ask(C.byref(st), key, pop, oracle.ptr(cand)))
    fit = np.ascontiguousarray([fitfn(c) for c in cand])
    oracle.check(L.eo_cma_tell(C.byref(st), oracle.ptr(cand), oracle.ptr(fit), pop))


def test_cma_symmetry_and_positive(oracle):
    # proj/tests/test_ec.cpp:263-280
    _, st = cma_state(oracle, np.zeros(5), 12, 6, 0.5)
    noise = oracle.gaussian_matrix(oracle.key_from_seed(82), 30, 12)
    for gen in range(30):
        k = oracle.fold_in(oracle.key_from_seed(83), gen)
        it = iter(noise[gen])
        _cma_gen(oracle, st, k, 12, lambda c: -(c @ c) + 0.01 * next(it))
        C_ = np.ctypeslib.as_array(st.C, shape=(25,)).reshape(5, 5)
        D = np.ctypeslib.as_array(st.D, shape=(5,))
        assert np.abs(C_ - C_.T).max() < 1e-12 and D.min() > 0 and math.isfinite(st.sigma)
    assert st.generation == 30


def test_cma_offset_sphere(oracle):
    # proj/tests/test_ec.cpp:282-298
    target = np.array([0.7, -0.3, 0.5, 0.1, -0.8, 0.25, -0.4, 0.6])
    _, st = cma_state(oracle, np.zeros(8), 16, 8, 0.3)
    root = oracle.key_from_seed(84)
    for gen in range(200):
        _cma_gen(oracle, st, oracle.fold_in(root, gen), 16, lambda c: -((c - target) @ (c - target)))
    mean = np.ctypeslib.as_array(st.mean, shape=(8,))
    assert np.linalg.norm(mean - target) < 1e-3


def test_sym_eig(oracle):
    rng = np.random.default_rng(3)
    A = rng.standard_normal((12, 12))
    A = A + A.T
    ev = np.empty(12)
    V = np.empty((12, 12))
    oracle.lib().eo_sym_eig(oracle.ptr(A), 12, oracle.ptr(ev), oracle.ptr(V))
    Vc = V.T  # stored column-major: V[col*n+row]
    assert np.allclose(ev, np.linalg.eigvalsh(A), atol=1e-12)
    assert np.allclose(Vc @ np.diag(ev) @ Vc.T, A, atol=1e-11)


def adam(oracle, p, g, m, v, t, **cfg):
    L = oracle.lib()
    c = L.eo_adam_default()
    for k, val in cfg.items():
        setattr(c, k, val)
    tt = C.c_int64(t)
    L.eo_adam_step(oracle.ptr(p), oracle.ptr(g), oracle.ptr(m), oracle.ptr(v), C.byref(tt),
                   C.c_int64(len(p)), C.byref(c))
    return tt.value


def test_adam_kats(oracle):
    # proj/tests/test_optim.cpp:9-68
    p = np.array([1.0, -2.0, 0.5])
    g = np.array([100.0, -0.001, 4.0])
    m, v = np.zeros(3), np.zeros(3)
    assert adam(oracle, p, g, m, v, 0, lr=0.1) == 1
    assert approx(p[0], 1.0 - 0.1 * (100.0 / (100.0 + 1e-8)), 1e-12)
    assert approx(p[1], -2.0 + 0.1 * (0.001 / (0.001 + 1e-8)), 1e-12)
    p = np.array([0.3, -0.7])
    q = p.copy()
    m, v = np.zeros(2), np.zeros(2)
    mm, vv = np.zeros(2), np.zeros(2)
    t = 0
    for g in (np.array([0.5, -1.5]), np.array([-0.25, 2.0])):
        t += 1
        mm = 0.9 * mm + 0.1 * g
        vv = 0.999 * vv + 0.001 * g * g
        q -= 0.01 * (mm / (1 - 0.9 ** t)) / (np.sqrt(vv / (1 - 0.999 ** t)) + 1e-8)
        adam(oracle, p, g, m, v, t - 1, lr=0.01)
    assert np.abs(p - q).max() < 1e-15
    p = np.array([2.0])
    m, v = np.zeros(1), np.zeros(1)
    adam(oracle, p, np.zeros(1), m, v, 0, lr=0.5, weight_decay=0.1)
    assert approx(p[0], 1.9, 1e-12) and m[0] == 0.0 and v[0] == 0.0


def welford(oracle, rows):
    w = oracle.Welford()
    L = oracle.lib()
    for r in rows:
        r = np.ascontiguousarray(r, np.float64)
        L.eo_welford_add(C.byref(w), oracle.ptr(r), len(r))
    return w


def test_welford_and_merge(oracle):
    # proj/tests/test_obs_norm.cpp:20-62
    rows = 5.0 + 2.5 * oracle.gaussian_matrix(oracle.key_from_seed(1), 997, 3)
    w = welford(oracle, rows)
    assert w.count == 997.0
    assert np.abs(np.array(w.mean[:3]) - rows.mean(0)).max() < 1e-8
    assert np.abs(np.array(w.m2[:3]) / w.count - rows.var(0)).max() < 1e-8
    a = -1.0 + 0.5 * oracle.gaussian_matrix(oracle.key_from_seed(2), 300, 2)
    b = 8.0 + 3.0 * oracle.gaussian_matrix(oracle.key_from_seed(3), 17, 2)
    whole = welford(oracle, np.vstack([a, b]))
    wa, wb = welford(oracle, a), welford(oracle, b)
    oracle.lib().eo_welford_merge(C.byref(wa), C.byref(wb))
    assert wa.count == whole.count
    assert np.abs(np.array(wa.mean[:2]) - np.array(whole.mean[:2])).max() < 1e-10
    assert np.abs(np.array(wa.m2[:2]) / wa.count - np.array(whole.m2[:2]) / whole.count).max() < 1e-8


def test_normalize_and_rs(oracle):
    # proj/tests/test_obs_norm.cpp:64-122
    L = oracle.lib()
    rows = 3.0 + 4.0 * oracle.gaussian_matrix(oracle.key_from_seed(4), 5000, 3)
    w = welford(oracle, rows)
    st = L.eo_obs_norm_from_stats(oracle.EO_NORM_VBN, C.byref(w))
    out = np.empty(3)
    normed = []
    for r in rows:
        r = np.ascontiguousarray(r)
        L.eo_normalize(C.byref(st), oracle.ptr(r), 3, oracle.ptr(out))
        normed.append(out.copy())
    normed = np.array(normed)
    assert np.abs(normed.mean(0)).max() < 1e-6 and np.abs(normed.std(0) - 1).max() < 1e-6
    same = np.array([4.0, -1.0])
    w = welford(oracle, [same] * 10)
    st = L.eo_obs_norm_from_stats(oracle.EO_NORM_VBN, C.byref(w))
    out = np.empty(2)
    L.eo_normalize(C.byref(st), oracle.ptr(same), 2, oracle.ptr(out))
    assert np.all(out == 0.0)
    allr = -2.0 + 1.7 * oracle.gaussian_matrix(oracle.key_from_seed(5), 600, 4)
    rs = L.eo_obs_norm_running_stats(4)
    for part in (allr[:100], allr[100:350], allr[350:]):
        b = welford(oracle, part)
        L.eo_rs_update(C.byref(rs), C.byref(b))
    ref = welford(oracle, allr)
    assert rs.count == 600.0
    assert np.abs(np.array(rs.mean) - np.array(ref.mean)).max() < 1e-10
    assert np.abs(np.array(rs.var) - np.array(ref.m2) / 600).max() < 1e-8
