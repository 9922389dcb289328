"""CMA-ES free functions on the device (evorl_cma_create / ask / tell: the
reference's CmaState::init / cmaes_ask / cmaes_tell, proj/src/ec.cpp:191-288)
against the oracle's eo_cma_init / eo_cma_ask / eo_cma_tell, and the
reference's own CMA unit tests (proj/tests/test_ec.cpp:231-297) run through
the device path.  Dimensions satisfy d <= mu + 1 so the eigenbasis is unique
and eigenvector-dependent quantities compare directly."""
import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def evb():
    import paper_2501_15129_b200 as m
    return m


def _oracle_state(oracle, mean, pop, elites, sigma0):
    L = oracle.lib()
    cfg = L.eo_cma_default()
    cfg.pop, cfg.elites, cfg.sigma0, cfg.max_dim = pop, elites, sigma0, 4096
    st = oracle.CmaState()
    mean = np.ascontiguousarray(mean, np.float64)
    assert L.eo_cma_init(C.byref(st), C.byref(cfg), oracle.ptr(mean), len(mean)) == 0
    return st


def _oracle_view(st):
    d = st.dim
    arr = lambda p, n: np.ctypeslib.as_array(p, shape=(n,)).copy()
    return dict(mean=arr(st.mean, d), C=arr(st.C, d * d).reshape(d, d), B=arr(st.B, d * d).reshape(d, d).T,
                D=arr(st.D, d), ps=arr(st.ps, d), pc=arr(st.pc, d), sigma=st.sigma, generation=st.generation)


def test_init_and_identity_ask(evb, oracle):
    # proj/tests/test_ec.cpp:231-261
    cma = evb.CmaEs(4, 8, 4, 0.2, mean0=np.linspace(1.0, 4.0, 4))
    s = cma.state()
    assert np.array_equal(s["C"], np.eye(4)) and np.array_equal(s["B"], np.eye(4))
    assert np.array_equal(s["D"], np.ones(4)) and s["sigma"] == 0.2 and s["generation"] == 0
    cand = cma.ask(oracle.key_from_seed(81))
    z = oracle.gaussian_matrix(oracle.key_from_seed(81), 8, 4)
    assert np.abs(cand - (0.2 * z + np.linspace(1.0, 4.0, 4))).max() < 1e-14
    with pytest.raises(evb.LengthError):
        evb.CmaEs(6, 16, 8, 0.3, max_dim=4)
    with pytest.raises(evb.InvalidArgument):
        evb.CmaEs(0, 16, 8, 0.3)


@pytest.mark.parametrize("d,pop,elites", [(5, 12, 6), (8, 16, 8), (31, 64, 32)])
def test_lockstep_matches_oracle(evb, oracle, d, pop, elites):
    """Each generation: both sides ask with the same key (candidates compared),
    then both tell the ORACLE's candidates with the same fitness, so the state
    comparison is per-step and free of closed-loop drift."""
    L = oracle.lib()
    st = _oracle_state(oracle, np.zeros(d), pop, elites, 0.3)
    cma = evb.CmaEs(d, pop, elites, 0.3)
    target = np.sin(np.arange(d) + 1.0)
    root = oracle.key_from_seed(90 + d)
    for gen in range(25):
        k = oracle.fold_in(root, gen)
        co = np.empty((pop, d))
        oracle.check(L.eo_cma_ask(C.byref(st), k, pop, oracle.ptr(co)))
        cg = cma.ask(k)
        assert np.allclose(cg, co, rtol=1e-9, atol=1e-11 * max(1.0, np.abs(co).max())), gen
        fit = np.ascontiguousarray(-((co - target) ** 2).sum(1))
        oracle.check(L.eo_cma_tell(C.byref(st), oracle.ptr(co), oracle.ptr(fit), pop))
        cma.tell(co, fit)
        so, sg = _oracle_view(st), cma.state()
        assert sg["generation"] == so["generation"] == gen + 1
        assert sg["sigma"] == pytest.approx(so["sigma"], rel=1e-10)
        assert np.allclose(cma.mean(), so["mean"], rtol=1e-10, atol=1e-13), gen
        for key in ("ps", "pc"):
            assert np.allclose(sg[key], so[key], rtol=1e-8, atol=1e-11), (gen, key)
        assert np.allclose(sg["C"], so["C"], rtol=1e-9, atol=1e-13 * np.abs(so["C"]).max()), gen
        assert np.allclose(sg["D"], so["D"], rtol=1e-8), gen
        assert np.allclose(sg["B"], so["B"], atol=1e-6), gen


def test_symmetry_and_positive(evb, oracle):
    # proj/tests/test_ec.cpp:263-280
    cma = evb.CmaEs(5, 12, 6, 0.5)
    noise = oracle.gaussian_matrix(oracle.key_from_seed(82), 30, 12)
    for gen in range(30):
        cand = cma.ask(oracle.fold_in(oracle.key_from_seed(83), gen))
        cma.tell(cand, -(cand * cand).sum(1) + 0.01 * noise[gen])
        s = cma.state()
        assert np.abs(s["C"] - s["C"].T).max() < 1e-12 and s["D"].min() > 0 and math.isfinite(s["sigma"])
    assert cma.state()["generation"] == 30


def test_solves_offset_sphere(evb, oracle):
    # proj/tests/test_ec.cpp:282-297
    target = np.array([0.7, -0.3, 0.5, 0.1, -0.8, 0.25, -0.4, 0.6])
    cma = evb.CmaEs(8, 16, 8, 0.3)
    root = oracle.key_from_seed(84)
    for gen in range(200):
        cand = cma.ask(oracle.fold_in(root, gen))
        cma.tell(cand, -((cand - target) ** 2).sum(1))
    assert np.linalg.norm(cma.mean() - target) < 1e-3


def test_cma_handle_refuses_workflow_calls(evb):
    cma = evb.CmaEs(4, 8, 4, 0.2)
    L = evb._lib.load()
    assert L.evorl_es_init(cma.h, 1, 2) == 1
    assert "cma-only" in L.evorl_last_error().decode()
    with pytest.raises(ValueError):
        cma.tell(np.zeros((7, 4)), np.zeros(7))
