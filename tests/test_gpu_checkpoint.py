"""Checkpoint interop: EVORL1 files written / read by
EsWorkflow.save / load through the C ABI, against the reference's format
(proj/src/checkpoint.cpp), segment layout (proj/src/workflow_es.cpp:181-249)
and resume invariant (proj/tests/test_workflow.cpp:173-199)."""
import os

import numpy as np
import pytest

import ckpt_format as ck

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def evb():
    import paper_2501_15129_b200 as m
    return m


CFGS = {
    "openes": dict(algo="openes", env="pendulum", fixed_horizon=True, pop=32, hidden=(16, 16),
                   max_episode_steps=60, vbn_samples=300),
    "ars": dict(algo="ars", env="pendulum", fixed_horizon=True, pop=32, hidden=(8,), max_episode_steps=60),
    "ves": dict(algo="ves", env="pendulum", fixed_horizon=True, pop=16, hidden=(8,), max_episode_steps=40,
                vbn_samples=200),
    "cmaes": dict(algo="cmaes", env="pendulum", fixed_horizon=True, pop=16, hidden=(4,),
                  max_episode_steps=40, vbn_samples=200, cmaes_elites=8, cmaes_sigma0=0.2),
    "cem": dict(algo="cem", env="cartpole", pop=20, hidden=(8,), max_episode_steps=50),
}


@pytest.mark.parametrize("algo", sorted(CFGS))
def test_segments_match_reference_layout_and_state(evb, tmp_path, algo):
    g = evb.EsWorkflow(evb.EsConfig(**CFGS[algo])).init((21, 22))
    g.step()
    g.step()
    path = str(tmp_path / "a.ckpt")
    g.save(path)
    assert not os.path.exists(path + ".tmp")
    wid, segs = ck.read(path)
    assert wid == "es"
    assert [(n, t) for n, t, _ in segs] == ck.BASE + ck.EC[algo]
    v = {n: a for n, _, a in segs}
    it, steps, eps = g.counters()
    assert list(v["iteration"]) == [it] and list(v["env_steps"]) == [steps] and list(v["episodes"]) == [eps]
    assert [int(x) & (2**64 - 1) for x in v["rng"]] == [21, 22]
    assert list(v["rl_updates"]) == [0]
    on = g.obs_norm()
    assert v["obs_norm/mode"][0] == on.mode
    nd = 0 if on.mode == 0 else on.dim
    assert np.array_equal(v["obs_norm/mean"], np.array(list(on.mean)[:nd]))
    assert np.array_equal(v["obs_norm/var"], np.array(list(on.var)[:nd]))
    assert v["obs_norm/count"][0] == on.count
    assert np.array_equal(v["ec/mean"], g.mean())
    if algo == "openes":
        m, vv, t = g.adam()
        assert np.array_equal(v["ec/adam/m"], m) and np.array_equal(v["ec/adam/v"], vv)
        assert list(v["ec/adam/t"]) == [t] and list(v["ec/table_seed"]) == [0]
    if algo == "cmaes":
        st = g.cma_state()
        d = g.dim
        assert np.array_equal(v["ec/C"], st["C"].reshape(-1))
        # Eigen column-major: flat[j*d + p] = component p of eigenvector j
        assert np.array_equal(v["ec/B"].reshape(d, d).T, st["B"])
        assert list(v["ec/generation"]) == [st["generation"]]


@pytest.mark.parametrize("algo", sorted(CFGS))
def test_resume_equivalence(evb, tmp_path, algo):
    """save after generation 1, load into a fresh handle: generations 2-3 are
    bit-identical to the uninterrupted run (proj/tests/test_workflow.cpp:173-199)."""
    cfg = CFGS[algo]
    g = evb.EsWorkflow(evb.EsConfig(**cfg)).init((31, 32))
    g.step()
    path = str(tmp_path / "r.ckpt")
    g.save(path)
    g.step()
    g.step()
    h = evb.EsWorkflow(evb.EsConfig(**cfg)).load(path)
    h.step()
    h.step()
    assert np.array_equal(h.fitness(), g.fitness())
    assert np.array_equal(h.mean(), g.mean())
    assert h.counters() == g.counters()
    h.save(str(tmp_path / "h.ckpt"))
    g.save(str(tmp_path / "g.ckpt"))
    assert open(tmp_path / "h.ckpt", "rb").read() == open(tmp_path / "g.ckpt", "rb").read()


def test_loads_reference_written_checkpoint(evb, oracle, tmp_path):
    """A checkpoint of the oracle's state after 2 generations, written in the
    reference's layout, loads into the device workflow; the next generation
    matches the oracle's next generation (fp64 closed-loop tolerance)."""
    kw = dict(algo="openes", env="pendulum", fixed_horizon=True, pop=32, hidden=[16, 16],
              max_episode_steps=60, vbn_samples=300)
    o = oracle.OracleEs(oracle.es_config(workers=0, **kw))
    key = oracle.key_from_seed(41)
    o.init(key)
    o.step()
    o.step()
    it, steps, eps = o.counters()
    on = o.obs_norm()
    m, v, t = o.adam()
    path = str(tmp_path / "ref.ckpt")
    ck.write(path, "es", [
        ("iteration", "i64", it), ("rng", "i64", np.array([key.hi, key.lo], np.uint64).view(np.int64)),
        ("env_steps", "i64", steps), ("episodes", "i64", eps), ("rl_updates", "i64", 0),
        ("obs_norm/mode", "i64", on.mode), ("obs_norm/mean", "f64", list(on.mean)[:on.dim]),
        ("obs_norm/var", "f64", list(on.var)[:on.dim]), ("obs_norm/count", "f64", on.count),
        ("ec/mean", "f64", o.mean()), ("ec/sigma", "f64", 0.02), ("ec/adam/m", "f64", m),
        ("ec/adam/v", "f64", v), ("ec/adam/t", "i64", t), ("ec/table_seed", "i64", 0)])
    g = evb.EsWorkflow(evb.EsConfig(**{k: (tuple(x) if k == "hidden" else x) for k, x in kw.items()}))
    g.load(path)
    assert g.counters() == o.counters()
    o.step()
    g.step()
    assert np.allclose(g.fitness(), o.fitness(), rtol=1e-9, atol=1e-12)
    assert np.array_equal(np.argsort(g.fitness(), kind="stable"), np.argsort(o.fitness(), kind="stable"))
    assert np.allclose(g.mean(), o.mean(), rtol=1e-9, atol=1e-12)


def test_checkpoint_errors(evb, tmp_path):
    cfg = CFGS["openes"]
    g = evb.EsWorkflow(evb.EsConfig(**cfg)).init((1, 2))
    path = str(tmp_path / "e.ckpt")
    g.save(path)
    good = open(path, "rb").read()
    h = evb.EsWorkflow(evb.EsConfig(**cfg))

    def load_bytes(b, name):
        p = str(tmp_path / name)
        open(p, "wb").write(b)
        h.load(p)

    with pytest.raises(evb.CheckpointError, match="bad magic"):
        load_bytes(b"EVORL2" + good[6:], "m.ckpt")
    with pytest.raises(evb.CheckpointError, match="format version 7"):
        load_bytes(good[:6] + (7).to_bytes(4, "little") + good[10:], "v.ckpt")
    with pytest.raises(evb.CheckpointError, match="truncated file"):
        load_bytes(good[:-3], "t.ckpt")
    with pytest.raises(evb.CheckpointError, match="trailing bytes"):
        load_bytes(good + b"\0", "x.ckpt")
    with pytest.raises(evb.CheckpointError, match="cannot open checkpoint"):
        h.load(str(tmp_path / "missing.ckpt"))
    wid, segs = ck.read(path)
    ck.write(str(tmp_path / "w.ckpt"), "td3", segs)
    with pytest.raises(evb.CheckpointError, match="workflow 'td3', expected 'es'"):
        h.load(str(tmp_path / "w.ckpt"))
    short = [(n, t, a[:-1] if n == "ec/mean" else a) for n, t, a in segs]
    ck.write(str(tmp_path / "s.ckpt"), "es", short)
    with pytest.raises(evb.CheckpointError, match="segment 'ec/mean' has wrong size"):
        h.load(str(tmp_path / "s.ckpt"))
    miss = [(n, t, a) for n, t, a in segs if n != "ec/adam/t"]
    ck.write(str(tmp_path / "n.ckpt"), "es", miss)
    with pytest.raises(evb.CheckpointError, match="missing integer segment 'ec/adam/t'"):
        h.load(str(tmp_path / "n.ckpt"))


def test_noise_table_checkpoint_resume(evb, tmp_path):
    """ec/table_seed carries the table across save/load (openes_rebuild_table,
    proj/src/workflow_es.cpp:223-224): resumed generations are bit-identical."""
    cfg = dict(CFGS["openes"], openes_noise_table=True, openes_noise_table_size=1 << 16)
    g = evb.EsWorkflow(evb.EsConfig(**cfg)).init((51, 52))
    g.step()
    path = str(tmp_path / "t.ckpt")
    g.save(path)
    _, segs = ck.read(path)
    assert dict((n, a) for n, _, a in segs)["ec/table_seed"][0] != 0
    g.step()
    h = evb.EsWorkflow(evb.EsConfig(**cfg)).load(path)
    h.step()
    assert np.array_equal(h.fitness(), g.fitness())
    assert np.array_equal(h.mean(), g.mean())
