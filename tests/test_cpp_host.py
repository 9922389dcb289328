"""The C++ host side (include/evorl_b200.hpp + examples/es_generation.cpp):
the reference's names and exception types over the C ABI.

CPU: the header compiles (every wrapper instantiated), the example builds and
links against the in-tree library, and without a GPU it fails loudly with the
mapped DeviceError (no CPU fallback).  GPU: the C++ host's generations are
bit-identical to the Python host's through the same ABI."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "es_generation")

TOUR = r'''
#include "evorl_b200.hpp"
int main() {
  namespace eb = evorl_b200;
  try {
    evorl_es_config c = eb::default_config();
    eb::EsWorkflow wf(c);
    wf.init({1, 2});
    eb::StepMetrics m = wf.step();
    eb::EvalReport r = wf.evaluate(4, {3, 4});
    std::vector<double> mean = wf.mean();
    wf.set_mean(mean);
    std::int64_t a, b, d;
    wf.counters(&a, &b, &d);
    wf.save("/tmp/x.ckpt");
    wf.load("/tmp/x.ckpt");
    (void)m; (void)r; (void)wf.fitness(c.pop);
    std::vector<double> f = {3.0, 1.0, 2.0};
    (void)eb::centered_ranks(f);
    (void)eb::rank_desc(f);
    (void)eb::gaussian_matrix({1, 2}, 2, 3);
    evorl_env_desc env{EVORL_ENV_PENDULUM, 1, 10};
    evorl_mlp_desc net{};
    (void)eb::batched_rollout(env, net, nullptr, f, 1, 1, 1, {5, 6});
    eb::CmaEs cma(4, 8, 4, 0.2);
    std::vector<double> cand = cma.ask(eb::fold_in(eb::key_from_seed(1), 2));
    cma.tell(cand, std::vector<double>(8, 0.0));
    cma.set_mean(cma.mean());
    (void)cma.sigma();
  } catch (const eb::DeviceError&) { return 3; }
  catch (const std::exception&) { return 4; }
  return 0;
}
'''


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)


def test_header_compiles_and_maps_errors(tmp_path):
    src = tmp_path / "tour.cpp"
    src.write_text(TOUR)
    exe = tmp_path / "tour"
    lib = os.path.join(ROOT, "paper_2501_15129_b200")
    subprocess.run(["g++", "-std=c++17", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                    str(src), "-L", lib, "-levorl_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    rc = subprocess.run([str(exe)]).returncode
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert rc == 3  # DeviceError: the B200 path has no CPU fallback


def test_example_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    _build()
    r = subprocess.run([EXE], capture_output=True, text=True)
    assert r.returncode == 2 and "no CUDA device available" in r.stderr


@pytest.mark.gpu
def test_cpp_host_matches_python_host():
    sys.path.insert(0, ROOT)
    import paper_2501_15129_b200 as evb
    _build()
    r = subprocess.run([EXE, "openes", "32", "3", "16", "16", "2", "f64"], capture_output=True, text=True,
                       check=True)
    lines = r.stdout.strip().splitlines()
    g = evb.EsWorkflow(evb.EsConfig(algo="openes", env="pendulum", fixed_horizon=True, max_episode_steps=100,
                                    pop=32, hidden=(16, 16), fitness_episodes=2, vbn_samples=500))
    g.init((0x1234, 0x5678))
    for i in range(3):
        m = g.step()
        want = f"gen {i} fitness_mean {float.hex(m['fitness/mean'])}"
        got = lines[i].split(" fitness_max")[0]
        assert float.fromhex(got.split()[-1]) == m["fitness/mean"], (got, want)
    mr, sd = g.evaluate(16, (7, 8))
    ev = lines[3].split()
    assert float.fromhex(ev[2]) == mr and float.fromhex(ev[4]) == sd
    assert lines[4] == "counters %d %d %d" % g.counters()


@pytest.mark.gpu
def test_cpp_cma_free_functions_match_python():
    """proj/tests/test_ec.cpp:282-297 through the C++ CmaEs wrapper; the same
    loop through the Python binding gives the bit-identical final state."""
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_ffi as oracle
    import paper_2501_15129_b200 as evb
    _build()
    r = subprocess.run([EXE, "cma-sphere"], capture_output=True, text=True, check=True)
    _, _, dist, _, sigma = r.stdout.split()
    target = np.array([0.7, -0.3, 0.5, 0.1, -0.8, 0.25, -0.4, 0.6])
    cma = evb.CmaEs(8, 16, 8, 0.3)
    for g in range(200):
        k = oracle.fold_in(oracle.key_from_seed(84), g)
        cand = cma.ask((k.hi, k.lo))
        cma.tell(cand, -((cand - target) ** 2).sum(1))
    d = cma.mean() - target
    assert float.fromhex(dist) == np.sqrt(np.sum(d * d)) or abs(float.fromhex(dist) - np.linalg.norm(d)) < 1e-15
    assert float.fromhex(dist) < 1e-3
    assert float.fromhex(sigma) == cma.state()["sigma"]
