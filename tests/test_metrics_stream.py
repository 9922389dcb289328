"""The JSONL metrics stream and learn() loop (
proj/src/metrics.cpp:12-67, proj/src/workflow.cpp:46-68).

CPU: the nlohmann-style serialiser (Python and the C++ header) produces the
same bytes, round-trips every double exactly, and places digits the way
nlohmann's format_buffer does.  GPU: learn() through the Python host and the
C++ host writes byte-identical step / eval records, and the records carry the
workflow's counters, metrics and the eval key's evaluation."""
import json
import os
import struct
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2501_15129_b200.learn import Budget, LearnOptions, MetricsWriter, dump_json  # noqa: E402

# (value, nlohmann's dump) -- format_buffer cases: integral .0, plain, 0.000ddd, d.ddde+XX
KNOWN = [(1.0, "1.0"), (0.1, "0.1"), (-2.5, "-2.5"), (1e-05, "1e-05"), (0.0001, "0.0001"),
         (0.0001234, "0.0001234"), (1e15, "1e+15"), (123456789012345.0, "123456789012345.0"),
         (1234567890123456.0, "1.234567890123456e+15"), (1e300, "1e+300"), (5e-324, "5e-324"),
         (0.0, "0.0"), (-0.0, "-0.0"), (float("nan"), "null"), (float("inf"), "null"),
         (-1219.3551025390625, "-1219.3551025390625"), (2.0 ** 60, "1.152921504606847e+18")]


def _random_doubles(n=3000):
    rng = np.random.default_rng(5)
    bits = rng.integers(0, 2 ** 63, n, dtype=np.int64).view(np.float64)
    vals = [float(x) for x in bits if np.isfinite(x)]
    vals += [float(x) for x in rng.standard_normal(500) * 10.0 ** rng.integers(-8, 18, 500)]
    return vals


def test_known_dumps():
    for v, want in KNOWN:
        assert dump_json(v) == want, v
    assert dump_json({"b": 1, "a": {"z": "q\"\n\x01", "y": True}, "A": 2.0}) == \
        '{"A":2.0,"a":{"y":true,"z":"q\\"\\n\\u0001"},"b":1}'


def test_roundtrip():
    for v in _random_doubles():
        s = dump_json(v)
        assert struct.pack("<d", float(s)) == struct.pack("<d", v), (v, s)


def test_cpp_header_serialiser_matches(tmp_path):
    vals = [v for v, _ in KNOWN] + _random_doubles(2000)
    src = tmp_path / "j.cpp"
    src.write_text(r'''
#include "evorl_b200.hpp"
#include <cstring>
int main() {
  std::uint64_t b;
  while (std::fread(&b, 8, 1, stdin) == 1) {
    double x;
    std::memcpy(&x, &b, 8);
    std::printf("%s\n", evorl_b200::detail::json_double(x).c_str());
  }
  std::printf("%s\n", evorl_b200::detail::json_object({{"b", "1"}, {"a", evorl_b200::detail::json_string("q\"\n\x01")}}).c_str());
}''')
    exe = tmp_path / "j"
    lib = os.path.join(ROOT, "paper_2501_15129_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"), str(src), "-L", lib,
                    "-levorl_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], input=np.array(vals, np.float64).tobytes(), capture_output=True,
                         check=True).stdout.decode().splitlines()
    assert out[:-1] == [dump_json(v) for v in vals]
    assert out[-1] == '{"a":"q\\"\\n\\u0001","b":1}'


def test_writer_records(tmp_path):
    m, t = str(tmp_path / "metrics.jsonl"), str(tmp_path / "timings.log")
    w = MetricsWriter(m, t)
    w.write_header("es", {"seed": "0", "ec.pop": "128", "workflow": "es"})
    w.write_step(1, 25600, 128, 0, {"fitness/mean": -1200.5, "es/sigma": 0.02, "es/update_skipped": 0})
    w.write_eval(10, 256000, 1280, 0, -150.25, 3.0, 128)
    w.write_timing(1, 12.3456789)
    w.close()
    lines = open(m).read().splitlines()
    assert lines[0] == '{"config":{"ec.pop":"128","seed":"0","workflow":"es"},"type":"header","workflow":"es"}'
    assert lines[1] == ('{"env_steps":25600,"episodes":128,"es/sigma":0.02,"es/update_skipped":0.0,'
                        '"fitness/mean":-1200.5,"iteration":1,"rl_updates":0,"type":"step"}')
    assert lines[2] == ('{"env_steps":256000,"episodes":1280,"eval/episode_return_mean":-150.25,'
                        '"eval/episode_return_std":3.0,"eval/episodes":128,"iteration":10,"rl_updates":0,'
                        '"type":"eval"}')
    assert open(t).read() == "1\t12.3457\n"
    with pytest.raises(RuntimeError, match="cannot open metrics file"):
        MetricsWriter(str(tmp_path / "nodir" / "m.jsonl"), t)


def test_budget():
    b = Budget(iterations=3, episodes=0, env_steps=100)
    assert not b.reached(2, 99, 0) and b.reached(3, 0, 0) and b.reached(0, 100, 0)
    assert not Budget().reached(10 ** 9, 10 ** 12, 10 ** 9)


@pytest.mark.gpu
def test_learn_python_and_cpp_hosts_write_identical_records(tmp_path):
    import paper_2501_15129_b200 as evb
    from paper_2501_15129_b200.learn import eval_key, key_from_seed, learn
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    cdir = tmp_path / "cpp"
    cdir.mkdir()
    subprocess.run([os.path.join(ROOT, "examples", "es_generation"), "learn", str(cdir)], check=True)
    cfg = evb.EsConfig(algo="openes", env="pendulum", fixed_horizon=True, max_episode_steps=60, pop=32,
                       hidden=(16, 16), vbn_samples=300)
    root = key_from_seed(3)
    wf = evb.EsWorkflow(cfg).init(root)
    pdir = tmp_path / "py"
    pdir.mkdir()
    mw = MetricsWriter(str(pdir / "metrics.jsonl"), str(pdir / "timings.log"))
    mw.write_header("es", {"workflow": "es", "seed": "3", "ec.pop": "32"})
    learn(wf, root, LearnOptions(Budget(iterations=5), eval_interval=2, eval_episodes=8,
                                 checkpoint_path=str(pdir / "checkpoint.bin")), mw)
    mw.close()
    py = open(pdir / "metrics.jsonl").read()
    assert py == open(cdir / "metrics.jsonl").read()
    assert open(pdir / "checkpoint.bin", "rb").read() == open(cdir / "checkpoint.bin", "rb").read()
    recs = [json.loads(x) for x in py.splitlines()]
    assert [r["type"] for r in recs] == ["header", "step", "step", "eval", "step", "step", "eval", "step"]
    assert [r["iteration"] for r in recs[1:]] == [1, 2, 2, 3, 4, 4, 5]
    assert recs[-1]["env_steps"] == 5 * 32 * 60 and recs[-1]["episodes"] == 5 * 32
    # the eval records are Workflow::evaluate at WorkflowState::eval_key
    h = evb.EsWorkflow(cfg).init(root)
    for _ in range(4):
        h.step()
    mr, sd = h.evaluate(8, eval_key(root, 4))
    assert recs[6]["eval/episode_return_mean"] == mr and recs[6]["eval/episode_return_std"] == sd
    assert len(open(pdir / "timings.log").read().splitlines()) == 5


def test_es_config_entries_use_registry_spelling():
    import paper_2501_15129_b200 as evb
    from paper_2501_15129_b200.learn import es_config_entries
    e = es_config_entries(evb.EsConfig(), seed=0)
    # registry defaults (proj/src/config.cpp:23-70)
    assert e["ec.openes.sigma"] == "0.02" and e["ec.cem.var_init"] == "1e-3" and e["ec.cem.noise_end"] == "1e-5"
    assert e["net.hidden"] == "64,64" and e["env.fixed_horizon"] == "false" and e["ec.openes.mirrored"] == "true"
    assert e["ec.openes.noise_table_size"] == "4194304" and e["workflow"] == "es" and e["seed"] == "0"


@pytest.mark.gpu
def test_learn_eval_keys_follow_the_loaded_state_rng(tmp_path):
    """Eval keys derive from WorkflowState::rng (proj/include/evorl/workflow.hpp:42):
    after load(), learn() evaluates at the checkpoint's key, and a caller key
    that differs from the state's is refused instead of silently used."""
    import paper_2501_15129_b200 as evb
    from paper_2501_15129_b200.learn import eval_key, key_from_seed, learn
    cfg = evb.EsConfig(algo="openes", env="pendulum", fixed_horizon=True, max_episode_steps=40, pop=16,
                       hidden=(8,), vbn_samples=200)
    root = key_from_seed(11)
    a = evb.EsWorkflow(cfg).init(root)
    a.step()
    a.save(str(tmp_path / "ck.bin"))
    b = evb.EsWorkflow(cfg).init(key_from_seed(12)).load(str(tmp_path / "ck.bin"))
    assert b.rng() == root
    with pytest.raises(ValueError):
        learn(b, key_from_seed(12), LearnOptions(Budget(iterations=2)), MetricsWriter(
            str(tmp_path / "m.jsonl"), str(tmp_path / "t.log")))
    mw = MetricsWriter(str(tmp_path / "m2.jsonl"), str(tmp_path / "t2.log"))
    learn(b, None, LearnOptions(Budget(iterations=2), eval_interval=2, eval_episodes=4), mw)
    mw.close()
    recs = [json.loads(x) for x in open(tmp_path / "m2.jsonl").read().splitlines()]
    ev = [r for r in recs if r["type"] == "eval"][0]
    a.step()
    mr, _ = a.evaluate(4, eval_key(root, 2))
    assert ev["eval/episode_return_mean"] == mr
