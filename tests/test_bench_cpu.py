"""bench.py's contract pieces that need no GPU: both arms print the same
workload `config` object (the driver compares the arms' configs), and the
parameter count it names is the one the reference layout gives."""
import json

import pytest


def test_reference_arm_prints_the_gpu_arms_workload_config(monkeypatch, capsys, oracle):
    import bench

    # a stand-in for the timed oracle sample (the real one takes seconds per step)
    monkeypatch.setattr(bench, "cpu_sample_run", lambda cfgd, steps, warmup, sample_pop=None:
                        (1000, [0.5] * steps, 4, sample_pop or cfgd["pop"]))

    class A:
        gpus, steps, warmup = 1, 3, 3

    for name in sorted(bench.CONFIGS):
        assert bench.run_reference_arm(A, bench.CONFIGS[name], name) == 0
        line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
        assert line["impl"] == "reference"
        assert line["config"] == bench.workload_config(name)
        assert line["steps"] == 3 and line["e2e"]["h2d_bytes_per_step"] == 0
        cfgd = bench.CONFIGS[name]
        spec = oracle.policy_net_spec(oracle.env_spec(cfgd["env"]), list(cfgd["hidden"]),
                                      allow_linear=cfgd.get("allow_linear", False))
        assert line["config"]["params"] == oracle.param_count(spec)


@pytest.mark.parametrize("name", ["1", "2", "3", "4"])
def test_workload_config_is_workload_only(name):
    import bench

    c = bench.workload_config(name)
    for k in ("parallelism", "policy_precision", "policy_team", "pop_sampled"):
        assert k not in c
    assert c["workload"] == bench.CONFIGS[name]["desc"]
