"""CPU-side checks of the drop-in boundary: the C-ABI library exists, loads,
exports every symbol include/evorl_b200.h declares, and refuses to compute
without a GPU (no silent CPU fallback)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "evorl_b200.h")).read()
    return sorted(set(re.findall(r"\b(evorl_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2501_15129_b200 import _lib
    L = _lib.load()
    declared = header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(L, name), name
    assert set(declared) == set(_lib.EXPORTS)
    assert L.evorl_abi_version() == 1


def test_sm100a_cubin_present():
    import subprocess
    so = os.path.join(ROOT, "paper_2501_15129_b200", "libevorl_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_config_matches_reference_registry():
    # proj/src/config.cpp:23-70 defaults
    from paper_2501_15129_b200 import _lib
    c = _lib.EsConfigC()
    _lib.load().evorl_es_default_config(C.byref(c))
    assert (c.pop, c.fitness_episodes, c.vbn_samples) == (128, 1, 10000)
    assert (c.openes_sigma, c.openes_lr, c.openes_weight_decay) == (0.02, 0.01, 0.005)
    assert (c.ars_sigma, c.ars_lr, c.ars_elites) == (0.03, 0.02, 16)
    assert (c.cmaes_sigma0, c.cmaes_elites, c.cmaes_max_dim) == (0.1, 64, 4096)
    assert list(c.hidden[:c.n_hidden]) == [64, 64]


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="GPU present")
def test_no_cpu_fallback_without_gpu():
    import paper_2501_15129_b200 as evb
    with pytest.raises(evb.DeviceError, match="no CPU fallback"):
        evb.gaussian_matrix((1, 2), 2, 2)
    with pytest.raises(evb.DeviceError):
        evb.EsWorkflow(evb.EsConfig())
