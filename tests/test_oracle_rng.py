"""Oracle RNG vs the reference's frozen KATs (proj/tests/test_rng.cpp) and vs
the reference's own rng.cpp compiled into oracle/_ref (bitwise)."""
import ctypes as C

import numpy as np
import pytest

FF = (1 << 64) - 1


def test_threefry_kats(oracle):
    # proj/tests/test_rng.cpp:15-29 (first block = Random123 KAT)
    assert oracle.threefry((0, 0), (0, 0)) == (0xC2B6E3A8C2C69865, 0x6F81ED42F350084D)
    assert oracle.threefry((FF, FF), (FF, FF)) == (0xE02CB7C4D95D277A, 0xD06633D0893B8B68)
    assert oracle.threefry((0x123456789ABCDEF0, 0x0FEDCBA987654321),
                           (0x1111111111111111, 0x2222222222222222)) == (
        0x2548FC88856CD77E, 0xADBCA20846B903C8)


def test_key_from_seed_and_fold_in(oracle):
    # proj/tests/test_rng.cpp:31-42
    assert oracle.key_from_seed(0).t() == (0xF2F49029F4075E39, 0x3C3D4A65617831ED)
    assert oracle.key_from_seed(1).t() == (0x0B6436BE3F21A6F0, 0xB8EB41B976A8A76F)
    assert oracle.key_from_seed(42).t() == (0x0661D05FD928D9EE, 0x6913EE86E86CC441)
    k = oracle.key_from_seed(7)
    assert oracle.fold_in(k, 0).t() == (0x12C2C44A2CA62D44, 0x2194946EA5E0E82E)
    assert oracle.fold_in(k, 13).t() == (0xB9D053AC08CD17EF, 0x90108DBD503F99B7)
    assert oracle.fold_in(oracle.fold_in(k, 3), 5).t() == (0xBCF4DFE7D648DB4B, 0xA21F99AA2129A00E)


def test_fold_in_injective(oracle):
    # proj/tests/test_rng.cpp:44-55
    k = oracle.key_from_seed(3)
    seen = {oracle.fold_in(k, i).t() for i in range(4096)}
    assert len(seen) == 4096 and k.t() not in seen


def test_stream_frozen_draws(oracle):
    # proj/tests/test_rng.cpp:63-84
    L = oracle.lib()
    k = oracle.key_from_seed(7)
    s = oracle.stream(k)
    words = [L.eo_next_u64(C.byref(s)) for _ in range(4)]
    assert words == [0xF2DC297DDC7C278F, 0xD13B6C13D62172DC, 0x549926A4763A6323, 0xAE8927F9FDF6B981]
    t = oracle.stream(k)
    assert [L.eo_uniform(C.byref(t)) for _ in range(4)] == [
        0.9486719066885461, 0.8173129604748561, 0.3304618979948173, 0.6817803368885177]
    n = oracle.stream(k)
    assert L.eo_normal(C.byref(n)) == 0.13324204080435406
    assert L.eo_normal(C.byref(n)) == -0.29602548786201777


def test_randint_unbiased(oracle):
    # proj/tests/test_rng.cpp:98-127
    L = oracle.lib()
    s = oracle.stream(oracle.key_from_seed(123))
    counts = np.zeros(256)
    for _ in range(1 << 16):
        counts[L.eo_randint(C.byref(s), 256)] += 1
    exp = (1 << 16) / 256
    assert ((counts - exp) ** 2 / exp).sum() < 330.5197436340
    s = oracle.stream(oracle.key_from_seed(5))
    c3 = np.bincount([L.eo_randint(C.byref(s), 3) for _ in range(30000)], minlength=3)
    assert np.all(np.abs(c3 - 10000) < 500)
    assert all(L.eo_randint(C.byref(s), 1) == 0 for _ in range(10))


def test_normal_moments(oracle):
    # proj/tests/test_rng.cpp:129-142
    z = oracle.gaussian_matrix(oracle.key_from_seed(77), 1, 200000)[0]
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1.0) < 0.02


def test_counter_addressable_normals(oracle):
    """normal #k of RandomStream(K) == Box-Muller(threefry(K,(1,k>>1)))[k&1]
    -- the identity the B200 noise kernel is built on."""
    import math
    k = oracle.key_from_seed(71)
    z = oracle.gaussian_matrix(k, 1, 64)[0]
    for i in range(64):
        w0, w1 = oracle.threefry(k.t(), (1, i >> 1))
        u1 = float((w0 >> 11) + 1) * 2.0 ** -53
        u2 = float(w1 >> 11) * 2.0 ** -53
        r = math.sqrt(-2.0 * math.log(u1))
        a = 2.0 * math.pi * u2
        assert z[i] == (r * math.cos(a) if i % 2 == 0 else r * math.sin(a))


@pytest.mark.skipif(not __import__("os").path.exists(
    __import__("oracle_ffi").REF_PATH) and not __import__("os").path.isdir("/root/reference/proj"),
    reason="reference rng.cpp not built")
def test_oracle_equals_reference_rng_bitwise(oracle):
    """Oracle restatement vs the reference's own rng.cpp (oracle/_ref)."""
    R = oracle.ref_lib()
    assert R is not None
    L = oracle.lib()
    rng = np.random.default_rng(0)
    for _ in range(200):
        key = tuple(int(x) for x in rng.integers(0, 2**63, 2, dtype=np.uint64))
        ctr = tuple(int(x) for x in rng.integers(0, 2**63, 2, dtype=np.uint64))
        o = (C.c_uint64 * 2)()
        R.ref_threefry2x64((C.c_uint64 * 2)(*key), (C.c_uint64 * 2)(*ctr), o)
        assert oracle.threefry(key, ctr) == (o[0], o[1])
    for seed in (0, 1, 7, 42, 2**40 + 3):
        o = (C.c_uint64 * 2)()
        R.ref_key_from_seed(C.c_uint64(seed), o)
        k = oracle.key_from_seed(seed)
        assert k.t() == (o[0], o[1])
        n = 4097
        for kind, dt in ((0, np.uint64), (1, np.float64), (2, np.float64), (3, np.uint64)):
            ref = np.empty(n, dt)
            R.ref_stream_draw((C.c_uint64 * 2)(*k.t()), kind, C.c_uint64(1000003), C.c_int64(n),
                              ref.ctypes.data_as(C.c_void_p))
            s = oracle.stream(k)
            if kind == 0:
                mine = np.array([L.eo_next_u64(C.byref(s)) for _ in range(n)], np.uint64)
            elif kind == 1:
                mine = np.array([L.eo_uniform(C.byref(s)) for _ in range(n)])
            elif kind == 2:
                mine = np.array([L.eo_normal(C.byref(s)) for _ in range(n)])
            else:
                mine = np.array([L.eo_randint(C.byref(s), 1000003) for _ in range(n)], np.uint64)
            assert np.array_equal(mine.view(np.uint64), ref.view(np.uint64)), kind
