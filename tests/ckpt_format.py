"""EVORL1 checkpoint format, restated for the tests (test infrastructure).

proj/src/checkpoint.cpp:6-212: magic "EVORL1", u32 version 1, u32-length-prefixed
workflow id, u32 segment count, then segments {u32 name length, name, u8 type
(0 = f64, 1 = i64), u64 element count, little-endian 64-bit payload}.
"""
import struct

import numpy as np


def write(path, workflow_id, segments):
    """segments: list of (name, 'f64' | 'i64', values)."""
    out = bytearray(b"EVORL1")
    out += struct.pack("<I", 1)
    out += struct.pack("<I", len(workflow_id)) + workflow_id.encode()
    out += struct.pack("<I", len(segments))
    for name, kind, vals in segments:
        vals = np.atleast_1d(np.asarray(vals, dtype=np.float64 if kind == "f64" else np.int64))
        out += struct.pack("<I", len(name)) + name.encode()
        out += struct.pack("<B", 0 if kind == "f64" else 1)
        out += struct.pack("<Q", vals.size)
        out += vals.astype("<f8" if kind == "f64" else "<i8").tobytes()
    with open(path, "wb") as f:
        f.write(bytes(out))


def read(path):
    """-> (workflow_id, [(name, 'f64' | 'i64', np.ndarray)]) in file order."""
    b = open(path, "rb").read()
    assert b[:6] == b"EVORL1"
    (ver,) = struct.unpack_from("<I", b, 6)
    assert ver == 1
    pos = 10
    (n,) = struct.unpack_from("<I", b, pos)
    pos += 4
    wid = b[pos:pos + n].decode()
    pos += n
    (nseg,) = struct.unpack_from("<I", b, pos)
    pos += 4
    segs = []
    for _ in range(nseg):
        (ln,) = struct.unpack_from("<I", b, pos)
        pos += 4
        name = b[pos:pos + ln].decode()
        pos += ln
        t = b[pos]
        pos += 1
        (cnt,) = struct.unpack_from("<Q", b, pos)
        pos += 8
        arr = np.frombuffer(b, dtype="<f8" if t == 0 else "<i8", count=cnt, offset=pos).copy()
        pos += 8 * cnt
        segs.append((name, "f64" if t == 0 else "i64", arr))
    assert pos == len(b)
    return wid, segs


# EsWorkflow::save segment order (proj/src/workflow.cpp:11-17, :146-165,
# proj/src/workflow_es.cpp:181-209)
BASE = [("iteration", "i64"), ("rng", "i64"), ("env_steps", "i64"), ("episodes", "i64"),
        ("rl_updates", "i64"), ("obs_norm/mode", "i64"), ("obs_norm/mean", "f64"),
        ("obs_norm/var", "f64"), ("obs_norm/count", "f64")]
EC = {
    "openes": [("ec/mean", "f64"), ("ec/sigma", "f64"), ("ec/adam/m", "f64"), ("ec/adam/v", "f64"),
               ("ec/adam/t", "i64"), ("ec/table_seed", "i64")],
    "ars": [("ec/mean", "f64")],
    "ves": [("ec/mean", "f64")],
    "cmaes": [("ec/mean", "f64"), ("ec/sigma", "f64"), ("ec/C", "f64"), ("ec/B", "f64"), ("ec/D", "f64"),
              ("ec/ps", "f64"), ("ec/pc", "f64"), ("ec/generation", "i64"),
              ("ec/recondition_count", "i64")],
    "cem": [("ec/mean", "f64"), ("ec/var", "f64"), ("ec/iter", "i64")],
}
