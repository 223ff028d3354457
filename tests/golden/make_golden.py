"""Generate tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref, compiled
from /root/reference/proj/src by oracle/Makefile).

Run here (the container that has /root/reference):
    make -C oracle && python tests/golden/make_golden.py

Every fixture records the generating call so the oracle restatement (and the
GPU kernel, through it) is pinned to reference outputs even on hosts where
/root/reference does not exist.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent

# (name, B, H, S, D, dtype, seed, heads_kept_for_O)
CASES = [
    ("cfg1_f16", 1, 8, 512, 64, oracle.F16, 0, 2),         # BASELINE configs[0]
    ("ragged130_bf16_d64", 1, 2, 130, 64, oracle.BF16, 77, 2),  # test_tiled.cpp:273-291 shape family
    ("ragged130_f16_d128", 1, 2, 130, 128, oracle.F16, 77, 2),
    ("short32_bf16_d128", 1, 2, 32, 128, oracle.BF16, 77, 2),
    ("s1_bf16_d64", 1, 1, 1, 64, oracle.BF16, 3, 1),         # test_reference.cpp:77-82
    ("s1000_bf16_d64", 1, 1, 1000, 64, oracle.BF16, 3, 1),   # ragged, several K/V tiles
]

SNAP_VALUES = np.array([1.0, 1.0 + 2**-11, 1.0 + 1.5 * 2**-11, 65519.0, 65520.0, 2**-25,
                        1.5 * 2**-25, 1.5 * 2**-24, -1.5, 257.0, 1.0 + 2**-8, 3.0, 0.1234567,
                        0.0, -0.333333, 1e-6, 7.77e4], dtype=np.float32)


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main() -> None:
    R = oracle.ref("exact")
    meta = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref/libtileattn_ref_exact.so",
            "cases": {}}
    for name, B, H, S, D, dt, seed, keep in CASES:
        n = B * H * S * D
        q = np.empty(n, np.float32)
        k = np.empty(n, np.float32)
        v = np.empty(n, np.float32)
        assert R.ref_make_input(B, H, S, D, dt, seed, q, k, v) == 0
        o = np.empty(n, np.float64)
        rs = np.empty(B * H * S, np.float64)
        assert R.ref_sdpa_reference(q, k, v, B, H, S, D, dt, 0, 0.0, 0, None, o, rs) == 0
        lse = np.empty(B * H * S, np.float64)
        assert R.ref_lse_via_primitives(q, k, v, B, H, S, D, 0, 0.0, 128, 0, B * H, lse) == 0
        tiled = np.empty(n, np.float32)
        visited = __import__("ctypes").c_uint64()
        assert R.ref_sdpa_tiled(q, k, v, B, H, S, D, dt, 0, 0.0, 0, None, 64, 128, 2, 0, 0, 0,
                                tiled, visited) == 0
        o4 = o.reshape(B * H, S, D)[:keep]
        np.savez_compressed(
            OUT / f"{name}.npz",
            o=o4.astype(np.float32), row_sums=rs.reshape(B * H, S), lse=lse.reshape(B * H, S),
            tiled_o=tiled.reshape(B * H, S, D)[:keep],
            v_head0=v.reshape(B * H, S, D)[0].copy())
        meta["cases"][name] = dict(shape=[B, H, S, D], dtype=dt, seed=seed, heads_kept=keep,
                                   input_sha256=sha(q, k, v),
                                   tiled_schedule=[64, 128, 2, "row"],
                                   tiled_kv_tiles_visited=int(visited.value))
        print(name, "ok")
    snapped = {str(dt): [float(R.ref_snap(float(x), dt)) for x in SNAP_VALUES]
               for dt in (oracle.F16, oracle.BF16)}
    meta["snap"] = {"values": [float(x) for x in SNAP_VALUES], "snapped": snapped}
    xs = -np.arange(0, 88000, 997, dtype=np.float32) / 1000.0
    meta["fast_expf"] = {"x": [float(x) for x in xs],
                         "y": [float(R.ref_fast_expf(float(x))) for x in xs]}
    (OUT / "golden.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
