"""CPU tests: pin the oracle restatement (oracle/oracle.c) to the reference.

Anchors (reference file:line):
  make_input determinism / grid membership  test_types.cpp:111-135
  snap_to_dtype RNE known answers           test_types.cpp:58-79
  sdpa_reference properties                 test_reference.cpp:62-163
  online-softmax algebra KATs               test_tiled.cpp:106-232
  tiled vs oracle tolerances                test_tiled.cpp:273-291, bench.cpp:56-63
Pinned against: oracle/_ref (the reference compiled from its own sources,
when present) and tests/golden/ (generated from oracle/_ref).
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"
META = json.loads((GOLD / "golden.json").read_text())


def _sha(*arrays):
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------- golden pins
@pytest.mark.parametrize("name", sorted(META["cases"]))
def test_make_input_bytes_match_reference_golden(name):
    c = META["cases"][name]
    q, k, v = O.make_input(tuple(c["shape"]), c["dtype"], c["seed"])
    assert _sha(q, k, v) == c["input_sha256"]


@pytest.mark.parametrize("name", sorted(META["cases"]))
def test_oracle_matches_reference_golden(name):
    c = META["cases"][name]
    g = np.load(GOLD / f"{name}.npz")
    q, k, v = O.make_input(tuple(c["shape"]), c["dtype"], c["seed"])
    keep = c["heads_kept"]
    B, H, S, D = c["shape"]
    r = O.sdpa_reference(q, k, v, heads=(0, B * H))
    o = r["o"].reshape(B * H, S, D)[:keep]
    assert np.abs(o - g["o"]).max() <= 1e-6  # fixture stored as f32
    assert np.abs(r["row_sums"].reshape(B * H, S) - g["row_sums"]).max() <= 1e-9
    assert np.abs(r["lse"].reshape(B * H, S) - g["lse"]).max() <= 1e-12
    # the reference's own CPU path (f32 accum, default schedule) is within the
    # gate tolerance of the oracle (bench.cpp:56-63)
    assert np.abs(g["tiled_o"] - o).max() <= O.REF_GATE_TOL[c["dtype"]]


def test_snap_known_answers_match_reference():
    vals = META["snap"]["values"]
    for dt in (O.F16, O.BF16):
        want = META["snap"]["snapped"][str(dt)]
        got = [O.snap(x, dt) for x in vals]
        for g, w in zip(got, want):
            assert (math.isinf(g) and math.isinf(w)) or g == w


def test_snap_kats_from_reference_tests():
    # test_types.cpp:58-79
    assert O.snap(1.0 + 2**-11, O.F16) == 1.0
    assert O.snap(1.0 + 1.5 * 2**-11, O.F16) == 1.0 + 2**-10
    assert O.snap(65519.0, O.F16) == 65504.0
    assert math.isinf(O.snap(65520.0, O.F16))
    assert O.snap(2**-25, O.F16) == 0.0
    assert O.snap(1.5 * 2**-25, O.F16) == 2**-24
    assert O.snap(1.5 * 2**-24, O.F16) == 2**-23
    assert O.snap(257.0, O.BF16) == 256.0
    assert O.snap(1.0 + 2**-8, O.BF16) == 1.0


def test_to_bits16_is_exact_reencoding():
    import torch
    for dt, tdt in ((O.F16, torch.float16), (O.BF16, torch.bfloat16)):
        q, _, _ = O.make_input((1, 2, 64, 16), dt, 9)
        bits = O.to_bits16(q, dt)
        want = torch.from_numpy(q).to(tdt).view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(bits, want)
        assert np.array_equal(O.from_bits16(bits, dt), q)


def test_make_input_deterministic_and_on_grid():
    a = O.make_input((2, 2, 16, 8), O.F32, 42)
    b = O.make_input((2, 2, 16, 8), O.F32, 42)
    c = O.make_input((2, 2, 16, 8), O.F32, 43)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert not np.array_equal(a[0], c[0])
    for dt in (O.F16, O.BF16):
        for t in O.make_input((1, 2, 32, 16), dt, 7):
            assert np.all(np.isfinite(t))
            assert all(O.snap(float(x), dt) == x for x in t.ravel()[:512])


# ------------------------------------------------------------ live reference
ref_missing = not O.ref_available("exact")


@pytest.mark.skipif(ref_missing, reason="oracle/_ref not built (needs /root/reference)")
@pytest.mark.parametrize("dt", [O.F32, O.F16, O.BF16])
@pytest.mark.parametrize("mask", [O.MASK_NONE, O.MASK_CAUSAL, O.MASK_PADDING])
def test_oracle_matches_live_reference(dt, mask):
    R = O.ref("exact")
    B, H, S, D = 2, 2, 70, 24
    q, k, v = O.make_input((B, H, S, D), dt, 11)
    vl = np.array([35, 70], np.int64)
    o = np.empty(q.size, np.float64)
    rs = np.empty(B * H * S, np.float64)
    rc = R.ref_sdpa_reference(q.ravel().copy(), k.ravel().copy(), v.ravel().copy(), B, H, S, D,
                              dt, 0, 0.0, mask, vl.ctypes.data if mask == 2 else None, o, rs)
    assert rc == 0
    r = O.sdpa_reference(q, k, v, mask_kind=mask, valid_len=vl)
    assert np.abs(r["o"].ravel() - o).max() <= 1e-12
    assert np.abs(r["row_sums"].ravel() - rs).max() <= 1e-12


@pytest.mark.skipif(ref_missing, reason="oracle/_ref not built (needs /root/reference)")
def test_lse_oracle_matches_reference_primitives():
    R = O.ref("exact")
    B, H, S, D = 1, 2, 300, 64
    q, k, v = O.make_input((B, H, S, D), O.BF16, 5)
    lse = np.empty(B * H * S, np.float64)
    assert R.ref_lse_via_primitives(q.ravel().copy(), k.ravel().copy(), v.ravel().copy(), B, H,
                                    S, D, 0, 0.0, 128, 0, B * H, lse) == 0
    r = O.sdpa_reference(q, k, v)
    assert np.abs(r["lse"].ravel() - lse).max() <= 1e-12


# ------------------------------------------------------------ oracle algebra
def test_worked_example_two_tiles():
    # test_tiled.cpp:106-131
    st = [-math.inf, 0.0, np.zeros(1)]
    O.online_update(st, [0.0], np.array([1.0], np.float32))
    assert st[0] == 0.0 and st[1] == 1.0 and st[2][0] == 1.0
    O.online_update(st, [math.log(3.0)], np.array([2.0], np.float32))
    assert st[1] == pytest.approx(4.0 / 3.0, rel=1e-14)
    assert st[2][0] == pytest.approx(7.0 / 3.0, rel=1e-14)
    assert O.finalize(st)[0] == pytest.approx(1.75, rel=1e-12)


def test_fully_masked_tile_keeps_init_state():
    st = [-math.inf, 0.0, np.zeros(3)]
    O.online_update(st, [-math.inf], np.full(3, 5.0, np.float32))
    assert st[0] == -math.inf and st[1] == 0.0 and not np.any(st[2])
    assert not np.any(O.finalize(st))  # l == 0 -> zero row (tiled.hpp:231-233)


def test_online_chain_equals_two_pass():
    rng = np.random.default_rng(123)
    for _ in range(100):
        keys, d = int(rng.integers(1, 9)), int(rng.integers(1, 5))
        s = rng.standard_normal(keys)
        v = rng.standard_normal((keys, d)).astype(np.float32)
        st = [-math.inf, 0.0, np.zeros(d)]
        pos = 0
        while pos < keys:
            cols = min(int(rng.integers(1, 4)), keys - pos)
            O.online_update(st, s[pos:pos + cols], v[pos:pos + cols])
            pos += cols
        w = np.exp(s - s.max())
        want = (w / w.sum()) @ v.astype(np.float64)
        assert np.allclose(O.finalize(st), want, rtol=1e-12, atol=1e-12)


def test_reference_properties():
    # S=1 -> v (test_reference.cpp:77-82)
    q, k, v = O.make_input((1, 1, 1, 4), O.F32, 3)
    assert np.array_equal(O.sdpa_reference(q, k, v)["o"].ravel(), v.ravel().astype(np.float64))
    # causal row 0 -> v0 (:84-89)
    q, k, v = O.make_input((1, 1, 2, 4), O.F32, 5)
    r = O.sdpa_reference(q, k, v, mask_kind=O.MASK_CAUSAL)
    assert np.array_equal(r["o"][0, 0, 0], v[0, 0, 0].astype(np.float64))
    # Q = 0 -> mean(V), row_sums == S, LSE == ln S (:91-103)
    q, k, v = O.make_input((1, 1, 6, 4), O.F32, 1)
    r = O.sdpa_reference(np.zeros_like(q), k, v)
    assert np.allclose(r["o"][0, 0], v[0, 0].astype(np.float64).mean(0)[None, :], rtol=1e-12)
    assert np.all(r["row_sums"] == 6.0)
    assert np.allclose(r["lse"], math.log(6.0), rtol=0, atol=1e-15)
    # padding rows with valid_len 0 -> zeros, LSE -inf (:105-113)
    q, k, v = O.make_input((2, 1, 8, 4), O.F32, 21)
    r = O.sdpa_reference(q, k, v, mask_kind=O.MASK_PADDING, valid_len=[0, 8])
    assert not np.any(r["o"][0]) and np.all(r["row_sums"][0] == 0)
    assert np.all(np.isneginf(r["lse"][0])) and np.all(r["row_sums"][1] > 0)
    # convex hull (:148-163)
    q, k, v = O.make_input((1, 2, 24, 8), O.F32, 31)
    o = O.sdpa_reference(q, k, v)["o"]
    lo, hi = v.min(axis=2, keepdims=True), v.max(axis=2, keepdims=True)
    assert np.all(o >= lo - 1e-12) and np.all(o <= hi + 1e-12)


def test_numpy_restatement_agrees_with_c_oracle():
    q, k, v = O.make_input((1, 2, 200, 64), O.BF16, 4)
    r = O.sdpa_reference(q, k, v)
    o, lse = O.sdpa_numpy(q, k, v)
    assert np.abs(o - r["o"]).max() <= 1e-12
    assert np.abs(lse - r["lse"]).max() <= 1e-12
    rc = O.sdpa_reference(q, k, v, mask_kind=O.MASK_CAUSAL)
    oc, lc = O.sdpa_numpy(q, k, v, causal=True)
    assert np.abs(oc - rc["o"]).max() <= 1e-12 and np.abs(lc - rc["lse"]).max() <= 1e-12


def test_schedule_rules_match_reference():
    # test_tiled.cpp:256-262
    assert O.schedule_supported(64, 128, 2)
    assert not O.schedule_supported(48, 128, 2)
    assert not O.schedule_supported(64, 512, 2)
    assert not O.schedule_supported(64, 128, 0)
    assert not O.schedule_supported(64, 128, 5)


def test_effective_scale():
    assert O.effective_scale(64) == 0.125
    assert O.effective_scale(128) == pytest.approx(0.0883883476483184406, rel=1e-15)
    assert O.effective_scale(64, 0.5) == 0.5
