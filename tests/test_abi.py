"""CPU tests of the C-ABI boundary (no compute calls need a GPU here).

* the library loads and exports every symbol include/*.h declares;
* host-side validation follows the reference's order and error classes
  (tiled.cpp:253-259; types.cpp:80-116; tiled.cpp:21-35);
* without an sm_100 device the compute entries fail loudly (no CPU fallback).
"""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

import paper_2603_01960_b200 as ta

ROOT = Path(__file__).resolve().parents[1]


def _declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        names |= set(re.findall(r"TA_API\s+[\w\s\*]+?\b(ta_\w+)\s*\(", h.read_text()))
    return names


def test_library_exports_every_declared_symbol():
    names = _declared_symbols()
    assert {"ta_sdpa_fwd", "ta_sdpa_fwd_host", "ta_last_error"} <= names
    out = subprocess.run(["nm", "-D", "--defined-only", str(ta._LIB_PATH)], check=True,
                         capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert names <= exported, names - exported
    L = ta.lib()
    for n in names:
        assert getattr(L, n) is not None


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(ta._LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert re.search(r"sm_(80|86|89|90)\b", out) is None


def test_abi_version():
    assert ta.lib().ta_abi_version() == 1


def test_schedule_rules_mirror_reference():
    S = ta.TileSchedule
    assert ta.schedule_supported(S(64, 128, 2, ta.ROW))
    assert ta.schedule_supported(S(128, 256, 4, ta.COL))
    for bad in (S(48, 128, 2), S(64, 512, 2), S(64, 128, 0), S(64, 128, 5), S(64, 64, 7)):
        assert not ta.schedule_supported(bad)


def test_effective_scale_mirrors_reference():
    assert ta.effective_scale(64) == 0.125
    assert ta.effective_scale(128) == pytest.approx(0.0883883476483184406, rel=1e-15)
    assert ta.effective_scale(64, 0.5) == 0.5
    for bad in ((64, 0.0), (64, -1.0)):
        with pytest.raises(ValueError):
            ta.effective_scale(*bad)
    with pytest.raises(ValueError):
        ta.effective_scale(0)


def _call(shape=(1, 1, 64, 64), dtype=ta.BF16, **kw):
    # fake but aligned non-null device pointers: validation runs before any
    # device access, and on a GPU-less host the call must then fail loudly.
    p = 1 << 20
    ta.sdpa_fwd(p, p, p, p, 0, shape, dtype, **kw)


def test_validation_order_and_error_classes():
    # shape first (types.cpp:80-83) even when the schedule is also bad
    with pytest.raises(ValueError, match="shape"):
        _call(shape=(0, 1, 64, 64), schedule=ta.TileSchedule(48, 128, 2))
    # mask next: padding needs valid_len entries in [0,S]
    with pytest.raises(ValueError, match="valid_len"):
        _call(mask_kind=ta.MASK_PADDING, valid_len=[65])
    # schedule (tiled.cpp:29-35) before scale
    with pytest.raises(ta.UnsupportedScheduleError, match="schedule"):
        _call(schedule=ta.TileSchedule(64, 64, 7), scale=-1.0)
    # scale (types.cpp:108-116)
    with pytest.raises(ValueError, match="scale"):
        _call(scale=0.0)
    # f32 and odd head dims are "unsupported" (status=unsupported rows)
    with pytest.raises(ta.UnsupportedScheduleError):
        _call(dtype=ta.F32)
    with pytest.raises(ta.UnsupportedScheduleError):
        _call(shape=(1, 1, 64, 44))
    with pytest.raises(ta.UnsupportedScheduleError):
        _call(shape=(1, 1, 64, 264))


def test_padding_length_must_match_batch():
    # a short valid_len list would be read past its end by the C-ABI
    with pytest.raises(ValueError, match="one valid_len per batch"):
        _call(shape=(3, 1, 64, 64), mask_kind=ta.MASK_PADDING, valid_len=[64, 64])
    with pytest.raises(ValueError, match="one valid_len per batch"):
        _call(shape=(1, 1, 64, 64), mask_kind=ta.MASK_PADDING, valid_len=[64, 64])
    # shape errors still come first (shape -> mask)
    with pytest.raises(ValueError, match="shape"):
        _call(shape=(0, 1, 64, 64), mask_kind=ta.MASK_PADDING, valid_len=[64, 64])


def test_scale_predicate_matches_reference():
    # types.cpp:108-116 throws only for *scale <= 0.0: NaN is accepted there
    # and propagates into the output; the C-ABI follows the same predicate
    import math
    assert math.isnan(ta.effective_scale(64, float("nan")))
    for bad in (0.0, -0.0, -1.0, float("-inf")):
        with pytest.raises(ValueError, match="scale"):
            ta.effective_scale(64, bad)
    assert ta.effective_scale(64, float("inf")) == float("inf")


def test_release_workspace_validates_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    with pytest.raises((ta.CudaError, ValueError)):
        ta.release_workspace(0)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    with pytest.raises(ta.CudaError):
        _call()
    with pytest.raises(ta.CudaError):
        import numpy as np
        x = np.zeros((1, 1, 64, 64), np.float32)
        ta.sdpa_tiled(x, x, x, dtype=ta.BF16)


def test_plan_cache_counts_only_successful_validations():
    ta.plan_cache_clear()
    assert ta.plan_cache_stats() == (0, 0)
    with pytest.raises(ValueError):
        _call(shape=(1, 0, 64, 64))
    assert ta.plan_cache_stats() == (0, 0)
