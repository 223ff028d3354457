"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the SDPA forward hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It is
the checker, never the product: the product path
(``paper_2603_01960_b200``) does not import it and fails loudly when its CUDA
library is missing.

Two CPU implementations live behind this module:

* ``liboracle.so`` — our plain-C restatement (oracle/oracle.c) of the
  reference algorithm: ``make_input`` (types.cpp:118-164), ``snap_to_dtype``
  (types.cpp:52-78), ``sdpa_reference`` (reference.cpp:8-55) extended with the
  row max and LSE, and the online-softmax primitives (tiled.hpp:124-238).
* ``oracle/_ref/libtileattn_ref_*.so`` — the reference's own
  types/reference/tiled.cpp compiled from /root/reference by oracle/Makefile
  (see ``ref_*`` functions).  It pins the restatement
  (tests/test_oracle.py) and is the timed CPU baseline.

Parity pinned: yes — against oracle/_ref (reference run here) and the golden
fixtures in tests/golden/ (generated from oracle/_ref by
tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
REF = HERE / "_ref"

F32, F16, BF16 = 0, 1, 2
MASK_NONE, MASK_CAUSAL, MASK_PADDING = 0, 1, 2

_c = ctypes
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")


def build(force: bool = False) -> None:
    """Compile oracle.c (and oracle/_ref when /root/reference is present)."""
    cmd = ["make", "-C", str(HERE), "-s", "-j4"]
    if force:
        cmd.append("-B")
    subprocess.run(cmd, check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        path = BUILD / "liboracle.so"
        if not path.exists():
            build()
        L = ctypes.CDLL(str(path))
        L.oracle_snap.restype = _c.c_float
        L.oracle_snap.argtypes = [_c.c_float, _c.c_int]
        L.oracle_make_input.restype = None
        L.oracle_make_input.argtypes = [_c.c_int64, _c.c_int, _c.c_uint64, _f32p, _f32p, _f32p]
        L.oracle_to_bits16.restype = None
        L.oracle_to_bits16.argtypes = [_f32p, _u16p, _c.c_int64, _c.c_int]
        L.oracle_from_bits16.restype = None
        L.oracle_from_bits16.argtypes = [_u16p, _f32p, _c.c_int64, _c.c_int]
        L.oracle_sdpa_reference.restype = _c.c_int
        L.oracle_sdpa_reference.argtypes = [
            _f32p, _f32p, _f32p, _c.c_int64, _c.c_int64, _c.c_int64, _c.c_int64, _c.c_double,
            _c.c_int, _c.c_void_p, _c.c_int64, _c.c_int64, _f64p, _f64p, _f64p, _f64p]
        L.oracle_online_update.restype = None
        L.oracle_online_update.argtypes = [
            _c.POINTER(_c.c_double), _c.POINTER(_c.c_double), _f64p, _c.c_int64, _f64p, _c.c_int,
            _f32p]
        L.oracle_finalize.restype = None
        L.oracle_finalize.argtypes = [_c.c_double, _f64p, _c.c_int64, _f64p]
        L.oracle_schedule_supported.restype = _c.c_int
        L.oracle_schedule_supported.argtypes = [_c.c_int, _c.c_int, _c.c_int]
        L.oracle_effective_scale.restype = _c.c_double
        L.oracle_effective_scale.argtypes = [_c.c_int, _c.c_double, _c.c_int64]
        _lib = L
    return _lib


def _cpu_has_avx512() -> bool:
    try:
        flags = Path("/proc/cpuinfo").read_text()
    except OSError:
        return False
    for line in flags.splitlines():
        if line.startswith("flags"):
            f = set(line.split(":", 1)[1].split())
            return {"avx512f", "avx512bw", "avx512vl", "avx512dq", "avx512cd"} <= f
    return False


def ref_variant(kind: str = "auto") -> Path:
    if kind == "auto":
        kind = "v4" if _cpu_has_avx512() else "v3"
    return REF / f"libtileattn_ref_{kind}.so"


def ref_available(kind: str = "exact") -> bool:
    return ref_variant(kind).exists()


_refs: dict = {}


def ref(kind: str = "exact"):
    """The reference itself (compiled from /root/reference sources)."""
    path = ref_variant(kind)
    key = str(path)
    if key in _refs:
        return _refs[key]
    if not path.exists():
        build()
    if not path.exists():
        raise FileNotFoundError(f"{path} missing: reference not built (needs /root/reference)")
    R = ctypes.CDLL(key)
    i64, cint, dbl = _c.c_int64, _c.c_int, _c.c_double
    R.ref_last_error.restype = _c.c_char_p
    R.ref_make_input.restype = cint
    R.ref_make_input.argtypes = [i64, i64, i64, i64, cint, _c.c_uint64, _f32p, _f32p, _f32p]
    R.ref_snap.restype = _c.c_float
    R.ref_snap.argtypes = [_c.c_float, cint]
    R.ref_effective_scale.restype = dbl
    R.ref_effective_scale.argtypes = [cint, dbl, i64]
    R.ref_sdpa_reference.restype = cint
    R.ref_sdpa_reference.argtypes = [_f32p, _f32p, _f32p, i64, i64, i64, i64, cint, cint, dbl,
                                     cint, _c.c_void_p, _f64p, _f64p]
    R.ref_sdpa_tiled.restype = cint
    R.ref_sdpa_tiled.argtypes = [_f32p, _f32p, _f32p, i64, i64, i64, i64, cint, cint, dbl, cint,
                                 _c.c_void_p, cint, cint, cint, cint, cint, cint, _f32p,
                                 _c.POINTER(_c.c_uint64)]
    R.ref_handle_new.restype = _c.c_void_p
    R.ref_handle_new.argtypes = [_f32p, _f32p, _f32p, i64, i64, i64, i64, cint]
    R.ref_handle_free.restype = None
    R.ref_handle_free.argtypes = [_c.c_void_p]
    R.ref_handle_run.restype = cint
    R.ref_handle_run.argtypes = [_c.c_void_p, cint, cint, cint, cint, cint,
                                 _c.POINTER(_c.c_float)]
    R.ref_lse_via_primitives.restype = cint
    R.ref_lse_via_primitives.argtypes = [_f32p, _f32p, _f32p, i64, i64, i64, i64, cint, dbl, cint,
                                         i64, i64, _f64p]
    R.ref_fast_expf.restype = _c.c_float
    R.ref_fast_expf.argtypes = [_c.c_float]
    _refs[key] = R
    return R


# --------------------------------------------------------------------------
# Restatement API (numpy in, numpy out)
# --------------------------------------------------------------------------

def make_input(shape, dtype: int, seed: int):
    """types.cpp:151-164 — q, k, v as f32 arrays [B,H,S,D] on the dtype grid."""
    B, H, S, D = shape
    n = B * H * S * D
    q = np.empty(n, np.float32)
    k = np.empty(n, np.float32)
    v = np.empty(n, np.float32)
    lib().oracle_make_input(n, dtype, seed, q, k, v)
    return q.reshape(shape), k.reshape(shape), v.reshape(shape)


def snap(x: float, dtype: int) -> float:
    return float(lib().oracle_snap(x, dtype))


def to_bits16(x: np.ndarray, dtype: int) -> np.ndarray:
    """Exact re-encoding of grid-valued f32 into 16-bit storage (fp16/bf16 bits)."""
    src = np.ascontiguousarray(x, np.float32).ravel()
    out = np.empty(src.size, np.uint16)
    lib().oracle_to_bits16(src, out, src.size, dtype)
    return out.reshape(np.shape(x))


def from_bits16(x: np.ndarray, dtype: int) -> np.ndarray:
    src = np.ascontiguousarray(x, np.uint16).ravel()
    out = np.empty(src.size, np.float32)
    lib().oracle_from_bits16(src, out, src.size, dtype)
    return out.reshape(np.shape(x))


def effective_scale(d: int, scale: float | None = None) -> float:
    return float(lib().oracle_effective_scale(0 if scale is None else 1,
                                              0.0 if scale is None else scale, d))


def sdpa_reference(q, k, v, scale=None, mask_kind=MASK_NONE, valid_len=None, heads=None):
    """reference.cpp:8-55 in C (double), plus row max and LSE.

    Returns dict(o=[B,H,S,D] f64, row_sums=[B,H,S], row_max=[B,H,S], lse=[B,H,S]).
    ``heads`` = (bh_begin, bh_end) restricts the work to those flattened heads;
    other heads are returned as zeros.
    """
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    B, H, S, D = q.shape
    sc = effective_scale(D, scale)
    o = np.zeros(q.shape, np.float64)
    rs = np.zeros((B, H, S), np.float64)
    rm = np.zeros((B, H, S), np.float64)
    lse = np.zeros((B, H, S), np.float64)
    b0, b1 = heads if heads is not None else (0, B * H)
    vl = None
    if mask_kind == MASK_PADDING:
        vl_arr = np.ascontiguousarray(valid_len, np.int64)
        vl = vl_arr.ctypes.data
    rc = lib().oracle_sdpa_reference(q, k, v, B, H, S, D, sc, mask_kind, vl, b0, b1, o, rs, rm,
                                     lse)
    if rc != 0:
        raise ValueError(f"oracle_sdpa_reference rc={rc}")
    return dict(o=o, row_sums=rs, row_max=rm, lse=lse)


def sdpa_numpy(q, k, v, scale=None, causal=False, valid_len=None):
    """Vectorised float64 restatement of the same math (BLAS-backed), for the
    larger sampled-head checks.  Agrees with sdpa_reference to ~1e-13
    (tests/test_oracle.py).  Returns (o [.., S, D] f64, lse [.., S] f64)."""
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    S, D = q.shape[-2], q.shape[-1]
    sc = effective_scale(D, scale)
    s = np.matmul(q, np.swapaxes(k, -1, -2)) * sc
    if causal:
        idx = np.arange(S)
        s = np.where(idx[None, :] <= idx[:, None], s, -np.inf)
    if valid_len is not None:
        if q.ndim == 2:  # one head: a single key-side length
            vl = int(np.asarray(valid_len).ravel()[0])
        else:            # [B, H, S, D]: one length per batch
            vl = np.asarray(valid_len).reshape(q.shape[0], *([1] * (q.ndim - 1)))
        s = np.where(np.arange(S) < vl, s, -np.inf)
    m = s.max(axis=-1, keepdims=True)
    finite = np.isfinite(m)
    m_safe = np.where(finite, m, 0.0)
    p = np.exp(s - m_safe)
    l = p.sum(axis=-1, keepdims=True)
    with np.errstate(invalid="ignore", divide="ignore"):
        o = np.where(finite, np.matmul(p, v) / np.where(l == 0, 1.0, l), 0.0)
        lse = np.where(finite, m_safe + np.log(np.where(l == 0, 1.0, l)), -np.inf)
    return o, lse[..., 0]


def online_update(state, scores, v_tile):
    """tiled.hpp:193-221 in double for a single row. state = [m, l, o(np f64)]."""
    m = _c.c_double(state[0])
    l = _c.c_double(state[1])
    o = state[2]
    sc = np.ascontiguousarray(scores, np.float64).copy()
    vt = np.ascontiguousarray(v_tile, np.float32)
    lib().oracle_online_update(_c.byref(m), _c.byref(l), o, o.size, sc, sc.size, vt)
    state[0], state[1] = m.value, l.value
    return sc


def finalize(state):
    out = np.empty_like(state[2])
    lib().oracle_finalize(state[1], state[2], state[2].size, out)
    return out


def schedule_supported(t_m, t_n, stages) -> bool:
    return bool(lib().oracle_schedule_supported(t_m, t_n, stages))


# Tolerances: reference gate (bench.cpp:56-63) and BASELINE.json.
REF_GATE_TOL = {F32: 1e-4, F16: 5e-3, BF16: 2e-2}
BASELINE_TOL = {F16: 1e-2, BF16: 2e-2}
LSE_TOL = 1e-3
