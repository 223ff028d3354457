"""B200-native SDPA forward (sm_100a tcgen05/TMA/TMEM) behind the reference API.

Python mirror of the reference operator interface:

* ``sdpa(q, k, v, causal=False, scale=None)`` — the paper's functional API
  (reference PAPER.md:139-145, "from tiledattention import sdpa").
* ``sdpa_tiled(...)`` — the reference C++ entry point
  ``tileattn::sdpa_tiled(input, mask, scale, sched, cache, options)``
  (proj/include/tileattn/tiled.hpp:274-277) with the same argument meaning and
  error classes (``ValueError`` for ``std::invalid_argument``,
  ``UnsupportedScheduleError`` for the reference's
  ``UnsupportedScheduleError``).

Everything computes in ``libtileattn_b200.so`` through the C-ABI declared in
include/tileattn_b200.h.  There is no CPU fallback: if the library or an sm_100
device is missing, calls raise.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence

__all__ = [
    "TileSchedule", "KernelStats", "UnsupportedScheduleError", "CudaError", "lib",
    "sdpa", "sdpa_fwd", "sdpa_fwd_host", "sdpa_tiled", "schedule_supported",
    "effective_scale", "plan_cache_stats", "plan_cache_clear", "release_workspace", "F32", "F16", "BF16",
    "MASK_NONE", "MASK_CAUSAL", "MASK_PADDING",
]

_PKG = Path(__file__).resolve().parent
import os as _os

# TILEATTN_B200_LIB: load an alternative build of the same C-ABI (tuning
# experiments); the default is the in-tree library.
_LIB_PATH = Path(_os.environ.get("TILEATTN_B200_LIB", _PKG / "_lib" / "libtileattn_b200.so"))

TA_OK, TA_ERR_INVALID_ARGUMENT, TA_ERR_UNSUPPORTED, TA_ERR_OOM, TA_ERR_CUDA = range(5)
F32, F16, BF16 = 0, 1, 2
MASK_NONE, MASK_CAUSAL, MASK_PADDING = 0, 1, 2
ROW, COL = 0, 1


class UnsupportedScheduleError(RuntimeError):
    """tileattn::UnsupportedScheduleError (tiled.hpp:39-41); also raised for
    shapes/dtypes the sm_100a kernel does not cover (status=unsupported,
    bench.cpp:290-292)."""


class CudaError(RuntimeError):
    """CUDA runtime failure or no sm_100 device."""


class _Schedule(ctypes.Structure):
    _fields_ = [("t_m", ctypes.c_int32), ("t_n", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("layout", ctypes.c_int32)]


class _Shape(ctypes.Structure):
    _fields_ = [("b", ctypes.c_int64), ("h", ctypes.c_int64), ("s", ctypes.c_int64),
                ("d", ctypes.c_int64)]


class _Stats(ctypes.Structure):
    _fields_ = [("kv_tiles_visited", ctypes.c_uint64), ("block_m", ctypes.c_int32),
                ("block_n", ctypes.c_int32), ("stages", ctypes.c_int32),
                ("q_tiles_per_cta", ctypes.c_int32), ("ctas", ctypes.c_int64),
                ("threads_per_cta", ctypes.c_int32), ("reserved", ctypes.c_int32)]


@dataclass(frozen=True)
class TileSchedule:
    """TileSchedule (tiled.hpp:30-37); default {64,128,2,row}."""
    t_m: int = 64
    t_n: int = 128
    stages: int = 2
    layout: int = ROW

    def _c(self) -> _Schedule:
        return _Schedule(self.t_m, self.t_n, self.stages, self.layout)


@dataclass
class KernelStats:
    """KernelStats (tiled.hpp:247-257) + the executed GPU tiling."""
    kv_tiles_visited: int = 0
    block_m: int = 0
    block_n: int = 0
    stages: int = 0
    q_tiles_per_cta: int = 0
    ctas: int = 0
    threads_per_cta: int = 0


_lib = None


def lib() -> ctypes.CDLL:
    """Load the sm_100a library (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise ImportError(f"{_LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (needs nvcc) — there is no CPU fallback")
    L = ctypes.CDLL(str(_LIB_PATH))
    vp, i64, cint, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    sig = [vp, vp, vp, vp, vp, _Shape, cint, cint, vp, cint, dbl, _Schedule, vp,
           ctypes.POINTER(_Stats)]
    L.ta_sdpa_fwd.restype = cint
    L.ta_sdpa_fwd.argtypes = sig
    L.ta_sdpa_fwd_host.restype = cint
    L.ta_sdpa_fwd_host.argtypes = sig
    L.ta_last_error.restype = ctypes.c_char_p
    L.ta_last_error.argtypes = []
    L.ta_abi_version.restype = cint
    L.ta_schedule_supported.restype = cint
    L.ta_schedule_supported.argtypes = [_Schedule]
    L.ta_effective_scale.restype = cint
    L.ta_effective_scale.argtypes = [cint, dbl, i64, ctypes.POINTER(dbl)]
    L.ta_plan_cache_stats.restype = None
    L.ta_plan_cache_stats.argtypes = [ctypes.POINTER(ctypes.c_uint64)] * 2
    L.ta_plan_cache_clear.restype = None
    L.ta_device_supported.restype = cint
    L.ta_device_supported.argtypes = [cint]
    L.ta_sdpa_check.restype = cint
    L.ta_sdpa_check.argtypes = [_Shape, cint, cint, vp, cint, dbl, _Schedule]
    # (ABI 1 additions: bound when present, so older builds of the same ABI
    # still load for A/B timing; tests/test_abi.py checks the product exports all)
    if hasattr(L, "ta_release_workspace"):
        L.ta_release_workspace.restype = cint
        L.ta_release_workspace.argtypes = [cint]
    if hasattr(L, "ta_debug_exp2"):
        L.ta_debug_exp2.restype = cint
        L.ta_debug_exp2.argtypes = [vp, vp, i64, cint, vp]
    L.ta_debug_umma_gemm.restype = cint
    L.ta_debug_umma_gemm.argtypes = [cint, cint, vp, vp, vp, vp]
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == TA_OK:
        return
    msg = lib().ta_last_error().decode(errors="replace")
    if rc == TA_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == TA_ERR_UNSUPPORTED:
        raise UnsupportedScheduleError(msg)
    if rc == TA_ERR_OOM:
        raise MemoryError(msg)
    raise CudaError(msg)


def schedule_supported(sched: TileSchedule) -> bool:
    return bool(lib().ta_schedule_supported(sched._c()))


def effective_scale(d: int, scale: Optional[float] = None) -> float:
    out = ctypes.c_double()
    _check(lib().ta_effective_scale(0 if scale is None else 1,
                                    0.0 if scale is None else float(scale), d,
                                    ctypes.byref(out)))
    return out.value


def plan_cache_stats() -> tuple[int, int]:
    h, c = ctypes.c_uint64(), ctypes.c_uint64()
    lib().ta_plan_cache_stats(ctypes.byref(h), ctypes.byref(c))
    return h.value, c.value


def plan_cache_clear() -> None:
    lib().ta_plan_cache_clear()


def release_workspace(device: int = 0) -> None:
    """Free the host-entry workspace and padding pool of ``device``."""
    _check(lib().ta_release_workspace(int(device)))


def _stats_out(st: _Stats, stats: Optional[KernelStats]) -> None:
    if stats is None:
        return
    for f in ("kv_tiles_visited", "block_m", "block_n", "stages", "q_tiles_per_cta", "ctas",
              "threads_per_cta"):
        setattr(stats, f, getattr(st, f))


_DEFAULT_SCHEDULE = None


def _default_schedule():
    global _DEFAULT_SCHEDULE
    if _DEFAULT_SCHEDULE is None:
        _DEFAULT_SCHEDULE = TileSchedule()._c()
    return _DEFAULT_SCHEDULE


def _current_stream(device) -> int:
    """Raw pointer of torch's current stream on ``device`` (fast path)."""
    import torch
    try:
        return torch._C._cuda_getCurrentRawStream(device.index)
    except (AttributeError, TypeError):
        return torch.cuda.current_stream(device).cuda_stream


def _mask_args(mask_kind: int, valid_len, shape):
    if mask_kind == MASK_PADDING:
        # the C-ABI reads valid_len[0..B-1]: a shorter list would be read past
        # its end (the reference validates the size, types.cpp:99-106).  A bad
        # shape is left to the library, which reports it first (shape -> mask).
        shape_ok = all(int(x) >= 1 for x in shape)
        if valid_len is None or (shape_ok and len(valid_len) != int(shape[0])):
            raise ValueError("padding mask needs one valid_len per batch")
        arr = (ctypes.c_int64 * len(valid_len))(*[int(x) for x in valid_len])
        return arr, ctypes.cast(arr, ctypes.c_void_p)
    return None, None


def sdpa_fwd(q_ptr: int, k_ptr: int, v_ptr: int, o_ptr: int, lse_ptr: int, shape: Sequence[int],
             dtype: int, *, mask_kind: int = MASK_NONE, valid_len=None,
             scale: Optional[float] = None, schedule: Optional[TileSchedule] = None,
             stream: int = 0, stats: Optional[KernelStats] = None) -> None:
    """Raw device-pointer entry (ta_sdpa_fwd)."""
    keep, vl = _mask_args(mask_kind, valid_len, shape)
    st = _Stats() if stats is not None else None
    sched = schedule._c() if schedule is not None else _default_schedule()
    rc = lib().ta_sdpa_fwd(q_ptr, k_ptr, v_ptr, o_ptr, lse_ptr or None, _Shape(*shape), dtype,
                           mask_kind, vl, 0 if scale is None else 1,
                           0.0 if scale is None else float(scale), sched, stream or None,
                           ctypes.byref(st) if st is not None else None)
    _check(rc)
    if st is not None:
        _stats_out(st, stats)


def sdpa_fwd_host(q_ptr: int, k_ptr: int, v_ptr: int, o_ptr: int, lse_ptr: int,
                  shape: Sequence[int], dtype: int, *, mask_kind: int = MASK_NONE,
                  valid_len=None, scale: Optional[float] = None,
                  schedule: Optional[TileSchedule] = None, stream: int = 0,
                  stats: Optional[KernelStats] = None) -> None:
    """Raw host-pointer entry (ta_sdpa_fwd_host): H2D, kernel, D2H, sync."""
    keep, vl = _mask_args(mask_kind, valid_len, shape)
    st = _Stats()
    sched = (schedule or TileSchedule())._c()
    rc = lib().ta_sdpa_fwd_host(q_ptr, k_ptr, v_ptr, o_ptr, lse_ptr or None, _Shape(*shape),
                                dtype, mask_kind, vl, 0 if scale is None else 1,
                                0.0 if scale is None else float(scale), sched, stream or None,
                                ctypes.byref(st))
    _check(rc)
    _stats_out(st, stats)


def _torch_dtype_code(t) -> int:
    import torch
    if t.dtype == torch.bfloat16:
        return BF16
    if t.dtype == torch.float16:
        return F16
    if t.dtype == torch.float32:
        return F32
    raise ValueError(f"unsupported dtype {t.dtype}")


def sdpa(q, k, v, causal: bool = False, scale: Optional[float] = None, *,
         return_lse: bool = False, valid_len=None, schedule: Optional[TileSchedule] = None,
         out=None, lse_out=None, stats: Optional[KernelStats] = None):
    """``o = sdpa(q, k, v, causal, scale)`` on CUDA tensors [B,H,S,D] (fp16/bf16).

    Returns ``o`` or ``(o, lse)`` with ``lse`` fp32 [B,H,S] (natural log).
    Runs on the current torch CUDA stream.
    """
    import torch
    if q.dim() != 4 or k.shape != q.shape or v.shape != q.shape:
        raise ValueError("q, k, v must share one [B,H,S,D] shape")
    if not (q.is_cuda and k.is_cuda and v.is_cuda):
        raise ValueError("q, k, v must be CUDA tensors (no CPU fallback)")
    if k.device != q.device or v.device != q.device:
        raise ValueError("q, k, v must be on one device")
    if q.dtype != k.dtype or q.dtype != v.dtype:
        raise ValueError("q, k, v must share one dtype")
    dt = _torch_dtype_code(q)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    B, H, S, D = q.shape
    # caller buffers are written through raw pointers as a contiguous
    # [B,H,S,D] 16-bit O and a contiguous [B,H,S] fp32 LSE: check exactly that
    if out is not None and (out.shape != q.shape or out.dtype != q.dtype
                            or out.device != q.device or not out.is_contiguous()):
        raise ValueError("out must be a contiguous tensor of q's shape, dtype and device")
    o = out if out is not None else torch.empty_like(q)
    lse = None
    if return_lse:
        if lse_out is not None and (tuple(lse_out.shape) != (B, H, S)
                                    or lse_out.dtype != torch.float32
                                    or lse_out.device != q.device
                                    or not lse_out.is_contiguous()):
            raise ValueError("lse_out must be a contiguous float32 [B,H,S] tensor on q's device")
        lse = lse_out if lse_out is not None else torch.empty((B, H, S), device=q.device,
                                                              dtype=torch.float32)
    mask_kind = MASK_CAUSAL if causal else (MASK_PADDING if valid_len is not None else MASK_NONE)
    stream = _current_stream(q.device)
    args = (q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
            lse.data_ptr() if lse is not None else 0, (B, H, S, D), dt)
    kw = dict(mask_kind=mask_kind, valid_len=valid_len, scale=scale, schedule=schedule,
              stream=stream, stats=stats)
    if torch.cuda.current_device() == q.device.index:
        sdpa_fwd(*args, **kw)
    else:
        with torch.cuda.device(q.device):
            sdpa_fwd(*args, **kw)
    return (o, lse) if return_lse else o


def sdpa_tiled(q, k, v, mask_kind: int = MASK_NONE, valid_len=None,
               scale: Optional[float] = None, schedule: Optional[TileSchedule] = None,
               stats: Optional[KernelStats] = None, dtype: Optional[int] = None):
    """Mirror of tileattn::sdpa_tiled (tiled.cpp:253-272) on HOST arrays.

    q, k, v: numpy float32 arrays [B,H,S,D] whose values lie on the 16-bit
    grid of ``dtype`` (AttnInput, types.hpp:88-104).  Returns a float32 numpy
    array [B,H,S,D] snapped to the dtype grid (tiled.cpp:216-220), computed by
    the sm_100a kernel through ta_sdpa_fwd_host.
    """
    import numpy as np
    import torch
    if dtype is None:
        raise ValueError("dtype (F16 or BF16) is required: the input grid is not inferable")
    tdt = {F16: torch.float16, BF16: torch.bfloat16}.get(dtype)
    if tdt is None:
        # validation order: let the library classify (F32 -> unsupported)
        tdt = torch.float16
    qa = np.ascontiguousarray(q, np.float32)
    shape = qa.shape
    if len(shape) != 4:
        raise ValueError("q must be [B,H,S,D]")
    ht = [torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(tdt).contiguous()
          for x in (q, k, v)]
    o = torch.empty(shape, dtype=tdt)
    sdpa_fwd_host(ht[0].data_ptr(), ht[1].data_ptr(), ht[2].data_ptr(), o.data_ptr(), 0,
                  shape, dtype, mask_kind=mask_kind, valid_len=valid_len, scale=scale,
                  schedule=schedule, stats=stats)
    return o.float().numpy()
