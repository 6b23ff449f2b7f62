"""ctypes binding of ``libpermatrace_b200.so`` (the C ABI declared in ``include/permatrace_b200.h``).

The library is the only compute path of this package: there is no CPU fallback.  Importing this
module only needs the shared object on disk (so symbol/ABI tests run without a GPU); the first
call that needs a device creates the context and raises ``RuntimeError`` when no B200 is there.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

__all__ = ["lib", "LIB_PATH", "context", "check", "ptr", "PtError", "RangeError", "DECLARED_SYMBOLS"]

# PERMATRACE_B200_LIB: an alternative build of the same library (A/B timing of kernel variants; tests never set it)
LIB_PATH = Path(os.environ.get("PERMATRACE_B200_LIB") or Path(__file__).resolve().parent / "libpermatrace_b200.so")

PT_OK = 0
PT_E_INVALID, PT_E_CUDA, PT_E_RANGE, PT_E_LIMIT, PT_E_NOMEM, PT_E_STATE = -1, -2, -3, -4, -5, -6


class PtError(RuntimeError):
    """Failure reported by libpermatrace_b200 (CUDA error, memory, call sequence)."""


class RangeError(PtError):
    """The lattice window does not fit the packed 64-bit keys."""


if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "or paper_2406_04795_b200/csrc/build.sh -- this package has no CPU fallback"
    )

lib = C.CDLL(str(LIB_PATH))

_vp, _ll, _i, _d = C.c_void_p, C.c_longlong, C.c_int, C.c_double
_pp = C.POINTER(C.c_void_p)


class TraceStats(C.Structure):
    _fields_ = [(k, _ll) for k in ("levels", "seeds", "visited_edges", "field_evaluations",
                                   "dropped_out_of_box", "candidates", "frontier")] + \
               [("complete", _i), ("closure_ok", _i)] + \
               [(k, _ll) for k in ("table_capacity", "sign_table_capacity", "n_stages", "ambiguous_signs")]


class RefineStats(C.Structure):
    _fields_ = [(k, _ll) for k in ("cells", "fine_vertices", "crossing_edges", "unique_fine_vertices",
                                   "unique_fine_edges", "points", "in_collision", "free_points",
                                   "dedup_rounds", "field_evaluations", "ambiguous_signs")]


_SIGS = {
    "pt_last_error": (C.c_char_p, []),
    "pt_version": (_i, []),
    "pt_ctx_create": (_i, [_i, _pp]),
    "pt_ctx_destroy": (None, [_vp]),
    "pt_ctx_set_stream": (_i, [_vp, _vp]),
    "pt_ctx_synchronize": (_i, [_vp]),
    "pt_ctx_trim": (_ll, [_vp]),
    "pt_host_alloc": (_vp, [_vp, _ll]),
    "pt_host_free": (None, [_vp, _vp]),
    "pt_ctx_profile_enable": (_i, [_vp, _i]),
    "pt_ctx_profile_reset": (_i, [_vp]),
    "pt_ctx_profile_dump": (_ll, [_vp, C.c_char_p, _ll]),
    "pt_ctx_launch_count": (_ll, [_vp]),
    "pt_ctx_work_counters": (_i, [_vp, _vp, _i]),
    "pt_ctx_retry_evaluations": (C.c_longlong, [_vp]),
    "pt_ctx_taylor_rows": (C.c_longlong, [_vp]),
    "pt_peak_fp64": (_d, [_vp]),
    "pt_peak_ex2": (_d, [_vp]),
    "pt_rbf_values": (_i, [_vp, _vp, _ll, _i, _vp, _ll, _vp, _d, _d, _vp]),
    "pt_sphere_box_hits": (_i, [_vp, _vp, _vp, _ll, _d, _d, _d, _vp]),
    "pt_sphere_cylinder_hits": (_i, [_vp, _vp, _vp, _ll, _d, _d, _vp]),
    "pt_sphere_sphere_hits": (_i, [_vp, _vp, _vp, _ll, _d, _vp]),
    "pt_field_create_rbf": (_i, [_vp, _i, _ll, _vp, _vp, _d, _d, _vp, _pp]),
    "pt_field_create_analytic": (_i, [_vp, _i, _i, _vp, _pp]),
    "pt_field_destroy": (None, [_vp]),
    "pt_field_set_precision": (_i, [_vp, _i]),
    "pt_field_values": (_i, [_vp, _vp, _vp, _ll, _vp, _vp]),
    "pt_field_gradients": (_i, [_vp, _vp, _vp, _ll, _vp]),
    "pt_intersection_points": (_i, [_vp, _vp, _vp, _vp, _ll, _d, _vp, _vp]),
    "pt_debug_tc_arg_error": (_i, [_vp, _vp, _vp, _vp, _ll, _vp]),
    "pt_checker_create": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _pp]),
    "pt_checker_destroy": (None, [_vp]),
    "pt_fk_batch": (_i, [_vp, _vp, _vp, _ll, _vp]),
    "pt_batch_check": (_i, [_vp, _vp, _vp, _ll, _i, _vp, C.POINTER(_ll)]),
    "pt_trace_create": (_i, [_vp, _vp, _i, _d, _vp, _vp, _vp, _ll, _d, _pp]),
    "pt_trace_destroy": (None, [_vp]),
    "pt_trace_locate": (_i, [_vp, _vp, _ll]),
    "pt_trace_expand": (_i, [_vp, C.POINTER(_ll)]),
    "pt_trace_run": (_i, [_vp, _vp, _ll]),
    "pt_trace_seed_edges": (_i, [_vp, _vp, _vp, _ll, _ll]),
    "pt_trace_get_stats": (_i, [_vp, C.POINTER(TraceStats)]),
    "pt_trace_stages": (_i, [_vp, _vp, _ll]),
    "pt_trace_edges": (_i, [_vp, _ll, _ll, _vp, _vp, _vp]),
    "pt_trace_frontier": (_i, [_vp, C.POINTER(_ll), C.POINTER(_ll)]),
    "pt_trace_points": (_i, [_vp, _vp]),
    "pt_trace_adjacency": (_ll, [_vp, _vp, _ll]),
    "pt_trace_shard": (_i, [_vp, _i, _i]),
    "pt_trace_wave_candidates": (_i, [_vp, _vp]),
    "pt_trace_wave_fetch": (_i, [_vp, _vp]),
    "pt_trace_wave_admit": (_i, [_vp, _vp, _ll, C.POINTER(_ll)]),
    "pt_trace_wave_winner_tags": (_i, [_vp, _vp]),
    "pt_trace_wave_commit": (_i, [_vp, _vp, _ll, _ll]),
    "pt_trace_gidx": (_i, [_vp, _ll, _ll, _vp]),
    "pt_cells_from_trace": (_i, [_vp, _pp]),
    "pt_cells_from_edges": (_i, [_vp, _i, _vp, _vp, _ll, _pp]),
    "pt_cells_from_host": (_i, [_vp, _i, _vp, _vp, _ll, _pp]),
    "pt_cells_slice": (_i, [_vp, _ll, _ll, _pp]),
    "pt_cells_keys": (_i, [_vp, _ll, _ll, _vp]),
    "pt_cells_merge_keys": (_i, [_vp, _vp, _ll, _pp]),
    "pt_cells_destroy": (None, [_vp]),
    "pt_cells_count": (_ll, [_vp]),
    "pt_cells_get": (_i, [_vp, _ll, _ll, _vp, _vp]),
    "pt_refine_run": (_i, [_vp, _vp, _vp, _i, _d, _vp, _i, _i, _vp, _i, _vp, _d, _d, _vp, _vp, _i, _pp]),
    "pt_refine_candidates": (_i, [_vp, _vp, _vp, _i, _d, _vp, _i, _i, _vp, _i, _vp, _d, _pp]),
    "pt_dedup_label": (_i, [_vp, _i, _vp, _ll, _d, _vp, _pp]),
    "pt_dedup_label_forced": (_i, [_vp, _i, _vp, _ll, _d, _vp, _vp, _pp]),
    "pt_refine_destroy": (None, [_vp]),
    "pt_refine_get_stats": (_i, [_vp, C.POINTER(RefineStats)]),
    "pt_refine_points": (_i, [_vp, _vp, _vp, _vp]),
    "pt_refine_batch_stats": (_i, [_vp, _vp, _i]),
    "pt_refine_set_labels": (_i, [_vp, _vp]),
    "pt_host_expansion_plan": (_i, [_i, C.c_uint32, _vp, _i]),
    "pt_host_cellcofaces": (_i, [_i, C.c_uint32, _vp, _i]),
    "pt_host_perm_rank": (_i, [_i, _vp]),
    "pt_host_perm_unrank": (_i, [_i, _i, _vp]),
}

DECLARED_SYMBOLS = tuple(sorted(_SIGS))

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)   # AttributeError here == a declared symbol is not exported
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    return (lib.pt_last_error() or b"").decode("utf-8", "replace")


def check(rc: int):
    """Map a C return code onto the reference's exception types."""
    if rc == PT_OK:
        return
    msg = last_error()
    if rc == PT_E_INVALID:
        raise ValueError(msg)
    if rc == PT_E_RANGE:
        raise RangeError(msg)
    if rc == PT_E_LIMIT:
        from .collision import LimitError
        raise LimitError(msg)
    if rc == PT_E_NOMEM:
        raise MemoryError(msg)
    raise PtError(msg)


def ptr(a):
    """Raw address of a numpy array / torch tensor / int / None."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(f"cannot take the address of {type(a).__name__}")


class _Context:
    """One library context per (process, device); created on first use."""

    def __init__(self, device: int):
        h = C.c_void_p()
        rc = lib.pt_ctx_create(device, C.byref(h))
        if rc != PT_OK:
            raise PtError(
                "libpermatrace_b200 could not create a CUDA context: " + last_error()
            )
        self.handle = h
        self.device = device

    def set_stream(self, stream_handle: int | None):
        check(lib.pt_ctx_set_stream(self.handle, C.c_void_p(stream_handle or 0)))

    def synchronize(self):
        check(lib.pt_ctx_synchronize(self.handle))

    def trim(self) -> int:
        """Return the context's cached device blocks to the driver; bytes released."""
        return int(lib.pt_ctx_trim(self.handle))

    def profile(self, on: bool):
        check(lib.pt_ctx_profile_enable(self.handle, 1 if on else 0))

    def profile_reset(self):
        check(lib.pt_ctx_profile_reset(self.handle))

    def profile_dump(self) -> dict[str, tuple[int, float]]:
        need = lib.pt_ctx_profile_dump(self.handle, None, 0)
        buf = C.create_string_buffer(int(need) + 16)
        lib.pt_ctx_profile_dump(self.handle, buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            name, launches, ms = line.rsplit(",", 2)
            out[name] = (int(launches), float(ms))
        return out

    def launch_count(self) -> int:
        return int(lib.pt_ctx_launch_count(self.handle))


class _PinnedBlock:
    """Owner of one page-locked host block; numpy arrays built on it keep it alive through `base`."""

    def __init__(self, ctx, nbytes: int, shape, dtype):
        self._ctx = ctx
        self._ptr = lib.pt_host_alloc(ctx.handle, max(int(nbytes), 1))
        if not self._ptr:
            raise MemoryError("pinned host allocation failed: " + last_error())
        dt = np.dtype(dtype)
        self.__array_interface__ = {"shape": tuple(int(v) for v in shape), "typestr": dt.str, "data": (int(self._ptr), False),
                                    "version": 3}

    def __del__(self):
        p, self._ptr = getattr(self, "_ptr", None), None
        if p:
            try:
                lib.pt_host_free(self._ctx.handle, p)
            except Exception:
                pass


def pinned_empty(shape, dtype=np.float64, ctx=None) -> np.ndarray:
    """Uninitialised numpy array in page-locked memory (for large device->host results)."""
    if isinstance(shape, int):
        shape = (shape,)
    ctx = ctx or context()
    nbytes = int(np.prod(shape, dtype=np.int64)) * np.dtype(dtype).itemsize
    return np.asarray(_PinnedBlock(ctx, nbytes, shape, dtype))


_lock = threading.Lock()
_contexts: dict[int, _Context] = {}


def context(device: int | None = None) -> _Context:
    if device is None:
        device = int(os.environ.get("PERMATRACE_B200_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    with _lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = _Context(device)
            _contexts[device] = ctx
        return ctx
