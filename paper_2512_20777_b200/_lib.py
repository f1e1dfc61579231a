"""ctypes binding of libexpmb.so (the C ABI in include/expmb.h).

The library is built in-tree (``make`` or ``__graft_entry__.build()``).  There
is no fallback: if it is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# EXPMB_LIB selects an A/B build of the same library (`make variant`), by file name
LIB_PATH = os.path.join(_HERE, os.path.basename(os.environ.get("EXPMB_LIB", "libexpmb.so")))

EXPMB_F32, EXPMB_F64 = 0, 1
EXPMB_SASTRE, EXPMB_PS, EXPMB_BASELINE = 0, 1, 2

ERR_TOLERANCE = -1
ERR_SHAPE = -2
ERR_SCHEME = -3
ERR_DTYPE = -4
ERR_WORKSPACE = -5
ERR_CUDA = -6
ERR_ALIGN = -7
ERR_UNSUPPORTED = -8

# Every symbol include/expmb.h declares (tests check the .so exports them all).
EXPORTS = (
    "expmb_version",
    "expmb_strerror",
    "expmb_unit_roundoff",
    "expmb_workspace_bytes",
    "expmb_expm",
    "expmb_select",
    "expmb_select_host",
    "expmb_lowrank_workspace_bytes",
    "expmb_expm_lowrank",
    "expmb_select_lowrank_host",
    "expmb_timegrid_workspace_bytes",
    "expmb_expm_timegrid",
    "expmb_expm_pipelined",
)

LR_BAD_INPUT, LR_NONFINITE, LR_NO_ORDER = 1, 2, 4

_lib = None


def lib() -> ctypes.CDLL:
    """Load libexpmb.so once; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the CUDA library first (`make` or "
            "`python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback."
        )
    L = ctypes.CDLL(LIB_PATH)
    c = ctypes
    vp, sz, i32, i64, ci, cd = c.c_void_p, c.c_size_t, c.c_int32, c.c_int64, c.c_int, c.c_double
    dp, ip = c.POINTER(c.c_double), c.POINTER(c.c_int)
    sigs = {
        "expmb_version": (ci, []),
        "expmb_strerror": (c.c_char_p, [ci]),
        "expmb_unit_roundoff": (cd, [ci]),
        "expmb_workspace_bytes": (sz, [i64, i32, ci, ci]),
        "expmb_expm": (ci, [vp, vp, i64, i32, ci, cd, ci] + [vp] * 7 + [vp, sz, vp]),
        "expmb_select": (ci, [vp, i64, i32, ci, cd, ci] + [vp] * 7 + [vp, sz, vp]),
        "expmb_select_host": (ci, [dp, cd, ci, ip, ip, dp, dp]),
        "expmb_lowrank_workspace_bytes": (sz, [i64, i32, i32, ci]),
        "expmb_expm_lowrank": (ci, [vp, vp, vp, i64, i32, i32, ci, cd] + [vp] * 7 + [sz, vp]),
        "expmb_select_lowrank_host": (ci, [dp, ci, cd, ip, dp, dp]),
        "expmb_timegrid_workspace_bytes": (sz, [i64, i32, ci]),
        "expmb_expm_timegrid": (ci, [vp, vp, vp, i64, i32, ci, cd, ci] + [vp] * 7 + [vp, sz, vp]),
        "expmb_expm_pipelined": (ci, [vp, vp, vp, vp, i64, i32, ci, cd, ci] + [vp] * 7 + [ci, vp, sz, vp, vp, vp]),
    }
    ab_build = "EXPMB_LIB" in os.environ  # an A/B build of another revision may lack newer entry points
    for name, (res, args) in sigs.items():
        if not hasattr(L, name):
            if not ab_build:
                raise OSError(f"{LIB_PATH} does not export {name} (stale build? run make)")
            setattr(L, name, None)
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def strerror(code: int) -> str:
    return lib().expmb_strerror(code).decode()


def select_host(norms, eps: float, scheme: int):
    """Run the kernels' selector on the host: returns (m, s, e1, e2, max_power)."""
    L = lib()
    arr = (ctypes.c_double * 4)(*(list(norms) + [float("nan")] * (4 - len(norms))))
    m, s = ctypes.c_int(), ctypes.c_int()
    e1, e2 = ctypes.c_double(), ctypes.c_double()
    have = L.expmb_select_host(arr, float(eps), int(scheme), ctypes.byref(m), ctypes.byref(s),
                               ctypes.byref(e1), ctypes.byref(e2))
    return m.value, s.value, e1.value, e2.value, have


def select_lowrank_host(nv: float, nv2: float | None, eps: float):
    """The low-rank kernel's ladder on the host: (rc, m, e1, e2); rc 0 = chosen,
    1 = ||V^2||_1 needed, -1 = no admissible order."""
    L = lib()
    arr = (ctypes.c_double * 2)(float(nv), float("nan") if nv2 is None else float(nv2))
    m = ctypes.c_int(-1)
    e1, e2 = ctypes.c_double(float("nan")), ctypes.c_double(float("nan"))
    rc = L.expmb_select_lowrank_host(arr, 0 if nv2 is None else 1, float(eps), ctypes.byref(m),
                                     ctypes.byref(e1), ctypes.byref(e2))
    return rc, m.value, e1.value, e2.value
