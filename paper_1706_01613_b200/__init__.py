"""B200-native hot path of the robust validity check of linear hexahedra.

Johnen, Weill, Remacle, "Robust and efficient validation of the linear
hexahedral element" (IMR26 2017; /root/reference/PAPER.md).  Every step of the
path runs in the hand-written sm_100a kernels of ``libhexval.so`` behind the C
ABI declared in ``include/hexval.h``; this module only marshals arguments
(ctypes) and uses PyTorch for device memory and streams.  There is no CPU
fallback: importing the package fails loudly when the library is missing.

Entry points mirror the C names:

* :func:`check_soa` / :func:`check_indexed`           device tensors, async
* :func:`check_soa_host` / :func:`check_indexed_host` host arrays, end to end
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = [
    "INVALID", "VALID", "UNDETERMINED", "NONFINITE", "FLAG_SUBDIVIDED", "MAX_DEPTH",
    "HexvalError", "lib", "library_path", "check_soa", "check_indexed", "check_soa_host",
    "check_indexed_host", "classify_bezier", "Stats", "Profile", "status_string", "version",
    "kernel_launches_per_call", "corner_quality_soa", "corner_quality_indexed", "min_detj_bounds_soa",
    "min_detj_bounds_indexed", "select_valid", "check_quad_soa", "check_screen_soa", "check_screen_indexed",
    "fp64_peak", "scratch_info", "scratch_release",
]

INVALID, VALID, UNDETERMINED, NONFINITE = 0, 1, 2, 3
FLAG_SUBDIVIDED = 4
MAX_DEPTH = 20
PHASES = ("pass1", "exact", "subdiv")          # "exact" is fused into "subdiv" (reads 0)

_HERE = os.path.dirname(os.path.abspath(__file__))
# HEXVAL_LIB selects an in-tree variant build (A/B measurements); default libhexval.so
_LIB_PATH = os.path.join(_HERE, os.environ.get("HEXVAL_LIB", "libhexval.so"))


class HexvalError(RuntimeError):
    pass


def library_path() -> str:
    return _LIB_PATH


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64


def _load() -> ctypes.CDLL:
    if not os.path.exists(_LIB_PATH):
        raise HexvalError(
            f"{_LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(_LIB_PATH)
    L.hexval_check_soa.argtypes = [_vp, _i64, _vp, _vp, _vp]
    L.hexval_check_indexed.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp]
    L.hexval_check_soa_ex.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp]
    L.hexval_check_indexed_ex.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _vp]
    L.hexval_classify_bezier.argtypes = [_vp, _i64, _vp, _vp, _vp]
    L.hexval_check_soa_host.argtypes = [_vp, _i64, _vp, _vp, _i64, _vp]
    L.hexval_check_indexed_host.argtypes = [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _vp]
    for f in ("hexval_classify_bezier", "hexval_check_soa", "hexval_check_indexed", "hexval_check_soa_ex", "hexval_check_indexed_ex",
              "hexval_check_soa_host", "hexval_check_indexed_host", "hexval_version",
              "hexval_kernel_launches_per_call"):
        getattr(L, f).restype = ctypes.c_int
    L.hexval_corner_quality_soa.argtypes = [_vp, _i64, _vp, _vp, _vp]
    L.hexval_corner_quality_indexed.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp]
    L.hexval_corner_quality_soa.restype = ctypes.c_int
    L.hexval_corner_quality_indexed.restype = ctypes.c_int
    L.hexval_check_screen_soa.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp]
    L.hexval_check_screen_indexed.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp, _vp]
    L.hexval_check_screen_soa.restype = ctypes.c_int
    L.hexval_check_screen_indexed.restype = ctypes.c_int
    L.hexval_min_detj_bounds_soa.argtypes = [_vp, _i64, ctypes.c_double, _vp, _vp, _vp, _vp, _vp]
    L.hexval_min_detj_bounds_indexed.argtypes = [_vp, _vp, _i64, ctypes.c_double, _vp, _vp, _vp, _vp, _vp]
    L.hexval_min_detj_bounds_soa.restype = ctypes.c_int
    L.hexval_min_detj_bounds_indexed.restype = ctypes.c_int
    L.hexval_select_valid.argtypes = [_vp, _i64, _vp, _i64, _vp, _vp, _vp, _vp]
    L.hexval_select_valid.restype = ctypes.c_int
    L.hexval_check_quad_soa.argtypes = [_vp, _i64, _vp, _vp, _vp]
    L.hexval_check_quad_soa.restype = ctypes.c_int
    L.hexval_scratch_info.argtypes = [ctypes.c_int, _vp, _vp]
    L.hexval_scratch_info.restype = ctypes.c_int
    L.hexval_scratch_release.argtypes = []
    L.hexval_scratch_release.restype = ctypes.c_int
    L.hexval_diag_fp64_peak.argtypes = [ctypes.c_int, _vp, _vp, _vp]
    L.hexval_diag_fp64_peak.restype = ctypes.c_int
    L.hexval_status_string.argtypes = [ctypes.c_int]
    L.hexval_status_string.restype = ctypes.c_char_p
    L.hexval_profile_create.argtypes = []
    L.hexval_profile_create.restype = _vp
    L.hexval_profile_destroy.argtypes = [_vp]
    L.hexval_profile_destroy.restype = None
    L.hexval_profile_read.argtypes = [_vp, _vp, _vp]
    L.hexval_profile_read.restype = ctypes.c_int
    return L


_lib: ctypes.CDLL | None = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def status_string(code: int) -> str:
    return lib().hexval_status_string(int(code)).decode()


def version() -> int:
    return lib().hexval_version()


def kernel_launches_per_call() -> int:
    return lib().hexval_kernel_launches_per_call()


def scratch_info(device: int | None = None) -> dict:
    """hexval_scratch_info: bytes reserved by the library's scratch arenas on `device` and their number."""
    if device is None:
        device = _torch().cuda.current_device()
    b = ctypes.c_size_t()
    c = ctypes.c_int()
    _check(lib().hexval_scratch_info(int(device), ctypes.byref(b), ctypes.byref(c)), "hexval_scratch_info")
    return {"bytes": b.value, "arenas": c.value}


def scratch_release() -> None:
    """hexval_scratch_release: free the idle scratch arenas of the current device."""
    _check(lib().hexval_scratch_release(), "hexval_scratch_release")


def fp64_peak(iters: int = 4096, stream=None) -> dict:
    """hexval_diag_fp64_peak: measured DFMA lane-instructions/s of the current device (roofline
    denominator of the FP64-bound kernels).  Synchronises the stream."""
    rate = ctypes.c_double()
    ms = ctypes.c_float()
    _check(lib().hexval_diag_fp64_peak(int(iters), ctypes.byref(rate), ctypes.byref(ms), _stream_handle(stream)),
           "hexval_diag_fp64_peak")
    return {"dfma_per_s": rate.value, "best_ms": ms.value}


def _check(code: int, what: str) -> None:
    if code != 0:
        raise HexvalError(f"{what} failed: {code} ({status_string(code)})")


def _torch():
    import torch
    return torch


def _stream_handle(stream) -> int:
    torch = _torch()
    if stream is None:
        # the current stream of the current device, as torch.cuda.current_stream()
        # gives it, without building a Stream object (3 us -> 0.3 us per call)
        raw, dev = getattr(torch._C, "_cuda_getCurrentRawStream", None), getattr(torch._C, "_cuda_getDevice", None)
        if raw is not None and dev is not None:
            return int(raw(dev()))
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


def _require(t, dtype, name: str, ndim: int | None = None, shape: tuple | None = None):
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (use check_*_host for host memory)")
    cur = getattr(torch._C, "_cuda_getDevice", None)
    if t.device.index != (cur() if cur is not None else torch.cuda.current_device()):
        # the library launches on the current device and stream: make them the tensor's
        raise ValueError(f"{name} is on {t.device}, the current device is cuda:{torch.cuda.current_device()} "
                         f"(call under torch.cuda.device({t.device}))")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must have {ndim} dims")
    if shape is not None and tuple(t.shape) != tuple(shape):
        # the kernels write exactly this many elements: a smaller buffer would be overrun
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


def _soa_input(coords, planes: int = 24) -> int:
    torch = _torch()
    _require(coords, torch.float64, "coords", 2)
    if coords.shape[0] != planes:
        raise ValueError(f"coords must have shape ({planes}, n)")
    return coords.shape[1]


def _indexed_inputs(vertices, hex_idx) -> int:
    """(nv, 3) float64 vertices and (n, 8) int32 connectivity on the current device; returns n."""
    torch = _torch()
    _require(vertices, torch.float64, "vertices", 2)
    _require(hex_idx, torch.int32, "hex_idx", 2)
    if vertices.shape[1] != 3 or hex_idx.shape[1] != 8:
        raise ValueError("vertices must be (nv, 3) and hex_idx (n, 8)")
    return hex_idx.shape[0]


class Stats:
    """Device-side counters (``hexval_stats``) accumulated by the *_ex calls."""

    FIELDS = ("n_valid", "n_invalid", "n_undetermined", "n_nonfinite", "n_subdivided",
              "n_exact", "n_nodes", "max_depth", "n_lane_steps")

    def __init__(self, device=None):
        torch = _torch()
        self.buf = torch.zeros(len(self.FIELDS), dtype=torch.int64,
                               device=device if device is not None else "cuda")

    def zero_(self):
        self.buf.zero_()
        return self

    def ptr(self) -> int:
        return self.buf.data_ptr()

    def read(self) -> dict:
        vals = self.buf.cpu().tolist()
        return dict(zip(self.FIELDS, vals))


class Profile:
    """Per-phase kernel times recorded with CUDA events on the call's stream."""

    def __init__(self):
        self.h = lib().hexval_profile_create()
        if not self.h:
            raise HexvalError("hexval_profile_create failed")

    def read(self) -> dict:
        ms = (ctypes.c_double * 3)()
        cnt = (ctypes.c_longlong * 3)()
        _check(lib().hexval_profile_read(self.h, ms, cnt), "hexval_profile_read")
        return {p: {"ms": ms[k], "launches": cnt[k]} for k, p in enumerate(PHASES)}

    def close(self):
        if self.h:
            lib().hexval_profile_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def check_soa(coords, flags=None, coeffs=None, stats: Stats | None = None,
              profile: Profile | None = None, stream=None):
    """hexval_check_soa(_ex): coords is a (24, n) float64 CUDA tensor (plane p = 3*node + axis).

    Returns ``(flags, coeffs)``; ``coeffs`` is a (27, n) tensor when ``coeffs``
    is True or a preallocated tensor, else None.  Asynchronous on ``stream``
    (default: torch's current stream).
    """
    torch = _torch()
    n = _soa_input(coords)
    if flags is None:
        flags = torch.empty(n, dtype=torch.uint8, device=coords.device)
    _require(flags, torch.uint8, "flags", shape=(n,))
    if coeffs is True:
        coeffs = torch.empty((27, n), dtype=torch.float64, device=coords.device)
    elif coeffs is False:
        coeffs = None
    if coeffs is not None:
        _require(coeffs, torch.float64, "coeffs", shape=(27, n))
    rc = lib().hexval_check_soa_ex(coords.data_ptr(), n, flags.data_ptr(),
                                   coeffs.data_ptr() if coeffs is not None else None,
                                   stats.ptr() if stats is not None else None,
                                   profile.h if profile is not None else None,
                                   _stream_handle(stream))
    _check(rc, "hexval_check_soa")
    return flags, coeffs


def check_indexed(vertices, hex_idx, flags=None, coeffs=None, stats: Stats | None = None,
                  profile: Profile | None = None, stream=None):
    """hexval_check_indexed(_ex): vertices (nv, 3) float64, hex_idx (n, 8) int32, CUDA tensors."""
    torch = _torch()
    n = _indexed_inputs(vertices, hex_idx)
    if flags is None:
        flags = torch.empty(n, dtype=torch.uint8, device=hex_idx.device)
    _require(flags, torch.uint8, "flags", shape=(n,))
    if coeffs is True:
        coeffs = torch.empty((27, n), dtype=torch.float64, device=hex_idx.device)
    elif coeffs is False:
        coeffs = None
    if coeffs is not None:
        _require(coeffs, torch.float64, "coeffs", shape=(27, n))
    rc = lib().hexval_check_indexed_ex(vertices.data_ptr(), hex_idx.data_ptr(), n, flags.data_ptr(),
                                       coeffs.data_ptr() if coeffs is not None else None,
                                       stats.ptr() if stats is not None else None,
                                       profile.h if profile is not None else None,
                                       _stream_handle(stream))
    _check(rc, "hexval_check_indexed")
    return flags, coeffs


def classify_bezier(coeffs, flags=None, stats: Stats | None = None, stream=None):
    """hexval_classify_bezier: Steps 4-5 on a (27, n) float64 CUDA tensor of Bezier coefficients."""
    torch = _torch()
    _require(coeffs, torch.float64, "coeffs", 2)
    if coeffs.shape[0] != 27:
        raise ValueError("coeffs must have shape (27, n)")
    n = coeffs.shape[1]
    if flags is None:
        flags = torch.empty(n, dtype=torch.uint8, device=coeffs.device)
    _require(flags, torch.uint8, "flags", shape=(n,))
    rc = lib().hexval_classify_bezier(coeffs.data_ptr(), n, flags.data_ptr(),
                                      stats.ptr() if stats is not None else None, _stream_handle(stream))
    _check(rc, "hexval_classify_bezier")
    return flags


def _host_array(a, dtype, name, shape=None):
    """numpy array or (pinned) CPU tensor -> (pointer, keepalive); `shape` (None entries: any)."""
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags["C_CONTIGUOUS"]:
            raise TypeError(f"{name} must be a C-contiguous {dtype} array")
        ptr = a.ctypes.data
    else:
        torch = _torch()
        if not isinstance(a, torch.Tensor):
            raise TypeError(f"{name}: unsupported type {type(a)}")
        if a.is_cuda or not a.is_contiguous():
            raise TypeError(f"{name} must be a contiguous CPU tensor")
        if a.element_size() != np.dtype(dtype).itemsize or a.dtype.is_floating_point != (np.dtype(dtype).kind == "f"):
            raise TypeError(f"{name} must hold {np.dtype(dtype)} elements")
        ptr = a.data_ptr()
    if shape is not None:
        got = tuple(a.shape)
        if len(got) != len(shape) or any(w is not None and g != w for g, w in zip(got, shape)):
            raise ValueError(f"{name} must have shape {shape}, got {got}")
    return ptr, a


def check_soa_host(coords, flags, coeffs=None, chunk_hexes: int = 0, stream=None):
    """hexval_check_soa_host: host (24, n) float64 in, host flags (and coeffs) out; synchronous."""
    cp, _k1 = _host_array(coords, np.float64, "coords", (24, None))
    n = coords.shape[1]
    fp, _k2 = _host_array(flags, np.uint8, "flags", (n,))
    kp = None
    if coeffs is not None:
        kp, _k3 = _host_array(coeffs, np.float64, "coeffs", (27, n))
    rc = lib().hexval_check_soa_host(cp, n, fp, kp, int(chunk_hexes),
                                     _stream_handle(stream) if stream is not None else 0)
    _check(rc, "hexval_check_soa_host")
    return flags


def check_indexed_host(vertices, hex_idx, flags, coeffs=None, chunk_hexes: int = 0, stream=None):
    vp, _k1 = _host_array(vertices, np.float64, "vertices", (None, 3))
    ip, _k2 = _host_array(hex_idx, np.int32, "hex_idx", (None, 8))
    nv = vertices.shape[0]
    n = hex_idx.shape[0]
    fp, _k3 = _host_array(flags, np.uint8, "flags", (n,))
    kp = None
    if coeffs is not None:
        kp, _k4 = _host_array(coeffs, np.float64, "coeffs", (27, n))
    rc = lib().hexval_check_indexed_host(vp, nv, ip, n, fp, kp, int(chunk_hexes),
                                         _stream_handle(stream) if stream is not None else 0)
    _check(rc, "hexval_check_indexed_host")
    return flags


def _quality_outputs(n, device, sj_min, test1):
    torch = _torch()
    if sj_min is None or sj_min is True:
        sj_min = torch.empty(n, dtype=torch.float64, device=device)
    if test1 is None or test1 is True:
        test1 = torch.empty(n, dtype=torch.uint8, device=device)
    _require(sj_min, torch.float64, "sj_min", shape=(n,))
    _require(test1, torch.uint8, "test1", shape=(n,))
    return sj_min, test1


def corner_quality_soa(coords, sj_min=None, test1=None, stream=None):
    """hexval_corner_quality_soa (NEXT-2): min corner scaled Jacobian and Ushakova Test 1 per hex."""
    n = _soa_input(coords)
    sj_min, test1 = _quality_outputs(n, coords.device, sj_min, test1)
    _check(lib().hexval_corner_quality_soa(coords.data_ptr(), n, sj_min.data_ptr(), test1.data_ptr(),
                                           _stream_handle(stream)), "hexval_corner_quality_soa")
    return sj_min, test1


def corner_quality_indexed(vertices, hex_idx, sj_min=None, test1=None, stream=None):
    """hexval_corner_quality_indexed (NEXT-2) on (nv, 3) float64 vertices and (n, 8) int32 connectivity."""
    n = _indexed_inputs(vertices, hex_idx)
    sj_min, test1 = _quality_outputs(n, hex_idx.device, sj_min, test1)
    _check(lib().hexval_corner_quality_indexed(vertices.data_ptr(), hex_idx.data_ptr(), n, sj_min.data_ptr(),
                                               test1.data_ptr(), _stream_handle(stream)),
           "hexval_corner_quality_indexed")
    return sj_min, test1


def check_screen_soa(coords, flags=None, sj_min=None, test1=None, stream=None):
    """hexval_check_screen_soa: validity flags plus the NEXT-2 screening outputs in one pass.

    Returns ``(flags, sj_min, test1)``, bit-identical to ``check_soa`` and ``corner_quality_soa``."""
    torch = _torch()
    n = _soa_input(coords)
    if flags is None:
        flags = torch.empty(n, dtype=torch.uint8, device=coords.device)
    _require(flags, torch.uint8, "flags", shape=(n,))
    sj_min, test1 = _quality_outputs(n, coords.device, sj_min, test1)
    _check(lib().hexval_check_screen_soa(coords.data_ptr(), n, flags.data_ptr(), sj_min.data_ptr(),
                                         test1.data_ptr(), _stream_handle(stream)), "hexval_check_screen_soa")
    return flags, sj_min, test1


def check_screen_indexed(vertices, hex_idx, flags=None, sj_min=None, test1=None, stream=None):
    """hexval_check_screen_indexed: ``check_indexed`` and ``corner_quality_indexed`` in one pass."""
    torch = _torch()
    n = _indexed_inputs(vertices, hex_idx)
    if flags is None:
        flags = torch.empty(n, dtype=torch.uint8, device=hex_idx.device)
    _require(flags, torch.uint8, "flags", shape=(n,))
    sj_min, test1 = _quality_outputs(n, hex_idx.device, sj_min, test1)
    _check(lib().hexval_check_screen_indexed(vertices.data_ptr(), hex_idx.data_ptr(), n, flags.data_ptr(),
                                             sj_min.data_ptr(), test1.data_ptr(), _stream_handle(stream)),
           "hexval_check_screen_indexed")
    return flags, sj_min, test1


def _bounds_outputs(n, device, lower, upper, status):
    torch = _torch()
    lower = torch.empty(n, dtype=torch.float64, device=device) if lower is None else lower
    upper = torch.empty(n, dtype=torch.float64, device=device) if upper is None else upper
    status = torch.empty(n, dtype=torch.uint8, device=device) if status is None else status
    _require(lower, torch.float64, "lower", shape=(n,))
    _require(upper, torch.float64, "upper", shape=(n,))
    _require(status, torch.uint8, "status", shape=(n,))
    return lower, upper, status


def _nodes_counter(nodes):
    if nodes is None:
        return None
    torch = _torch()
    _require(nodes, torch.int64, "nodes")
    if nodes.numel() < 1:
        raise ValueError("nodes must hold at least one int64")
    return nodes.data_ptr()


def min_detj_bounds_soa(coords, rel_tol: float, lower=None, upper=None, status=None, nodes=None, stream=None):
    """hexval_min_detj_bounds_soa (NEXT-1): certified [lower, upper] on min det J per hex.

    ``nodes``: optional int64 CUDA tensor of one element to which the split count is added."""
    n = _soa_input(coords)
    lower, upper, status = _bounds_outputs(n, coords.device, lower, upper, status)
    _check(lib().hexval_min_detj_bounds_soa(coords.data_ptr(), n, float(rel_tol), lower.data_ptr(), upper.data_ptr(),
                                            status.data_ptr(), _nodes_counter(nodes),
                                            _stream_handle(stream)), "hexval_min_detj_bounds_soa")
    return lower, upper, status


def min_detj_bounds_indexed(vertices, hex_idx, rel_tol: float, lower=None, upper=None, status=None, nodes=None,
                            stream=None):
    n = _indexed_inputs(vertices, hex_idx)
    lower, upper, status = _bounds_outputs(n, hex_idx.device, lower, upper, status)
    _check(lib().hexval_min_detj_bounds_indexed(vertices.data_ptr(), hex_idx.data_ptr(), n, float(rel_tol),
                                                lower.data_ptr(), upper.data_ptr(), status.data_ptr(),
                                                _nodes_counter(nodes),
                                                _stream_handle(stream)), "hexval_min_detj_bounds_indexed")
    return lower, upper, status


def select_valid(flags, group=None, n_groups: int = 0, ids=None, group_counts=None, stream=None):
    """hexval_select_valid (NEXT-3): returns (ids[:count], count, group_counts).

    ``count`` is read back to the host (one 8-byte D2H copy) to size the ids view."""
    torch = _torch()
    _require(flags, torch.uint8, "flags", 1)
    n = flags.numel()
    if ids is None:
        ids = torch.empty(n, dtype=torch.int32, device=flags.device)
    _require(ids, torch.int32, "ids", shape=(n,))
    count = torch.zeros(1, dtype=torch.int64, device=flags.device)
    if group is not None:
        _require(group, torch.int32, "group", shape=(n,))
        if group_counts is None:
            group_counts = torch.zeros(n_groups, dtype=torch.int32, device=flags.device)
        _require(group_counts, torch.int32, "group_counts", shape=(int(n_groups),))
    _check(lib().hexval_select_valid(flags.data_ptr(), n, group.data_ptr() if group is not None else None,
                                     int(n_groups), ids.data_ptr(), count.data_ptr(),
                                     group_counts.data_ptr() if group is not None else None,
                                     _stream_handle(stream)), "hexval_select_valid")
    c = int(count.item())
    return ids[:c], c, group_counts


def check_quad_soa(coords, flags=None, J=None, stream=None):
    """hexval_check_quad_soa (NEXT-4): coords is an (8, n) float64 CUDA tensor (plane 2k + a).

    Returns ``(flags, J)``; ``J`` is a (4, n) tensor of corner values when requested."""
    torch = _torch()
    n = _soa_input(coords, 8)
    if flags is None:
        flags = torch.empty(n, dtype=torch.uint8, device=coords.device)
    _require(flags, torch.uint8, "flags", shape=(n,))
    if J is True:
        J = torch.empty((4, n), dtype=torch.float64, device=coords.device)
    elif J is False:
        J = None
    if J is not None:
        _require(J, torch.float64, "J", shape=(4, n))
    _check(lib().hexval_check_quad_soa(coords.data_ptr(), n, flags.data_ptr(), J.data_ptr() if J is not None else None,
                                       _stream_handle(stream)), "hexval_check_quad_soa")
    return flags, J
