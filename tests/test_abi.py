"""C-ABI library checks that need no GPU (-m "not gpu").

The library links the CUDA runtime statically, so it loads on a machine
without a GPU; argument validation happens before any CUDA call, so those
paths are testable here.  No compute call is made.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1706_01613_b200 as hv
from paper_1706_01613_b200 import build as hvbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hexval.h")


@pytest.fixture(scope="module")
def L():
    hvbuild.build()
    return hv.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hexval_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    fns = declared_functions()
    assert "hexval_check_soa" in fns and "hexval_check_indexed" in fns
    assert len(fns) >= 10


def test_library_exports_every_declared_symbol(L):
    for name in declared_functions():
        assert hasattr(L, name), name


def test_status_strings(L):
    assert hv.status_string(0) == "ok"
    for code in (-1, -2, -3, -4):
        assert hv.status_string(code) != "unknown status"
    assert hv.version() >= 100
    assert hv.kernel_launches_per_call() == 2            # pass 1 + subdivision (exact path fused)


def test_argument_errors_without_gpu(L):
    buf = (ctypes.c_double * 64)()
    flags = (ctypes.c_uint8 * 64)()
    addr = ctypes.addressof(buf)
    # n < 0, n > INT32_MAX, NULL with n > 0
    assert L.hexval_check_soa(addr, -1, ctypes.addressof(flags), None, None) == -1
    assert L.hexval_check_soa(addr, 2 ** 31, ctypes.addressof(flags), None, None) == -1
    assert L.hexval_check_soa(None, 4, ctypes.addressof(flags), None, None) == -1
    assert L.hexval_check_soa(addr, 4, None, None, None) == -1
    assert L.hexval_check_indexed(addr, None, 4, ctypes.addressof(flags), None, None) == -1
    assert L.hexval_classify_bezier(None, 3, ctypes.addressof(flags), None, None) == -1
    # misaligned double pointer
    assert L.hexval_check_soa(addr + 4, 4, ctypes.addressof(flags), None, None) == -2
    assert L.hexval_check_indexed(addr, addr + 2, 4, ctypes.addressof(flags), None, None) == -2
    # n == 0 is a no-op
    assert L.hexval_check_soa(None, 0, None, None, None) == 0
    assert L.hexval_check_indexed(None, None, 0, None, None, None) == 0
    assert L.hexval_check_soa_host(None, 0, None, None, 0, None) == 0


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    import paper_1706_01613_b200 as pkg
    monkeypatch.setattr(pkg, "_LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(pkg.HexvalError):
        pkg._load()


def test_product_path_never_touches_the_oracle():
    """The CUDA path shares no code with oracle/ and never imports it."""
    pkg = os.path.join(ROOT, "paper_1706_01613_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "oracle.h" not in text and "liboracle" not in text, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".c", ".h", ".py")):
            text = open(os.path.join(ROOT, "oracle", f)).read()
            for bad in ("import paper_1706_01613_b200", "from paper_1706_01613_b200", "hexval_device",
                        "hexval.h", "import hexgen", "from hexgen"):
                assert bad not in text, (f, bad)


def test_binding_validation_without_gpu():
    """The Python binding checks dtype, device and shape before any call (CPU tensors here)."""
    torch = pytest.importorskip("torch")
    with pytest.raises(ValueError):
        hv.check_soa(torch.zeros((24, 4), dtype=torch.float64))           # not CUDA
    with pytest.raises(TypeError):
        hv.check_soa(torch.zeros((24, 4), dtype=torch.float32))           # wrong dtype
    with pytest.raises(ValueError):
        hv.check_indexed(torch.zeros((4, 3), dtype=torch.float64), torch.zeros((4, 8), dtype=torch.int64))
    with pytest.raises(TypeError):
        hv.check_soa([[0.0]])                                            # not a tensor
    with pytest.raises(ValueError):
        hv.check_screen_soa(torch.zeros((24, 4), dtype=torch.float64))    # not CUDA
    with pytest.raises(ValueError):
        hv.check_screen_indexed(torch.zeros((4, 3), dtype=torch.float64), torch.zeros((4, 8), dtype=torch.int32))
    with pytest.raises(TypeError):
        hv.check_soa_host(np.zeros((24, 3), np.float32), np.zeros(3, np.uint8))


def test_host_call_rejects_mis_shaped_buffers_before_any_copy():
    """check_*_host validate every host buffer's shape before the library is called: an
    undersized flags / coeffs array or a wrongly shaped coords / connectivity array would
    otherwise be overrun by the device-to-host copies."""
    coords = np.zeros((24, 10))
    with pytest.raises(ValueError):
        hv.check_soa_host(coords, np.zeros(9, np.uint8))
    with pytest.raises(ValueError):
        hv.check_soa_host(np.zeros((23, 10)), np.zeros(10, np.uint8))
    with pytest.raises(ValueError):
        hv.check_soa_host(coords, np.zeros(10, np.uint8), coeffs=np.zeros((10, 27)))
    with pytest.raises(TypeError):
        hv.check_soa_host(coords, np.zeros(10, np.int32))
    verts, idx = np.zeros((5, 3)), np.zeros((10, 8), np.int32)
    with pytest.raises(ValueError):
        hv.check_indexed_host(verts, np.zeros((10, 4), np.int32), np.zeros(10, np.uint8))
    with pytest.raises(ValueError):
        hv.check_indexed_host(np.zeros((5, 4)), idx, np.zeros(10, np.uint8))
    with pytest.raises(ValueError):
        hv.check_indexed_host(verts, idx, np.zeros(10, np.uint8), coeffs=np.zeros((27, 9)))
