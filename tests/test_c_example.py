"""The C ABI used from plain C99 (examples/check_hexes.c): the header compiles as
C with -Werror and the program links against the in-tree library (CPU); on a
GPU it runs and prints the expected verdicts for both entry points."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1706_01613_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build_example(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    lib = os.path.join(PKG, "libhexval.so")
    if not os.path.exists(lib):
        from paper_1706_01613_b200 import build as hvbuild
        hvbuild.build()
    exe = str(tmp_path / "check_hexes")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "check_hexes.c"),
           "-L", PKG, "-lhexval", f"-Wl,-rpath,{PKG}", "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-o", exe]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return exe


def test_example_compiles_as_c99_and_links(tmp_path):
    build_example(tmp_path)


@pytest.mark.gpu
def test_example_runs_on_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    exe = build_example(tmp_path)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    want = ["VALID", "INVALID", "INVALID", "NONFINITE"]
    host = [l.split(": ")[1].split()[0] for l in out.stdout.splitlines() if l.startswith("host")]
    dev = [l.split(": ")[1].split()[0] for l in out.stdout.splitlines() if l.startswith("device")]
    assert host == want and dev == want, out.stdout


@pytest.mark.gpu
def test_python_mesh_example_runs_on_gpu(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import sys
    sys.path.insert(0, os.path.join(ROOT, "examples"))
    import numpy as np
    import check_mesh
    verts, idx = check_mesh.jittered_grid(20, 0.45, 1)
    np.savez(tmp_path / "m.npz", vertices=verts, hex_idx=idx)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "examples", "check_mesh.py"), str(tmp_path / "m.npz")],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "8000 hexahedra" in out.stdout and "must be 0" in out.stdout
    assert "(on valid ones: 0, must be 0)" in out.stdout
