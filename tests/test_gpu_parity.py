"""Parity of the CUDA path (through the C ABI) with the CPU oracle (-m gpu).

Flags must match bit for bit on every hex the oracle does not mark
near-boundary (and configs 0-3 must have no near-boundary hexes).  Bezier
coefficients must match within 1e-12 * max|b| of the hex (BASELINE.json
north_star).  Full-size configs run on the GPU in the same launch
configuration bench.py times; the oracle checks a sample of the outputs
(random hexes plus every hex that took the exact-sign or subdivision path)
and, for config 4, the closed-form verdict of every hex.
"""
import functools
import os

import numpy as np
import pytest

import hexgen
import oracle
from tests import pins

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1706_01613_b200 as hv  # noqa: E402

COEFF_TOL = 1e-12


@functools.lru_cache(maxsize=None)
def full_config(cfg: int):
    """hexgen.make(cfg), generated once per session (configs 1-3 take seconds to tens of
    seconds on the host); callers must not modify the arrays."""
    return hexgen.make(cfg)


def gpu_soa(coords: np.ndarray, coeffs=False, stats=None):
    dev = torch.from_numpy(np.ascontiguousarray(coords)).cuda()
    f, k = hv.check_soa(dev, coeffs=coeffs, stats=stats)
    torch.cuda.synchronize()
    return f.cpu().numpy(), (k.cpu().numpy() if k is not None else None)


def gpu_indexed(verts: np.ndarray, idx: np.ndarray, coeffs=False, stats=None):
    v = torch.from_numpy(np.ascontiguousarray(verts)).cuda()
    i = torch.from_numpy(np.ascontiguousarray(idx)).cuda()
    f, k = hv.check_indexed(v, i, coeffs=coeffs, stats=stats)
    torch.cuda.synchronize()
    return f.cpu().numpy(), (k.cpu().numpy() if k is not None else None)


def assert_flags_match(gpu_flags, ref, allow_near=False):
    near = ref["near"].astype(bool)
    if not allow_near:
        assert near.sum() == 0, f"{near.sum()} near-boundary hexes"
    bad = np.nonzero((gpu_flags != ref["flags"]) & ~near)[0]
    assert bad.size == 0, (f"{bad.size} flag mismatches, first {bad[:10]}: "
                           f"gpu {gpu_flags[bad[:10]]} oracle {ref['flags'][bad[:10]]}")


def assert_coeffs_match(gpu_coeffs, ref_coeffs, flags):
    ok = (flags & 3) != hv.NONFINITE
    scale = np.max(np.abs(ref_coeffs), axis=0)
    err = np.max(np.abs(gpu_coeffs - ref_coeffs), axis=0)
    bad = np.nonzero(ok & (err > COEFF_TOL * scale))[0]
    assert bad.size == 0, f"{bad.size} coefficient mismatches; worst rel {np.max(err[ok] / scale[ok])}"


# --------------------------------------------------------------------------
# paper examples and closed forms through the C ABI
# --------------------------------------------------------------------------

def test_root_emulation_is_bit_exact():
    """tests/gpu_emulation.py (the CPU emulation the tau pins of tests/test_tau_bounds.py use
    for the CUDA path's values) reproduces the kernels' 27 root coefficients bit for bit:
    random, high-noise, degenerate, 2^+-200-scaled and config-4 hexes."""
    from tests import gpu_emulation as gemu
    from tests.test_tau_bounds import _degenerate_hexes
    X = np.concatenate([
        hexgen.soa_to_nodes(hexgen.soa_config(600, 0.35, 61)),
        hexgen.soa_to_nodes(hexgen.soa_config(300, 0.6, 62)),
        np.stack(_degenerate_hexes(300, 63)),
        hexgen.soa_to_nodes(hexgen.soa_config(200, 0.4, 64)) * 2.0 ** 200,
        hexgen.soa_to_nodes(hexgen.soa_config(200, 0.4, 65)) * 2.0 ** -200,
        hexgen.soa_to_nodes(hexgen.adversarial_config(400, 4, start=77_000)[0])])
    coords = hexgen.nodes_to_soa(X)
    _, k = gpu_soa(coords, coeffs=True)
    emu = np.array([gemu.root_coeffs(X[i]) for i in range(X.shape[0])]).T
    assert np.array_equal(k.view(np.uint64), emu.view(np.uint64))


def test_binding_rejects_mis_shaped_outputs():
    """Every caller-supplied output is checked against n before the library writes it
    (ADVICE r1): undersized or transposed buffers raise instead of being overrun."""
    coords = torch.from_numpy(hexgen.soa_config(100, 0.3, 5)).cuda()
    verts, idx = hexgen.indexed_config(3, start=0, count=100)
    v, i = torch.from_numpy(verts).cuda(), torch.from_numpy(idx).cuda()
    f99 = torch.empty(99, dtype=torch.uint8, device="cuda")
    d99 = torch.empty(99, dtype=torch.float64, device="cuda")
    bad = [
        lambda: hv.check_soa(coords, flags=f99),
        lambda: hv.check_soa(coords, coeffs=torch.empty((100, 27), dtype=torch.float64, device="cuda")),
        lambda: hv.check_indexed(v, i, flags=f99),
        lambda: hv.check_indexed(v, i[:, :4].contiguous()),
        lambda: hv.corner_quality_indexed(v, i[:, :4].contiguous()),
        lambda: hv.corner_quality_soa(coords, sj_min=d99),
        lambda: hv.check_screen_soa(coords, test1=f99),
        lambda: hv.min_detj_bounds_soa(coords, 1e-3, lower=d99),
        lambda: hv.min_detj_bounds_indexed(v, i[:, :4].contiguous(), 1e-3),
        lambda: hv.classify_bezier(torch.empty((27, 100), dtype=torch.float64, device="cuda"), flags=f99),
        lambda: hv.check_quad_soa(torch.zeros((8, 100), dtype=torch.float64, device="cuda"),
                                  J=torch.empty((4, 99), dtype=torch.float64, device="cuda")),
        lambda: hv.select_valid(torch.zeros(100, dtype=torch.uint8, device="cuda"), ids=torch.empty(
            99, dtype=torch.int32, device="cuda")),
        lambda: hv.select_valid(torch.zeros(100, dtype=torch.uint8, device="cuda"),
                                group=torch.zeros(100, dtype=torch.int32, device="cuda"), n_groups=10,
                                group_counts=torch.zeros(9, dtype=torch.int32, device="cuda")),
    ]
    for k, call in enumerate(bad):
        with pytest.raises(ValueError):
            call()


def test_paper_figures(golden_hexes):
    X = np.stack([golden_hexes[k][0] for k in ("fig5_invalid", "fig6_valid", "fig7_invalid")])
    coords = hexgen.nodes_to_soa(X)
    f, k = gpu_soa(coords, coeffs=True)
    assert (f & 3).tolist() == [hv.INVALID, hv.VALID, hv.INVALID]
    assert f.tolist() == [hv.INVALID | hv.FLAG_SUBDIVIDED, hv.VALID | hv.FLAG_SUBDIVIDED, hv.INVALID]
    ref = oracle.check_soa(coords, want_coeffs=True)
    assert_flags_match(f, ref)
    assert_coeffs_match(k, ref["coeffs"], f)


def test_closed_forms():
    rng = np.random.default_rng(1)
    U = pins.KAPPA.astype(float)
    hexes = [U, U * [2, 3, 4], U * [-1, 1, 1]]
    for _ in range(50):
        A = rng.normal(size=(3, 3))
        hexes.append(U @ A.T + rng.normal(size=3))
    X = np.stack(hexes)
    f, k = gpu_soa(hexgen.nodes_to_soa(X), coeffs=True)
    assert f[0] == hv.VALID and np.all(k[:, 0] == 1.0)
    assert f[1] == hv.VALID and np.all(k[:, 1] == 24.0)
    assert f[2] == hv.INVALID and np.all(k[:, 2] == -1.0)
    for j in range(3, X.shape[0]):
        d = np.linalg.det(X[j, [1, 3, 4]] - X[j, 0])
        assert np.max(np.abs(k[:, j] - d)) <= 1e-13 * max(1.0, np.abs(X[j]).max() ** 3)
        assert f[j] == (hv.VALID if d > 0 else hv.INVALID)


def test_nonfinite_and_empty():
    U = pins.KAPPA.astype(float)
    X = np.stack([U.copy() for _ in range(6)])
    X[0, 3, 1] = np.nan
    X[1, 0, 0] = np.inf
    X[2, 7, 2] = -np.inf
    X[3, 5, 0] = 2.0 ** 301
    X[4] *= 2.0 ** 299
    f, _ = gpu_soa(hexgen.nodes_to_soa(X))
    assert f.tolist() == [3, 3, 3, 3, 1, 1]
    empty = torch.empty((24, 0), dtype=torch.float64, device="cuda")
    fl, _ = hv.check_soa(empty)
    torch.cuda.synchronize()
    assert fl.numel() == 0


def test_cuda_graph_capture_and_replay():
    """The call is stream-ordered end to end (scratch via cudaMallocAsync, no host
    sync), so a caller can capture it in a CUDA graph and replay it on new data."""
    n = 20011
    a = hexgen.ragged_soa(n, seed=7, amp=0.45)
    b = hexgen.ragged_soa(n, seed=8, amp=0.45)
    ref_b = oracle.check_soa(b)
    static_in = torch.from_numpy(a).cuda()
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        hv.check_soa(static_in, flags=flags)                     # warm (device info, pool)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        hv.check_soa(static_in, flags=flags)
    for _ in range(3):
        static_in.copy_(torch.from_numpy(b))
        g.replay()
    torch.cuda.synchronize()
    assert_flags_match(flags.cpu().numpy(), ref_b, allow_near=True)
    static_in.copy_(torch.from_numpy(a))
    g.replay()
    torch.cuda.synchronize()
    eager, _ = gpu_soa(a)
    assert np.array_equal(flags.cpu().numpy(), eager)


def test_binding_uses_torchs_current_stream():
    """The binding's fast current-stream lookup equals torch.cuda.current_stream()."""
    from paper_1706_01613_b200 import _stream_handle
    assert _stream_handle(None) == torch.cuda.current_stream().cuda_stream
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        assert _stream_handle(None) == s.cuda_stream == torch.cuda.current_stream().cuda_stream
    assert _stream_handle(s) == s.cuda_stream


def test_side_stream_matches_default_stream():
    coords = hexgen.ragged_soa(4099, seed=11, amp=0.45)
    dev = torch.from_numpy(coords).cuda()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        f1, _ = hv.check_soa(dev)
    f2, _ = hv.check_soa(dev, stream=s)
    s.synchronize()
    f0, _ = gpu_soa(coords)
    assert np.array_equal(f1.cpu().numpy(), f0) and np.array_equal(f2.cpu().numpy(), f0)


def test_scratch_arenas_are_persistent_and_per_stream():
    """Scratch is borrowed from persistent library-owned arenas: a repeated call
    on the same stream allocates nothing (the reserved bytes do not change), a second stream
    with work in flight gets its own arena, and hexval_scratch_release frees them."""
    hv.scratch_release()
    assert hv.scratch_info()["arenas"] == 0
    coords = torch.from_numpy(hexgen.soa_config(2_000_000, 0.35, 1)).cuda()
    f0, _ = hv.check_soa(coords)
    torch.cuda.synchronize()
    a = hv.scratch_info()
    assert a["arenas"] == 1 and a["bytes"] > 0
    for _ in range(3):
        f1, _ = hv.check_soa(coords)
    torch.cuda.synchronize()
    assert hv.scratch_info() == a                               # steady state: no allocation
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = []
    for st in (s1, s2):
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            out.append(hv.check_soa(coords)[0])
    torch.cuda.synchronize()
    assert all(torch.equal(o, f0) for o in out) and torch.equal(f1, f0)
    assert 1 <= hv.scratch_info()["arenas"] <= 3
    hv.scratch_release()
    assert hv.scratch_info() == {"bytes": 0, "arenas": 0}
    f2, _ = hv.check_soa(coords)                                # works again after a release
    torch.cuda.synchronize()
    assert torch.equal(f2, f0)


def test_concurrent_calls_on_two_streams_and_threads():
    """Scratch is per call and device setup is guarded, so calls from two host
    threads on two streams (ctypes releases the GIL) give the single-call results."""
    import threading
    a = hexgen.ragged_soa(300_001, seed=21, amp=0.45)
    b = hexgen.ragged_soa(200_003, seed=22, amp=0.45)
    fa0, _ = gpu_soa(a)
    fb0, _ = gpu_soa(b)
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    out = {}

    def run(key, dev):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(5):
                f, _ = hv.check_soa(dev, stream=s)
        s.synchronize()
        out[key] = f.cpu().numpy()

    torch.cuda.synchronize()
    ts = [threading.Thread(target=run, args=("a", da)), threading.Thread(target=run, args=("b", db))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert np.array_equal(out["a"], fa0) and np.array_equal(out["b"], fb0)


# --------------------------------------------------------------------------
# small configs, ragged sizes, exact path, subdivision
# --------------------------------------------------------------------------

def test_config0_full_parity():
    _, coords = hexgen.make(0)
    stats = hv.Stats()
    f, k = gpu_soa(coords, coeffs=True, stats=stats)
    ref = oracle.check_soa(coords, want_coeffs=True)
    assert_flags_match(f, ref)
    assert_coeffs_match(k, ref["coeffs"], f)
    st = stats.read()
    assert st["n_valid"] + st["n_invalid"] + st["n_undetermined"] + st["n_nonfinite"] == coords.shape[1]
    assert st["n_subdivided"] == int(np.sum((f & 4) > 0))


@pytest.mark.parametrize("n", [1, 31, 255, 256, 257, 1000, 3 * 256 + 37, 20011])
def test_ragged_sizes_high_noise(n):
    coords = hexgen.ragged_soa(n, seed=100 + n, amp=0.45)
    f, k = gpu_soa(coords, coeffs=True)
    ref = oracle.check_soa(coords, want_coeffs=True)
    assert_flags_match(f, ref, allow_near=True)
    assert ref["near"].sum() <= max(1, n // 5000)
    assert_coeffs_match(k, ref["coeffs"], f)


@pytest.mark.parametrize("n", [256 * 148 * 4 + 1, 256 * 148 * 3, 256 * 300 + 255])
def test_tma_pipeline_sizes(n):
    """Several chunks per persistent warp, odd n (shifted plane copies) and a ragged tail."""
    coords = hexgen.ragged_soa(n, seed=n % 1000, amp=0.45)
    f, k = gpu_soa(coords, coeffs=True)
    ref = oracle.check_soa(coords, want_coeffs=True)
    assert_flags_match(f, ref, allow_near=True)
    assert ref["near"].sum() <= max(1, n // 5000)
    assert_coeffs_match(k, ref["coeffs"], f)


def test_misaligned_base_uses_plain_path_with_same_results():
    """An 8-B aligned (not 16-B) coordinate pointer takes the plain kernel: same bits."""
    n = 5003
    coords = hexgen.ragged_soa(n, seed=77, amp=0.45)
    big = torch.empty(24 * n + 1, dtype=torch.float64, device="cuda")
    big[1:] = torch.from_numpy(coords.ravel()).cuda()
    view = big[1:].view(24, n)
    assert view.data_ptr() % 16 == 8
    f1, k1 = hv.check_soa(view, coeffs=True)
    f2, k2 = gpu_soa(coords, coeffs=True)
    torch.cuda.synchronize()
    assert np.array_equal(f1.cpu().numpy(), f2) and np.array_equal(k1.cpu().numpy(), k2)


@pytest.mark.parametrize("shift_idx,shift_verts", [(1, 0), (2, 1), (0, 1)])
def test_indexed_misaligned_pointers_same_results(shift_idx, shift_verts):
    """Connectivity 4-B (not 16-B) aligned takes the plain gather kernel; vertices
    8-B (not 16-B) aligned stay on the pipelined one: same bits either way."""
    verts, idx = hexgen.indexed_config(3, start=777, count=256 * 148 + 999)
    ref_f, ref_k = gpu_indexed(verts, idx, coeffs=True)
    bi = torch.empty(idx.size + shift_idx, dtype=torch.int32, device="cuda")
    bi[shift_idx:] = torch.from_numpy(idx.ravel()).cuda()
    bv = torch.empty(verts.size + shift_verts, dtype=torch.float64, device="cuda")
    bv[shift_verts:] = torch.from_numpy(verts.ravel()).cuda()
    iv = bi[shift_idx:].view(idx.shape)
    vv = bv[shift_verts:].view(verts.shape)
    f, k = hv.check_indexed(vv, iv, coeffs=True)
    torch.cuda.synchronize()
    assert np.array_equal(f.cpu().numpy(), ref_f) and np.array_equal(k.cpu().numpy(), ref_k)


@pytest.mark.parametrize("n", [256 * 148 * 2 + 77, 256 * 148 * 3 + 256 * 5])
def test_pass1_variants_bit_identical(tmp_path, n):
    """HEXVAL_PASS1=ldg|wtma|cp|bulk (tuning knob) give identical flags and coefficients
    (odd n: shifted plane rows and a ragged tail; even n: full tiles only)."""
    import subprocess
    import sys
    coords = hexgen.ragged_soa(n, seed=5, amp=0.5)
    np.save(tmp_path / "c.npy", coords)
    script = (
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {str(hexgen.__file__.rsplit('/', 2)[0])!r})\n"
        "import paper_1706_01613_b200 as hv\n"
        f"c = torch.from_numpy(np.load({str(tmp_path / 'c.npy')!r})).cuda()\n"
        "f, k = hv.check_soa(c, coeffs=True); torch.cuda.synchronize()\n"
        f"np.save({str(tmp_path)!r} + '/f_' + sys.argv[1] + '.npy', f.cpu().numpy())\n"
        f"np.save({str(tmp_path)!r} + '/k_' + sys.argv[1] + '.npy', k.cpu().numpy())\n")
    for v in ("ldg", "wtma", "cp", "bulk"):
        env = dict(os.environ, HEXVAL_PASS1=v)
        subprocess.run([sys.executable, "-c", script, v], env=env, check=True, timeout=300)
    f0, k0 = np.load(tmp_path / "f_ldg.npy"), np.load(tmp_path / "k_ldg.npy")
    for v in ("wtma", "cp", "bulk"):
        assert np.array_equal(np.load(tmp_path / f"f_{v}.npy"), f0), v
        assert np.array_equal(np.load(tmp_path / f"k_{v}.npy"), k0), v


def test_indexed_variants_bit_identical(tmp_path):
    """Indexed pass 1: plain gather kernel (HEXVAL_PASS1=ldg) and the cp.async gather pipeline
    give identical flags and coefficients on a ragged config-3 slice (duplicates included)."""
    import subprocess
    import sys
    verts, idx = hexgen.indexed_config(3, start=12345, count=256 * 148 * 2 + 101)
    np.save(tmp_path / "v.npy", verts)
    np.save(tmp_path / "i.npy", idx)
    script = (
        "import sys, numpy as np, torch\n"
        f"sys.path.insert(0, {str(hexgen.__file__.rsplit('/', 2)[0])!r})\n"
        "import paper_1706_01613_b200 as hv\n"
        f"v = torch.from_numpy(np.load({str(tmp_path / 'v.npy')!r})).cuda()\n"
        f"i = torch.from_numpy(np.load({str(tmp_path / 'i.npy')!r})).cuda()\n"
        "f, k = hv.check_indexed(v, i, coeffs=True); torch.cuda.synchronize()\n"
        f"np.save({str(tmp_path)!r} + '/f_' + sys.argv[1] + '.npy', f.cpu().numpy())\n"
        f"np.save({str(tmp_path)!r} + '/k_' + sys.argv[1] + '.npy', k.cpu().numpy())\n")
    for v in ("ldg", "cp"):
        env = dict(os.environ, HEXVAL_PASS1=v)
        subprocess.run([sys.executable, "-c", script, v], env=env, check=True, timeout=300)
    assert np.array_equal(np.load(tmp_path / "f_ldg.npy"), np.load(tmp_path / "f_cp.npy"))
    assert np.array_equal(np.load(tmp_path / "k_ldg.npy"), np.load(tmp_path / "k_cp.npy"))


def test_subdivision_heavy_random_hexes():
    """Amplitude 0.5 gives many subdivided hexes of both final verdicts."""
    coords = hexgen.ragged_soa(200_000, seed=7, amp=0.5)
    stats = hv.Stats()
    f, _ = gpu_soa(coords, stats=stats)
    ref = oracle.check_soa(coords)
    assert_flags_match(f, ref, allow_near=True)
    sub = (f & 4) > 0
    assert sub.sum() > 50
    assert np.any((f[sub] & 3) == hv.INVALID) and np.any((f[sub] & 3) == hv.VALID)
    # node counts are order independent for VALID hexes: totals must agree
    valid_sub = sub & ((f & 3) == hv.VALID)
    st = stats.read()
    assert st["n_subdivided"] == sub.sum()
    assert st["n_nodes"] >= ref["nodes"][valid_sub].sum()


def _degenerate_soa(n, seed):
    rng = np.random.default_rng(seed)
    U = pins.KAPPA.astype(float)
    X = U[None] + rng.uniform(-0.3, 0.3, size=(n, 8, 3))
    for h in range(n):
        kind = h % 4
        i, j = rng.choice(8, size=2, replace=False)
        if kind == 0:
            X[h, j] = X[h, i]                       # duplicate (maybe diagonal)
        elif kind == 1:
            X[h, 2] = X[h, 0]                       # nodes 1, 3 coincide: c2 exactly 0, fp +-tiny
        elif kind == 2:
            X[h, :, 2] = np.round(X[h, :, 2] * 4) / 4   # coplanar dyadic layers
            X[h, j, 2] = X[h, i, 2]
    return hexgen.nodes_to_soa(X)


def test_exact_sign_path_degenerate_hexes():
    coords = _degenerate_soa(4000, 3)
    stats = hv.Stats()
    f, k = gpu_soa(coords, coeffs=True, stats=stats)
    ref = oracle.check_soa(coords, want_coeffs=True)
    assert_flags_match(f, ref, allow_near=True)
    assert ref["near"].sum() <= 4
    assert stats.read()["n_exact"] > 100          # the K5 kernel really ran
    assert ref["exact"].sum() > 100


def test_classify_bezier_depth_cap_and_random():
    """Steps 4-5 on given coefficients vs the oracle's classify_coeffs (UNDETERMINED, node counts)."""
    a = 1.0 / 3.0
    q = np.array([a * a, a * (a - 1.0), (1.0 - a) ** 2])
    point_zero = np.array([q[i] + q[j] + q[k] for i, j, k in pins.XI2])
    rng = np.random.default_rng(5)
    B = [point_zero, point_zero + 1e-3]
    for _ in range(3000):
        b = rng.uniform(0.05, 1.0, size=27)
        b[8 + rng.integers(0, 19, size=rng.integers(1, 4))] -= rng.uniform(0.0, 1.5)
        B.append(b)
    B = np.array(B).T.copy()                      # (27, m) coefficient-major
    stats = hv.Stats()
    f = hv.classify_bezier(torch.from_numpy(B).cuda(), stats=stats)
    torch.cuda.synchronize()
    f = f.cpu().numpy()
    assert f[0] == (hv.UNDETERMINED | hv.FLAG_SUBDIVIDED)
    assert f[1] == (hv.VALID | hv.FLAG_SUBDIVIDED)
    ref_flags, nodes_full = [], 0
    for j in range(B.shape[1]):
        r = oracle.classify_coeffs(B[:, j], 1.0)
        ref_flags.append(r["flags"])
        if (r["flags"] & 3) != oracle.INVALID and not r["near_boundary"]:
            nodes_full += r["nodes"]
    ref_flags = np.array(ref_flags)
    assert np.array_equal(f, ref_flags)
    assert np.sum((f & 3) == hv.INVALID) > 100 and np.sum(f == (hv.VALID | 4)) > 100
    assert stats.read()["n_nodes"] >= nodes_full


def test_subdivision_decisions_identical_to_the_oracle_recursion():
    """K4 keeps power-of-two scaled coefficients whose values are bit for bit the oracle's
    de Casteljau values (oracle_subdivide) times their scales, so from the same root it takes
    exactly the oracle's decisions: on the oracle's own root coefficients of config-4 hexes
    (pushed corners, twisted prisms down to |r| = 1e-5) and random hexes, hexval_classify_bezier
    returns the oracle's flags on EVERY item (near-boundary ones included), and over the VALID
    items exactly the oracle's number of subdivision nodes."""
    c4, _ = hexgen.adversarial_config(6000, seed=4, start=200_000)
    rnd = hexgen.soa_config(4000, 0.45, 77)
    coords = np.ascontiguousarray(np.concatenate([c4, rnd], axis=1))
    b = oracle.check_soa(coords, want_coeffs=True)["coeffs"]
    m = b.shape[1]
    ref = [oracle.classify_coeffs(b[:, j], 1.0) for j in range(m)]
    ref_flags = np.array([r["flags"] for r in ref], np.uint8)
    f = hv.classify_bezier(torch.from_numpy(b).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(f.cpu().numpy(), ref_flags)
    sub = ref_flags & 4 != 0
    assert sub.sum() > 2500 and ((ref_flags & 3) == 0).sum() > 1000
    valid = np.nonzero(ref_flags == (hv.VALID | hv.FLAG_SUBDIVIDED))[0]
    stats = hv.Stats()
    fv = hv.classify_bezier(torch.from_numpy(np.ascontiguousarray(b[:, valid])).cuda(), stats=stats)
    torch.cuda.synchronize()
    assert np.all(fv.cpu().numpy() == (hv.VALID | hv.FLAG_SUBDIVIDED))
    assert stats.read()["n_nodes"] == sum(ref[j]["nodes"] for j in valid)


def test_indexed_equals_soa_and_host_path():
    verts, idx = hexgen.indexed_config(3, start=0, count=300_000)
    coords = hexgen.indexed_to_soa(verts, idx)
    f1, k1 = gpu_soa(coords, coeffs=True)
    f2, k2 = gpu_indexed(verts, idx, coeffs=True)
    assert np.array_equal(f1, f2)
    assert np.array_equal(k1, k2)                 # same arithmetic, same bits
    f3 = np.zeros(coords.shape[1], np.uint8)
    hv.check_soa_host(coords, f3, chunk_hexes=70_000)
    assert np.array_equal(f1, f3)
    f4 = np.zeros(idx.shape[0], np.uint8)
    k4 = np.zeros((27, idx.shape[0]))
    hv.check_indexed_host(verts, idx, f4, coeffs=k4, chunk_hexes=100_003)
    assert np.array_equal(f1, f4) and np.array_equal(k1, k4)


# --------------------------------------------------------------------------
# full-size configurations (launch configuration of bench.py)
# --------------------------------------------------------------------------

def _sample(n, flags, k, seed):
    rng = np.random.default_rng(seed)
    special = np.nonzero((flags & 4) > 0)[0]
    return np.unique(np.concatenate([rng.choice(n, size=min(n, k), replace=False), special[:20000]]))


def test_config1_full_size_sampled():
    _, coords = full_config(1)
    n = coords.shape[1]
    stats = hv.Stats()
    f, _ = gpu_soa(coords, stats=stats)
    st = stats.read()
    assert st["n_valid"] + st["n_invalid"] + st["n_undetermined"] + st["n_nonfinite"] == n
    sel = _sample(n, f, 30000, 1)
    ref = oracle.check_soa(np.ascontiguousarray(coords[:, sel]))
    assert_flags_match(f[sel], ref)
    frac_sub = np.mean((f & 4) > 0)
    assert 1e-6 < frac_sub < 1e-3                 # ~3.2e-5


def test_config2_full_size_sampled():
    _, verts, idx = full_config(2)
    f, _ = gpu_indexed(verts, idx)
    sel = _sample(idx.shape[0], f, 30000, 2)
    ref = oracle.check_indexed(verts, idx[sel])
    assert_flags_match(f[sel], ref)


def test_config3_full_size_sampled():
    _, verts, idx = full_config(3)
    stats = hv.Stats()
    f, _ = gpu_indexed(verts, idx, stats=stats)
    n = idx.shape[0]
    dup = np.nonzero(np.array([len(set(r)) < 8 for r in idx[:400_000].tolist()]))[0]
    sel = np.unique(np.concatenate([_sample(n, f, 30000, 3), dup[:20000]]))
    ref = oracle.check_indexed(verts, idx[sel])
    assert_flags_match(f[sel], ref)
    assert ref["exact"][np.isin(sel, dup)].sum() > 0       # the oracle needed exact signs there
    st = stats.read()
    assert st["n_valid"] + st["n_invalid"] + st["n_undetermined"] + st["n_nonfinite"] == n


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_full_size_every_hex_against_the_oracle(cfg):
    """Configs 1-3 at full size, every hex (not a sample): the oracle runs on all host
    cores (about 6 M hex/s), so the whole config is compared bit for bit, and the
    near-boundary count must be 0 (BASELINE.json north star)."""
    if cfg == 1:
        _, coords = full_config(1)
        f, k = gpu_soa(coords, coeffs=True)
        ref = oracle.check_soa(coords, want_coeffs=True)
        assert_coeffs_match(k, ref["coeffs"], f)             # all 270M coefficients, 1e-12 x max|b|
    else:
        _, verts, idx = full_config(cfg)
        f, _ = gpu_indexed(verts, idx)
        ref = oracle.check_indexed(verts, idx)
    assert_flags_match(f, ref)


def test_config4_full_size_closed_form_and_sampled():
    _, coords, r = hexgen.make(4)
    stats = hv.Stats()
    f, _ = gpu_soa(coords, stats=stats)
    verdict = f & 3
    expect = np.where(r > 0, hv.VALID, hv.INVALID)
    assert np.array_equal(verdict, expect)        # closed form, every hex
    even = np.arange(r.size) % 2 == 0
    assert not np.any(f[even] & 4)
    rng = np.random.default_rng(4)
    sel = np.unique(rng.choice(r.size, size=3000, replace=False))
    ref = oracle.check_soa(np.ascontiguousarray(coords[:, sel]))
    assert_flags_match(f[sel], ref)


def test_config4_every_hex_against_the_oracle():
    """Config 4 (4M adversarial hexes, ~5e9 subdivision nodes) compared on EVERY hex, whole
    flags byte (verdict and SUBDIVIDED bit), against the oracle's flags stored by
    tools/make_config4_golden.py (which calls only oracle/; 26 min on 8 host cores).  The
    oracle marks no hex near-boundary.  For the VALID hexes the subdivision node counts are
    order independent (reading G4): their GPU total equals the oracle's."""
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "config4_oracle.npz"))
    _, coords, _ = hexgen.make(4)
    assert int(g["n"]) == coords.shape[1] and int(g["seed"]) == 4
    assert int(g["near"].sum()) == 0
    f, _ = gpu_soa(coords)
    assert np.array_equal(f, g["flags"])
    valid = np.nonzero(g["flags"] == (hv.VALID | hv.FLAG_SUBDIVIDED))[0]
    stats = hv.Stats()
    fv, _ = gpu_soa(np.ascontiguousarray(coords[:, valid]), stats=stats)
    assert np.all(fv == hv.VALID | hv.FLAG_SUBDIVIDED)
    assert stats.read()["n_nodes"] == int(g["nodes"][valid].astype(np.int64).sum())


def test_subdivision_node_count_equals_oracle_for_valid_hexes():
    """VALID hexes explore their whole capped tree, so the number of subdivided nodes is
    order independent (reading G4): the warp-cooperative K4 must count exactly what the
    oracle's depth-first recursion counts."""
    coords, r = hexgen.adversarial_config(4000, seed=4, start=100_001)
    ids = np.arange(100_001, 104_001)
    sel = np.nonzero((ids % 2 == 1) & (r > 0))[0]           # twisted prisms, valid
    c = np.ascontiguousarray(coords[:, sel])
    ref = oracle.check_soa(c)
    assert not ref["near"].any()
    assert np.all(ref["flags"] == (hv.VALID | hv.FLAG_SUBDIVIDED))
    stats = hv.Stats()
    f, _ = gpu_soa(c, stats=stats)
    assert np.array_equal(f, ref["flags"])
    st = stats.read()
    assert st["n_subdivided"] == sel.size
    assert st["n_nodes"] == int(ref["nodes"].sum())


# --------------------------------------------------------------------------
# NEXT-2: corner scaled Jacobian and Ushakova Test 1
# --------------------------------------------------------------------------

def _quality_parity(coords, sj, t1):
    ref = oracle.corner_quality_soa(coords)
    nan_ref = np.isnan(ref["sj_min"])
    assert np.array_equal(np.isnan(sj), nan_ref)
    ok = ~nan_ref
    assert np.max(np.abs(sj[ok] - ref["sj_min"][ok]), initial=0.0) <= 1e-13
    # Test 1 is decided exactly on both sides (corner samples within the rounding bound take
    # their exact sign): equal on every item, near-zero corners included
    assert np.array_equal(t1, ref["test1"])
    return ref


@pytest.mark.parametrize("n", [1, 255, 257, 20011])
def test_corner_quality_parity(n, golden_hexes):
    coords = hexgen.ragged_soa(n, seed=300 + n, amp=0.45)
    dev = torch.from_numpy(coords).cuda()
    sj, t1 = hv.corner_quality_soa(dev)
    torch.cuda.synchronize()
    _quality_parity(coords, sj.cpu().numpy(), t1.cpu().numpy())


def test_corner_quality_special_cases(golden_hexes):
    U = pins.KAPPA.astype(float)
    S = U.copy(); S[:, 0] += 0.5 * S[:, 1]
    D = U.copy(); D[1] = D[0]                                   # zero-length corner edge
    N = U.copy(); N[4, 2] = np.nan
    X = np.stack([U, S, U * [-1, 1, 1], D, N, golden_hexes["fig7_invalid"][0], golden_hexes["fig5_invalid"][0]])
    coords = hexgen.nodes_to_soa(X)
    sj, t1 = hv.corner_quality_soa(torch.from_numpy(coords).cuda())
    torch.cuda.synchronize()
    sj, t1 = sj.cpu().numpy(), t1.cpu().numpy()
    assert sj[0] == 1.0 and abs(sj[1] - 1 / np.sqrt(1.25)) <= 1e-15 and sj[2] == -1.0
    assert np.isnan(sj[3]) and np.isnan(sj[4])
    assert abs(sj[5] - 0.6471) < 5e-5                           # Fig. 7 caption "0.64"
    assert t1.tolist() == [1, 1, 0, 0, 0, 1, 1]                  # Fig. 5 passes Test 1 (necessary only)
    _quality_parity(coords, sj, t1)


@pytest.mark.parametrize("e", [-250, -100, -70, 70, 100, 250])
def test_corner_quality_at_extreme_scales(e):
    """The scaled Jacobian is scale invariant and Test 1 is a sign: at coordinate scales 2^e
    where the squared-length products would overflow or underflow, the kernels recompute sj in
    a power-of-two rescaled frame; both outputs equal the oracle's on the scaled hexes (and
    the unscaled values), standalone and fused."""
    coords = np.ldexp(hexgen.ragged_soa(3001, seed=77, amp=0.45), e)
    dev = torch.from_numpy(coords).cuda()
    sj, t1 = hv.corner_quality_soa(dev)
    _, sj2, t12 = hv.check_screen_soa(dev)
    torch.cuda.synchronize()
    ref = _quality_parity(coords, sj.cpu().numpy(), t1.cpu().numpy())
    _quality_parity(coords, sj2.cpu().numpy(), t12.cpu().numpy())
    base = oracle.corner_quality_soa(np.ldexp(coords, -e))
    ok = ~np.isnan(base["sj_min"])
    assert np.max(np.abs(ref["sj_min"][ok] - base["sj_min"][ok]), initial=0.0) <= 1e-14
    assert np.array_equal(ref["test1"], base["test1"])


@pytest.mark.parametrize("n", [1, 255, 257, 256 * 148 * 2 + 77])
def test_fused_screen_equals_separate_calls(n):
    """hexval_check_screen_soa: flags bit-identical to check_soa, sj/test1 bit-identical to
    corner_quality_soa (same corner samples, same arithmetic), NaN/NONFINITE rows included."""
    coords = hexgen.ragged_soa(n, seed=900 + n % 97, amp=0.45)
    if n > 300:
        coords[7, 5] = np.nan
        coords[0, 6:9] = coords[3, 6:9]                         # nodes 1 and 2 coincide: zero edge
        coords[1, 6:9] = coords[4, 6:9]
        coords[2, 6:9] = coords[5, 6:9]
    dev = torch.from_numpy(coords).cuda()
    f, sj, t1 = hv.check_screen_soa(dev)
    f0, _ = hv.check_soa(dev)
    sj0, t10 = hv.corner_quality_soa(dev)
    torch.cuda.synchronize()
    assert np.array_equal(f.cpu().numpy(), f0.cpu().numpy())
    a, b = sj.cpu().numpy(), sj0.cpu().numpy()
    assert np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])
    assert np.array_equal(t1.cpu().numpy(), t10.cpu().numpy())
    ref = oracle.check_soa(coords)
    assert_flags_match(f.cpu().numpy(), ref, allow_near=True)


@pytest.mark.parametrize("cfg", [1, 3])
def test_test1_is_necessary_at_full_size(cfg):
    """Ushakova's Test 1 is necessary for validity: over the whole
    config, no hex the robust check calls VALID fails Test 1 (a property that holds at
    any size, checked on every hex through the fused screening call)."""
    if cfg == 1:
        _, coords = full_config(1)
        f, sj, t1 = hv.check_screen_soa(torch.from_numpy(coords).cuda())
    else:
        _, verts, idx = full_config(3)
        f, sj, t1 = hv.check_screen_indexed(torch.from_numpy(verts).cuda(), torch.from_numpy(idx).cuda())
    torch.cuda.synchronize()
    valid = (f & 3) == hv.VALID
    assert int(valid.sum().item()) > 0
    assert bool((t1[valid] == 1).all().item())
    assert bool((sj[valid] > 0).all().item())


def test_fused_screen_range_decision():
    """The fused screening pass takes NONFINITE from the edge-scale key (3 masked keys on the
    fast path, the exact test out of line): NaN / Inf / 2^301 coordinates, in-range hexes at
    2^298 .. 2^300 (suspects that must still be validated), a huge offset with unit edges (edge
    key small, node-1 key large) and one beyond the range (edges 0 in fp64), all equal to the
    plain validity call and, where defined, to the oracle."""
    U = pins.KAPPA.astype(float)
    X = np.stack([U.copy() for _ in range(11)])
    X[0, 3, 1] = np.nan
    X[1, 0, 0] = np.inf
    X[2, 7, 2] = -np.inf
    X[3, 5, 0] = 2.0 ** 301
    X[4] *= 2.0 ** 299
    X[5] *= 2.0 ** 298
    X[6] *= 2.0 ** 296
    X[7] = (U - 0.5) * 2.0 ** 300                       # |x| = 2^299: in range, edges 2^300
    X[8] = U + 2.0 ** 40                                # large offset, unit edges
    X[9] = U * 2.0 ** 250 + 2.0 ** 301                  # out of range through the offset alone
    X[10, 6, 2] = -(2.0 ** 300) * (1 + 2.0 ** -52)      # just beyond 2^300
    reps = 40                                            # several warps, mixed with ordinary hexes
    coords = np.concatenate([hexgen.nodes_to_soa(X), hexgen.ragged_soa(700, seed=77, amp=0.4)] * reps, axis=1)
    dev = torch.from_numpy(np.ascontiguousarray(coords)).cuda()
    f, sj, t1 = hv.check_screen_soa(dev)
    f0, _ = hv.check_soa(dev)
    sj0, t10 = hv.corner_quality_soa(dev)
    torch.cuda.synchronize()
    f, f0 = f.cpu().numpy(), f0.cpu().numpy()
    assert np.array_equal(f, f0)
    assert f[:11].tolist() == [3, 3, 3, 3, 1, 1, 1, 1, 1, 3, 3]
    a, b = sj.cpu().numpy(), sj0.cpu().numpy()
    assert np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])
    assert np.array_equal(t1.cpu().numpy(), t10.cpu().numpy())
    assert np.all(np.isnan(a[:4])) and np.all(t1.cpu().numpy()[:4] == 0) and np.all(np.isnan(a[9:11]))
    assert np.allclose(a[4:8], 1.0, rtol=1e-13, atol=0) and np.all(t1.cpu().numpy()[4:8] == 1)
    ref = oracle.check_soa(coords)
    assert_flags_match(f, ref, allow_near=True)
    # the indexed path: the same 11 hexes as 88 vertices
    verts = np.ascontiguousarray(X.reshape(-1, 3))
    idx = np.arange(88, dtype=np.int32).reshape(11, 8)
    fi, sji, t1i = hv.check_screen_indexed(torch.from_numpy(verts).cuda(), torch.from_numpy(idx).cuda())
    torch.cuda.synchronize()
    assert fi.cpu().numpy().tolist() == f[:11].tolist()
    ai = sji.cpu().numpy()
    assert np.array_equal(np.isnan(ai), np.isnan(a[:11])) and np.array_equal(ai[~np.isnan(ai)], a[:11][~np.isnan(a[:11])])
    assert np.array_equal(t1i.cpu().numpy(), t1.cpu().numpy()[:11])


def test_fused_screen_indexed_config3_slice():
    verts, idx = hexgen.indexed_config(3, start=4242, count=256 * 148 + 555)
    v, i = torch.from_numpy(verts).cuda(), torch.from_numpy(idx).cuda()
    f, sj, t1 = hv.check_screen_indexed(v, i)
    f0, _ = hv.check_indexed(v, i)
    sj0, t10 = hv.corner_quality_indexed(v, i)
    torch.cuda.synchronize()
    assert np.array_equal(f.cpu().numpy(), f0.cpu().numpy())
    a, b = sj.cpu().numpy(), sj0.cpu().numpy()
    assert np.array_equal(np.isnan(a), np.isnan(b)) and np.array_equal(a[~np.isnan(a)], b[~np.isnan(b)])
    assert np.array_equal(t1.cpu().numpy(), t10.cpu().numpy())


def test_corner_quality_indexed_config3_slice():
    verts, idx = hexgen.indexed_config(3, start=777, count=50_000)
    sj, t1 = hv.corner_quality_indexed(torch.from_numpy(verts).cuda(), torch.from_numpy(idx).cuda())
    torch.cuda.synchronize()
    _quality_parity(hexgen.indexed_to_soa(verts, idx), sj.cpu().numpy(), t1.cpu().numpy())


# --------------------------------------------------------------------------
# NEXT-1: certified bounds on min det J
# --------------------------------------------------------------------------

def _bounds_parity(coords, rel_tol, lo, up, st):
    """Both sides return intervals of width <= tol containing min det J; the refinement
    orders differ (GPU: warp-parallel by levels; oracle: depth first), so what is unique is
    checked: each interval contains the other's witness range and both are tol-tight."""
    ref = oracle.min_detj_bounds_soa(coords, rel_tol)
    X = hexgen.soa_to_nodes(coords)
    nf = np.isnan(ref["lower"])
    assert np.array_equal(np.isnan(lo), nf) and np.array_equal(np.isnan(up), nf)
    assert np.all((st[nf] & 2) == 2)
    ok = ~nf
    tol = np.array([rel_tol * np.abs(oracle.check_hex(X[j])["b"]).max() if ok[j] else 0 for j in range(len(lo))])
    eps = 1e-12 * np.maximum(1.0, np.abs(up))
    capped = ((st & 1) == 1) | (ref["capped"] == 1)
    tight = ok & ~capped
    assert np.all(up[tight] - lo[tight] <= tol[tight] + eps[tight])
    # the true minimum lies in both intervals: they overlap, and each lower is below the other's upper
    assert np.all(lo[ok] <= ref["upper"][ok] + eps[ok]) and np.all(ref["lower"][ok] <= up[ok] + eps[ok])
    assert np.all(np.abs(up[tight] - ref["upper"][tight]) <= tol[tight] + eps[tight])
    assert np.all(np.abs(lo[tight] - ref["lower"][tight]) <= tol[tight] + eps[tight])
    return ref


def _bounds_parity_vec(coords, rel_tol, lo, up, st):
    """_bounds_parity without per-hex Python work (full-size inputs): tol from the oracle's
    root coefficients."""
    ref = oracle.min_detj_bounds_soa(coords, rel_tol)
    nf = np.isnan(ref["lower"])
    assert np.array_equal(np.isnan(lo), nf) and np.array_equal(np.isnan(up), nf)
    ok = ~nf
    b = oracle.check_soa(coords, want_coeffs=True)["coeffs"]
    tol = rel_tol * np.abs(b).max(axis=0)
    eps = 1e-12 * np.maximum(1.0, np.abs(np.where(ok, up, 0.0)))
    tight = ok & ~(((st & 1) == 1) | (ref["capped"] == 1))
    assert np.all(up[tight] - lo[tight] <= tol[tight] + eps[tight])
    assert np.all(lo[ok] <= ref["upper"][ok] + eps[ok]) and np.all(ref["lower"][ok] <= up[ok] + eps[ok])
    assert np.all(np.abs(up[tight] - ref["upper"][tight]) <= tol[tight] + eps[tight])
    assert np.all(np.abs(lo[tight] - ref["lower"][tight]) <= tol[tight] + eps[tight])


@pytest.mark.parametrize("row", ["quality", "bounds", "quads", "select"])
def test_next_rows_full_size_every_item(row):
    """Each NEXT row at its bench workload size, compared on every item (the oracle runs on
    all host cores)."""
    if row == "quads":
        coords = hexgen.quad_soa(10_000_000, 0.35, 5)
        f, J = hv.check_quad_soa(torch.from_numpy(coords).cuda(), J=True)
        torch.cuda.synchronize()
        ref = oracle.check_quad_soa(coords)
        assert np.array_equal(f.cpu().numpy(), ref["flags"]) and np.array_equal(J.cpu().numpy(), ref["J"])
        return
    if row == "select":
        _, verts, idx = full_config(3)
        f, _ = gpu_indexed(verts, idx)
        n = idx.shape[0]
        grp = (np.arange(n) % 99 ** 3).astype(np.int32)
        ids, c, counts = hv.select_valid(torch.from_numpy(f).cuda(), torch.from_numpy(grp).cuda(), 99 ** 3)
        torch.cuda.synchronize()
        ref_ids, ref_counts = oracle.select_valid(f, grp, 99 ** 3)
        assert c == ref_ids.size and np.array_equal(ids.cpu().numpy(), ref_ids)
        assert np.array_equal(counts.cpu().numpy(), ref_counts)
        return
    _, coords = full_config(1)
    dev = torch.from_numpy(coords).cuda()
    if row == "quality":
        sj, t1 = hv.corner_quality_soa(dev)
        torch.cuda.synchronize()
        _quality_parity(coords, sj.cpu().numpy(), t1.cpu().numpy())
    else:
        lo, up, st = hv.min_detj_bounds_soa(dev, 1e-3)
        torch.cuda.synchronize()
        _bounds_parity_vec(coords, 1e-3, lo.cpu().numpy(), up.cpu().numpy(), st.cpu().numpy())


@pytest.mark.parametrize("op", ["quality", "screen"])
def test_test1_exact_on_every_config3_candidate(op):
    """NEXT-2 on all 40M config-3 candidates (18% have a duplicate vertex, many a corner
    det J exactly 0): Test 1 equals the oracle's exact-sign Test 1 on every item, for the
    standalone screening kernel and the fused validity + screening pass; the scaled
    Jacobian matches where it is defined."""
    _, verts, idx = full_config(3)
    v, i = torch.from_numpy(verts).cuda(), torch.from_numpy(idx).cuda()
    if op == "quality":
        sj, t1 = hv.corner_quality_indexed(v, i)
    else:
        _, sj, t1 = hv.check_screen_indexed(v, i)
    torch.cuda.synchronize()
    sj, t1 = sj.cpu().numpy(), t1.cpu().numpy()
    n = idx.shape[0]
    step = 8_000_000
    for a in range(0, n, step):
        ref = oracle.corner_quality_indexed(verts, idx[a:a + step])
        assert np.array_equal(t1[a:a + step], ref["test1"]), a
        nan_ref = np.isnan(ref["sj_min"])
        s = sj[a:a + step]
        assert np.array_equal(np.isnan(s), nan_ref)
        assert np.max(np.abs(s[~nan_ref] - ref["sj_min"][~nan_ref]), initial=0.0) <= 1e-13


@pytest.mark.parametrize("rel_tol", [1e-2, 1e-5])
def test_min_detj_bounds_random(rel_tol):
    coords = hexgen.ragged_soa(5003, seed=41, amp=0.5)
    lo, up, st = hv.min_detj_bounds_soa(torch.from_numpy(coords).cuda(), rel_tol)
    torch.cuda.synchronize()
    _bounds_parity(coords, rel_tol, lo.cpu().numpy(), up.cpu().numpy(), st.cpu().numpy())


def test_min_detj_bounds_closed_forms(golden_hexes):
    coords, r = hexgen.adversarial_config(3000, seed=4, start=9000)
    U = pins.KAPPA.astype(float)
    N = U.copy(); N[2, 1] = np.inf
    extra = np.stack([U, U * [2, 3, 4], N, golden_hexes["fig5_invalid"][0], golden_hexes["fig6_valid"][0],
                      golden_hexes["fig7_invalid"][0]])
    coords = np.ascontiguousarray(np.concatenate([coords, hexgen.nodes_to_soa(extra)], axis=1))
    rel_tol = 1e-4
    nodes = torch.zeros(1, dtype=torch.int64, device="cuda")
    lo, up, st = hv.min_detj_bounds_soa(torch.from_numpy(coords).cuda(), rel_tol, nodes=nodes)
    torch.cuda.synchronize()
    lo, up, st = lo.cpu().numpy(), up.cpu().numpy(), st.cpu().numpy()
    _bounds_parity(coords, rel_tol, lo, up, st)
    m = r.size
    X = hexgen.soa_to_nodes(coords)
    for j in range(m):                                         # min det J = r * volume (closed form)
        b = oracle.check_hex(X[j])["b"]
        m_star = r[j] * b.mean()
        eps = 1e-12 * np.abs(b).max()
        assert lo[j] <= m_star + eps <= up[j] + 2 * eps
    assert lo[m] == up[m] == 1.0 and lo[m + 1] == up[m + 1] == 24.0
    assert np.isnan(lo[m + 2]) and st[m + 2] == 2
    assert up[m + 3] < 0 and lo[m + 4] > 0 and up[m + 5] < 0      # Figs. 5, 6, 7
    assert int(nodes.item()) > 0


# --------------------------------------------------------------------------
# NEXT-3: candidate-set filtering
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [0, 1, 4095, 4096, 4097, 1_000_003])
def test_select_valid_parity(n):
    rng = np.random.default_rng(n)
    flags = rng.choice(np.array([0, 1, 2, 3, 5, 6], np.uint8), size=n, p=[.3, .4, .05, .05, .1, .1])
    group = rng.integers(0, 1000, size=n).astype(np.int32)
    f = torch.from_numpy(flags).cuda()
    g = torch.from_numpy(group).cuda()
    ids, c, counts = hv.select_valid(f, g, 1000)
    torch.cuda.synchronize()
    ref_ids, ref_counts = oracle.select_valid(flags, group, 1000)
    assert c == ref_ids.size
    assert np.array_equal(ids.cpu().numpy(), ref_ids)
    assert np.array_equal(counts.cpu().numpy(), ref_counts)
    if n > 1:                                   # misaligned flags view (scalar path)
        ids2, c2, _ = hv.select_valid(f[1:])
        torch.cuda.synchronize()
        assert np.array_equal(ids2.cpu().numpy(), oracle.select_valid(flags[1:])[0])
        # flags and group views offset by one element: the group ids no longer take the
        # 16-B vector loads (scalar fallback) and the staged ordered write starts mid-row
        ids3, c3, counts3 = hv.select_valid(f[1:], g[1:], 1000)
        torch.cuda.synchronize()
        ref3_ids, ref3_counts = oracle.select_valid(flags[1:], group[1:], 1000)
        assert c3 == ref3_ids.size
        assert np.array_equal(ids3.cpu().numpy(), ref3_ids)
        assert np.array_equal(counts3.cpu().numpy(), ref3_counts)


def test_select_valid_config3_pipeline():
    """The paper's motivating pipeline on a config-3 slice: check candidates, keep the valid
    ones, count valid candidates per grid cell (candidate h uses cell h mod 99^3)."""
    start, count = 5_000_000, 2_000_000
    verts, idx = hexgen.indexed_config(3, start=start, count=count)
    f, _ = gpu_indexed(verts, idx)
    cells = ((np.arange(start, start + count) % (99 ** 3))).astype(np.int32)
    ids, c, counts = hv.select_valid(torch.from_numpy(f).cuda(), torch.from_numpy(cells).cuda(), 99 ** 3)
    torch.cuda.synchronize()
    ref_ids, ref_counts = oracle.select_valid(f, cells, 99 ** 3)
    assert np.array_equal(ids.cpu().numpy(), ref_ids) and np.array_equal(counts.cpu().numpy(), ref_counts)
    sel = np.random.default_rng(3).choice(count, 20000, replace=False)
    ref = oracle.check_indexed(verts, idx[sel])
    assert_flags_match(f[sel], ref)


# --------------------------------------------------------------------------
# NEXT-4: linear quadrangles
# --------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 255, 257, 100_003])
def test_quad_parity(n):
    coords = hexgen.quad_soa(n, 0.45, seed=n)
    f, J = hv.check_quad_soa(torch.from_numpy(coords).cuda(), J=True)
    torch.cuda.synchronize()
    f, J = f.cpu().numpy(), J.cpu().numpy()
    ref = oracle.check_quad_soa(coords)
    assert np.array_equal(f, ref["flags"])                    # exact signs on both sides: no exclusions
    assert np.array_equal(J, ref["J"])                        # same two products and difference
    if n > 1000:
        assert np.any(f == hv.INVALID) and np.any(f == hv.VALID)


def test_quad_degenerate_and_special():
    """Collinear / coincident nodes (exact zeros decided exactly), NaN, bowtie, chevron."""
    rng = np.random.default_rng(71)
    Q = [hexgen.UNIT_SQUARE, hexgen.UNIT_SQUARE[[0, 1, 3, 2]], np.array([[0, 0], [2, 0], [1, .5], [0, 2]], float)]
    for _ in range(2000):
        P = np.round((hexgen.UNIT_SQUARE + rng.uniform(-0.5, 0.5, size=(4, 2))) * 4) / 4   # dyadic grid: many zeros
        if rng.random() < 0.3:
            i, j = rng.choice(4, 2, replace=False)
            P[j] = P[i]
        Q.append(P)
    N = hexgen.UNIT_SQUARE.copy(); N[1, 1] = np.nan
    Q.append(N)
    Q = np.stack(Q)
    coords = np.ascontiguousarray(Q.reshape(len(Q), 8).T)
    f, _ = hv.check_quad_soa(torch.from_numpy(coords).cuda())
    torch.cuda.synchronize()
    f = f.cpu().numpy()
    ref = oracle.check_quad_soa(coords)
    assert np.array_equal(f, ref["flags"])
    assert f[0] == hv.VALID and f[1] == hv.INVALID and f[2] == hv.INVALID and f[-1] == hv.NONFINITE
    assert ref["near"].sum() > 100                             # the exact path was exercised


# --------------------------------------------------------------------------
# properties of the CUDA path that hold at any size (checked without the oracle)
# --------------------------------------------------------------------------

def test_power_of_two_scaling_and_translation_invariance():
    """Scaling all coordinates by 2^k scales every det J value, and so every computed
    coefficient, by exactly 8^k (no rounding changes); verdicts are unchanged.  A
    translation by a small dyadic vector changes rounding only: verdicts of hexes the
    oracle does not mark near-boundary are unchanged."""
    coords = hexgen.ragged_soa(50_000, seed=81, amp=0.45)
    f0, k0 = gpu_soa(coords, coeffs=True)
    for s in (2.0 ** -30, 2.0 ** 7):
        f, k = gpu_soa(coords * s, coeffs=True)
        assert np.array_equal(f, f0)
        assert np.array_equal(k, k0 * s ** 3)
    ref = oracle.check_soa(coords)
    ft, _ = gpu_soa(coords + 0.125)
    sure = ref["near"] == 0
    assert np.array_equal(ft[sure], f0[sure])


def test_tiny_scales_keep_the_verdict():
    """Hexes scaled by 2^-340 .. 2^-360 (Bezier coefficients down to ~2^-1080, subnormal or
    below: their high words no longer carry the sign of tiny positive values).  An
    exact power-of-two scaling does not change any exact sign, so the verdict must equal the
    oracle's on the unscaled hex; the subdivision kernel normalises such roots before splitting.
    The SUBDIVIDED bit may differ (pass 1 cannot confirm Step 4 on subnormal coefficients)."""
    base = hexgen.soa_config(3000, 0.35, 71)
    ref = oracle.check_soa(base)
    sure = ref["near"] == 0
    cube = hexgen.nodes_to_soa(pins.KAPPA.astype(float)[None])
    for e in (-340, -352, -360):
        f, _ = gpu_soa(np.ldexp(base, e))
        assert np.array_equal((f & 3)[sure], (ref["flags"] & 3)[sure]), e
        fc, _ = gpu_soa(np.ldexp(cube, e))
        assert (fc[0] & 3) == hv.VALID, (e, fc[0])


def test_node_relabelling_by_cube_rotation_preserves_verdict():
    """A proper rotation of the reference cube relabels the nodes (det J composed with an
    orientation-preserving map of [0,1]^3): validity is unchanged."""
    coords = hexgen.ragged_soa(20_000, seed=82, amp=0.45)
    X = hexgen.soa_to_nodes(coords)
    f0, _ = gpu_soa(coords)
    ref = oracle.check_soa(coords)
    sure = ref["near"] == 0
    # rotation by 90 degrees about zeta: node k -> image of its reference corner
    perm = [1, 2, 3, 0, 5, 6, 7, 4]
    f1, _ = gpu_soa(hexgen.nodes_to_soa(X[:, perm]))
    assert np.array_equal((f1 & 3)[sure], (f0 & 3)[sure])


def test_debug_build_invariants(tmp_path):
    """The HEXVAL_DEBUG build traps on any violated stack-capacity / index invariant
    (compute-sanitizer is not available on the GPU pool): run every entry point on small
    and adversarial inputs against it in a subprocess and require a clean exit."""
    import subprocess
    import sys
    from paper_1706_01613_b200 import build as hvbuild
    if not os.path.exists(hvbuild.DEBUG_LIB):
        pytest.skip("libhexval_debug.so not built")
    root = hexgen.__file__.rsplit("/", 2)[0]
    env = dict(os.environ, HEXVAL_LIB="libhexval_debug.so")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize_small.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


def test_small_stack_capacity_gives_the_same_results(tmp_path):
    """K4's capacity-adaptive pop size (hexval.cu "Stack capacity"): a build with 416 stack
    slots per warp (and the invariant traps on) throttles its pops down to the one-node
    depth-first mode on config-4 trees, wide random Bezier trees and the NEXT-1 bounds --
    verdicts, SUBDIVIDED bits, depth-cap outcomes and bounds must equal the default build's."""
    import subprocess
    import sys
    from paper_1706_01613_b200 import build as hvbuild
    if not os.path.exists(hvbuild.SMALLCAP_LIB):
        pytest.skip("libhexval_smallcap.so not built")
    root = hexgen.__file__.rsplit("/", 2)[0]
    sys.path.insert(0, os.path.join(root, "tools"))
    import smallcap_check
    ours = smallcap_check.run()
    out = str(tmp_path / "smallcap.npz")
    env = dict(os.environ, HEXVAL_LIB="libhexval_smallcap.so")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "smallcap_check.py"), out], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and r.stdout.startswith("ok libhexval_smallcap.so"), r.stdout + r.stderr
    small = np.load(out)
    for key in ("f4", "fb", "s", "n_valid", "n_invalid", "n_undetermined"):
        assert np.array_equal(ours[key], small[key]), key
    # the NEXT-1 bounds depend on the traversal order (a node is split iff its minimum is below the
    # upper bound *found so far* minus tol), so the two builds' certified intervals may differ --
    # but both contain min det J: they overlap, and their ends differ by at most the wider width
    lo_a, up_a, lo_b, up_b = ours["lo"], ours["up"], small["lo"], small["up"]
    assert np.array_equal(np.isnan(lo_a), np.isnan(lo_b)) and not np.isnan(lo_a).any()
    width = np.maximum(up_a - lo_a, up_b - lo_b)
    assert np.all(lo_a <= up_a) and np.all(lo_b <= up_b)
    assert np.all(np.maximum(lo_a, lo_b) <= np.minimum(up_a, up_b))
    assert np.all(np.abs(lo_a - lo_b) <= width) and np.all(np.abs(up_a - up_b) <= width)
    assert float(np.mean(lo_a == lo_b)) > 0.5                                # mostly the same trees
    assert int((ours["f4"] & hv.FLAG_SUBDIVIDED != 0).sum()) > 5000          # K4 really ran
    assert set((ours["fb"] & 3).tolist()) >= {hv.INVALID, hv.VALID, hv.UNDETERMINED}   # all verdicts on the Bezier trees


# --------------------------------------------------------------------------
# large sizes: 64-bit plane offsets (p * n * 8 > 2^32) and long queues
# --------------------------------------------------------------------------

def test_large_soa_input_sampled():
    """n = 2^28 + 3 hexes (51.5 GB of coordinates): plane offsets exceed 32 bits, the
    persistent kernels run ~3600 tiles per CTA; generated on the device from a seeded
    torch generator (perturbed unit cubes, amplitude 0.45), checked on a sample that
    includes the last hexes of the array."""
    n = (1 << 28) + 3
    free, _ = torch.cuda.mem_get_info()
    if free < 60e9:
        pytest.skip("needs ~60 GB of free device memory")
    g = torch.Generator(device="cuda").manual_seed(1234)
    coords = torch.rand((24, n), generator=g, device="cuda", dtype=torch.float64).mul_(0.9).sub_(0.45)
    cube = torch.from_numpy(pins.KAPPA.astype(np.float64).reshape(24, 1)).cuda()
    coords.add_(cube)
    stats = hv.Stats()
    f, _ = hv.check_soa(coords, stats=stats)
    torch.cuda.synchronize()
    st = stats.read()
    assert st["n_valid"] + st["n_invalid"] + st["n_undetermined"] + st["n_nonfinite"] == n
    rng = np.random.default_rng(9)
    sel = np.unique(np.concatenate([rng.choice(n, 20000, replace=False), np.arange(n - 300, n)]))
    sub_ids = torch.nonzero((f & 4) > 0).flatten()[:5000].cpu().numpy()
    sel = np.unique(np.concatenate([sel, sub_ids]))
    sel_t = torch.from_numpy(sel).cuda()
    sample = coords.index_select(1, sel_t).cpu().numpy()
    fs = f.index_select(0, sel_t).cpu().numpy()
    del coords
    torch.cuda.empty_cache()
    ref = oracle.check_soa(sample)
    assert_flags_match(fs, ref, allow_near=True)
    assert ref["near"].sum() <= 2


def test_large_indexed_input_sampled():
    """n = 2^28 + 5 candidate hexes (8.6 GB of int32 connectivity): grid cells of a jittered
    100^3 vertex grid chosen by a seeded device generator; sampled parity incl. the tail."""
    n = (1 << 28) + 5
    free, _ = torch.cuda.mem_get_info()
    if free < 20e9:
        pytest.skip("needs ~20 GB of free device memory")
    verts = hexgen.grid_vertices(100, 0.2, 3)
    g = torch.Generator(device="cuda").manual_seed(4321)
    cells = torch.randint(0, 99 ** 3, (n,), generator=g, device="cuda", dtype=torch.int64)
    ci, cj, ck = cells % 99, (cells // 99) % 99, cells // (99 * 99)
    off = torch.from_numpy(pins.KAPPA.astype(np.int64)).cuda()
    idx = ((ci[:, None] + off[None, :, 0]) + 100 * ((cj[:, None] + off[None, :, 1]) + 100 * (ck[:, None] + off[None, :, 2]))).to(torch.int32)
    del cells, ci, cj, ck
    v = torch.from_numpy(verts).cuda()
    f, _ = hv.check_indexed(v, idx)
    torch.cuda.synchronize()
    rng = np.random.default_rng(10)
    sel = np.unique(np.concatenate([rng.choice(n, 20000, replace=False), np.arange(n - 300, n)]))
    sel_t = torch.from_numpy(sel).cuda()
    idx_s = idx.index_select(0, sel_t).cpu().numpy()
    fs = f.index_select(0, sel_t).cpu().numpy()
    del idx
    torch.cuda.empty_cache()
    ref = oracle.check_indexed(verts, idx_s)
    assert_flags_match(fs, ref)
