"""Host-side pieces of bench.py that need no GPU (-m "not gpu"): the workload recipes,
the algorithmic-byte counts the roofline divides by, and the reference arm's JSON line
(the CPU oracle timed on a bounded sample, BASELINE.json metric and unit)."""
import json
import subprocess
import sys
import os

import numpy as np

import bench
import hexgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_algorithmic_bytes_match_survey():
    """193 B/hex SoA; indexed = 32 B ids + vertex bytes + 1 B flag."""
    assert bench.algorithmic_bytes("soa", 10, None) == 1930
    verts = np.zeros((201 ** 3, 3))
    assert bench.algorithmic_bytes("indexed", 200 ** 3, (verts, None)) == 33 * 200 ** 3 + 24 * 201 ** 3


def test_make_inputs_weak_shards_are_disjoint_slices_of_the_stream():
    layout, n, (c0,) = bench.make_inputs(0, 0)
    assert layout == "soa" and n == 10_000 and c0.shape == (24, n)
    _, _, (c1,) = bench.make_inputs(0, 1)                     # rank 1: hexes n .. 2n-1
    assert np.array_equal(c1, hexgen.soa_config(n, 0.25, 0, start=n))
    assert not np.array_equal(c0, c1)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                          "--steps", "1", "--warmup", "0", "--cpu-seconds", "0.2"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == "hex/s"
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "hex/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def _dry_run(cfg: int, gpus: int = 2):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--dry-run",
                          "--config", str(cfg)], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])


def test_gpus_flag_spawns_ranks_with_disjoint_shards_and_summed_verdicts():
    """`bench.py --gpus 2` without torchrun launches 2 ranks itself (here with --dry-run: gloo,
    no GPU); each rank owns a distinct range of the workload and the verdict counters are
    summed over ranks."""
    for cfg in (1, 3):
        line = _dry_run(cfg)
        assert line["world"] == 2
        (a, b) = sorted(line["shards"], key=lambda d: d["rank"])
        assert a["range"][1] <= b["range"][0] and a["range"][0] < a["range"][1]
        assert a["first_coord"] != b["first_coord"]            # distinct hexes, not a copy
        v = line["verdicts_summed"]
        assert sum(v.values()) == 2 * line["sample_per_rank"] and v["valid"] > 0


def test_config2_weak_shards_are_distinct_slabs():
    _, va, ia = bench.shard_inputs(2, 0, 0, 10)
    _, vb, ib = bench.shard_inputs(2, 1, 0, 10)
    assert np.array_equal(ia, ib)                              # same local connectivity
    assert vb[:, 2].min() > 199 and va[:, 2].max() < 201       # slab 1 stacked on slab 0
    m = 201
    assert np.array_equal(va[200 * m * m:], vb[:m * m])        # shared boundary plane
