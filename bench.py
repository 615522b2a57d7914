#!/usr/bin/env python
"""Benchmark of the hexahedron-validity hot path on B200 (one JSON line on rank 0).

Workload (BASELINE.json configs[1], the configuration the metric is quoted on):
10M independent hexahedra, fp64 SoA, unit-cube corners + U[-0.35, 0.35]^3
noise.  A step is one whole pass of the hot path over that batch: pass 1 (20
determinants, 27 Bezier coefficients, classification, compaction), the exact
sign kernel and the subdivision kernel, through the C ABI
(hexval_check_soa_ex).  Inputs are resident in HBM; 1.92 GB of input per step
is far above the 126 MB L2, so no L2 flush is needed between steps.

Multi-GPU (torchrun): every rank checks its own 10M hexes (weak scaling; the
hexes are independent, so there is no data-path collective); timing is the
max over ranks of CUDA-event time.

``--impl reference`` times the CPU oracle (oracle/, all host cores) on a
bounded sample of the same workload and prints the same line with
"impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "hexahedra validated/sec (fp64, 1 B200); % of HBM roofline; subdivision rate"
UNIT = "hex/s"
FALLBACK_HBM_GBS = 6650.0
# fp64 operations per subdivision node: 147 new de Casteljau values, one add and one
# multiply each; peak = 148 SMs x 64 FP64 lanes x 1.965 GHz
FP64_OPS_PER_NODE = 294
# fp64 operations per hex of pass 1 (36 + 36 vector components, 180 for the 20 triple
# products, 19 Step-2 compares, ~90 for T~, 18 Step-4 compares)
FP64_OPS_PER_HEX = 381
FP64_PEAK_GOPS = 148 * 64 * 1.965            # datasheet-level fallback when the probe cannot run
K4_L1_BYTES_PER_NODE = 2 * 224               # K4's stack round trip: 7 x 32 B pushed + 7 x 32 B popped per node
K4_L1_PEAK_GBS = 148 * 64 * 1.965            # L1 data pipe at 64 B/clk/SM for 256-bit accesses (ncu, K4)
CONFIG_DESC = {
    0: "config0: 10k perturbed unit cubes, SoA fp64, noise U[-0.25,0.25]^3, seed 0",
    1: "config1: 10M perturbed unit cubes, SoA fp64, noise U[-0.35,0.35]^3, seed 1",
    2: "config2: 200^3 structured grid, 201^3 vertices jittered +-0.3, int32 connectivity, seed 2",
    3: "config3: 40M candidate hexes on a 100^3 jittered grid (+-0.2), p_swap 0.1, int32 connectivity, seed 3",
    4: "config4: 4M adversarial SoA hexes (pushed-corner parallelepipeds + twisted prisms), seed 4",
}
L2_NOTE = {
    0: "inputs 1.9 MB fit in L2 (small parity case; not a bench line)",
    1: "no flush: 1.92 GB of input per step >> 126 MB L2",
    2: "no flush: 256 MB connectivity per step >> L2; 195 MB vertex array partially L2-reused by design",
    3: "no flush: 1.28 GB connectivity per step >> L2; 24 MB vertex array L2-resident by design",
    4: "no flush: 768 MB of input per step >> L2",
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", type=int, default=1, choices=sorted(CONFIG_DESC))
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--clock-ms", type=float, default=0.5,
                   help="NVML clock sampling period during the timed region (ms)")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the secondary block (config-4 subdivision and config-3 pass 1 against the "
                        "measured FP64 peak)")
    p.add_argument("--dry-run", action="store_true",
                   help="no GPU: shard ranges + oracle verdict counts on a sample of each rank's shard, summed "
                        "over ranks (gloo); tests the multi-rank plumbing on CPU")
    p.add_argument("--workers", type=int, default=min(16, os.cpu_count() or 1),
                   help="host processes generating the synthetic inputs")
    p.add_argument("--no-cupti", action="store_true",
                   help="skip the torch.profiler (CUPTI) kernel-duration pass (e.g. under ncu)")
    p.add_argument("--graph", action="store_true",
                   help="also time the call captured in a CUDA graph (launch-bound small batches)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=8.0, help="target wall time of the CPU baseline sample")
    p.add_argument("--ref-seconds", type=float, default=150.0,
                   help="reference arm: wall-time budget of all warm-up + timed steps (whole configuration per "
                        "step when it fits, else a prefix sample)")
    p.add_argument("--coeffs", action="store_true",
                   help="also write the 27 Bezier coefficients per hex (409 B/hex, SURVEY.md 8(d))")
    p.add_argument("--op", choices=["check", "quality", "screen", "bounds", "select", "quads"], default="check",
                   help="check: the hot path (headline); quality: NEXT-2 corner screening kernel; "
                        "bounds: NEXT-1 certified min det J bounds; select: NEXT-3 candidate filtering "
                        "(on the config's flags); quads: NEXT-4 linear quadrangles (10M, noise 0.35)")
    p.add_argument("--rel-tol", type=float, default=1e-3, help="NEXT-1 tolerance (relative to max|b|)")
    p.add_argument("--variant", choices=["ldg", "wtma", "cp", "bulk"], default=None,
                   help="pass-1 kernel variant for SoA inputs (sets HEXVAL_PASS1; default: the library's)")
    args = p.parse_args()
    if args.variant:
        os.environ["HEXVAL_PASS1"] = args.variant
    return args


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per pass-1 launch from the committed ncu --set full capture, if any."""
    path = os.path.join(ROOT, "profiles", "pass1_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d
    except Exception:
        return None


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (NVML)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int, period_s: float = 0.010):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self.period_s = period_s
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.period_s)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if self.nv is None or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        reasons = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------
def cupti_kernel_us(step, steps: int) -> dict:
    """Mean device duration (us) per kernel name over `steps` calls, from CUPTI
    activity records (torch.profiler): the kernels' own execution time, without
    the launch bubble an event pair around a single kernel includes."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
    per = {}
    for ev in p.events():
        if ev.device_type.name != "CUDA":
            continue
        key = ev.name.split("<")[0].split("::")[-1].strip()
        d = per.setdefault(key, [0, 0.0])
        d[0] += 1
        d[1] += ev.time_range.end - ev.time_range.start
    return {k: tot / c for k, (c, tot) in per.items()}, {k: c for k, (c, _) in per.items()}


def spawn_ranks(gpus: int) -> int:
    """`bench.py --gpus N` without a process group: re-run this command under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1 and return its exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(gpus: int, dry_run: bool = False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if dry_run:
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if gpus != world:
        raise SystemExit(f"--gpus {gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    return world, rank, local


def dist_max(x: float, world: int) -> float:
    from paper_1706_01613_b200 import shard
    return shard.max_over_ranks(x) if world > 1 else x


def barrier(world: int):
    from paper_1706_01613_b200 import shard
    if world > 1:
        shard.barrier()


# ---------------------------------------------------------------------------
# CPU oracle (baseline / reference arm)
# ---------------------------------------------------------------------------
def oracle_sample(cfg: int, m: int, start: int = 0, nthreads: int = 0, rank: int = 0, workers: int = 1):
    """A callable running the oracle on hexes start..start+m-1 of this rank's shard of `cfg`."""
    import oracle
    layout, *arrays = shard_inputs(cfg, rank, start, m, workers)
    if layout == "soa":
        coords = arrays[0]
        return lambda: oracle.check_soa(coords, nthreads=nthreads)
    verts, idx = arrays
    return lambda: oracle.check_indexed(verts, idx, nthreads=nthreads)


def oracle_rate(cfg: int, seconds: float, start: int = 0, gpu_flags=None, workers: int = 1):
    """Time the oracle, as it stands, on a bounded prefix sample of the workload (all host threads).

    With `gpu_flags` (the flags of a timed GPU step, host copy) the sample's oracle verdicts are also
    compared with them: `parity` = flag mismatches on hexes the oracle does not mark near-boundary,
    and the near-boundary count (BASELINE north_star: must be 0 on configs 0-3)."""
    import hexgen
    import oracle
    n = hexgen.config_size(cfg)
    cores = oracle.num_threads(0)
    probe_n = min(n, 20_000)
    run = oracle_sample(cfg, probe_n, start)
    run()                                                     # warm (thread pool, page-in)
    t0 = time.perf_counter()
    run()
    r0 = probe_n / (time.perf_counter() - t0)
    m = int(min(n, max(probe_n, r0 * seconds)))
    run = oracle_sample(cfg, m, start, workers=workers)
    t0 = time.perf_counter()
    ref = run()
    dt = time.perf_counter() - t0
    parity = None
    if gpu_flags is not None:
        import numpy as np
        g = np.asarray(gpu_flags[start:start + m])
        near = ref["near"].astype(bool)
        parity = {"compared": int(m), "mismatches": int(np.sum((g != ref["flags"]) & ~near)),
                  "near_boundary": int(near.sum()),
                  "what": "whole flags byte of the last timed GPU step vs the oracle on the same hexes"}
    # one thread on a smaller slice of the same stream (per-core rate, the unit of the
    # paper's ~6 M hex/s on one core)
    m1 = max(1000, min(m, int(m / max(1, cores) / 4)))
    run1 = oracle_sample(cfg, m1, start, nthreads=1)
    t1 = time.perf_counter()
    run1()
    dt1 = time.perf_counter() - t1
    out = {"value": m / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"hexes {start}..{start + m - 1} of {CONFIG_DESC[cfg]} ({m} hexes, {dt:.2f} s wall on {cores} threads)",
           "single_thread": {"value": m1 / dt1, "unit": UNIT, "sample": f"hexes {start}..{start + m1 - 1}, 1 thread"}}
    if parity is not None:
        out["parity"] = parity
    return out


def run_reference(args, world, rank):
    """The reference arm: the CPU oracle, as it stands, on the host cores, timed per step on the
    whole configuration when the K steps fit the time budget (--ref-seconds), else on a prefix
    sample of the configuration sized to it."""
    import oracle
    if rank != 0:
        return 0
    layout, n, host = make_inputs(args.config, 0, args.workers)
    cores = oracle.num_threads(0)

    def run(m):
        if layout == "soa":
            return oracle.check_soa(np.ascontiguousarray(host[0][:, :m]))
        return oracle.check_indexed(host[0], np.ascontiguousarray(host[1][:m]))

    probe = min(n, 20_000)
    run(probe)                                                # warm: thread pool, page-in
    t0 = time.perf_counter()
    run(probe)
    est = (time.perf_counter() - t0) * n / probe             # seconds for the whole configuration
    budget = args.ref_seconds / max(1, args.steps + args.warmup)
    m = n if est <= budget else max(probe, int(n * budget / est))
    for _ in range(args.warmup):
        run(min(m, probe * 4))
    per_step = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run(m)
        per_step.append(m / (time.perf_counter() - t0))
    value = statistics.median(per_step)
    whole = m == n
    sample = (f"hexes 0..{m - 1} of {CONFIG_DESC[args.config]} ({m} hexes per step"
              f"{', the whole configuration' if whole else ', a prefix sample'}, {cores} threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * n / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIG_DESC[args.config], "n_hexes": n, "layout": layout,
                   "note": ("each step runs the CPU oracle (oracle/, as it stands) on the whole configuration"
                            if whole else "each step times the CPU oracle (oracle/, as it stands) on a bounded "
                            "prefix sample; ms_per_step is extrapolated to the full batch")},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def shard_inputs(cfg: int, rank: int, offset: int = 0, count: int | None = None, workers: int = 1):
    """(layout, *arrays) of hexes offset..offset+count-1 of rank `rank`'s weak-scaling shard.

    Every rank gets its own, distinct hexes of the configuration's family:
    configs 0, 1, 4: the synthetic hexes r*n .. r*n+n-1 of the stream; config 3: candidates
    r*n .. r*n+n-1 of the candidate stream on the shared 100^3 grid (the 24 MB vertex array is
    replicated); config 2: the k-slab r of a 200 x 200 x 200N structured grid (its own 201^3
    vertices, boundary plane shared with slab r-1)."""
    import hexgen
    from paper_1706_01613_b200 import shard
    start, n = shard.weak_shard(hexgen.config_size(cfg), rank)
    count = n - offset if count is None else count
    if cfg == 2:
        return ("indexed", *hexgen.indexed_config(2, start=offset, count=count, slab=rank))
    out = hexgen.make(cfg, start=start + offset, count=count, workers=workers)
    return ("soa", out[1]) if out[0] == "soa" else ("indexed", out[1], out[2])


def shard_range(cfg: int, rank: int) -> tuple[int, int]:
    """[first, last) global hex index of rank `rank`'s shard (config 2: global cell ids of its k-slab)."""
    import hexgen
    from paper_1706_01613_b200 import shard
    start, n = shard.weak_shard(hexgen.config_size(cfg), rank)
    return start, start + n


def make_inputs(cfg: int, rank: int, workers: int = 1):
    """Host arrays of this rank's shard (weak scaling: every rank its own n hexes)."""
    layout, *arrays = shard_inputs(cfg, rank, workers=workers)
    n = arrays[0].shape[1] if layout == "soa" else arrays[1].shape[0]
    return layout, n, tuple(arrays)


def algorithmic_bytes(layout: str, n: int, arrays, coeffs: bool = False) -> int:
    """Compulsory HBM bytes of one pass-1 launch: inputs once + 1 flag byte/hex
    (+ 27 fp64 coefficients per hex when they are written)."""
    out = n + (216 * n if coeffs else 0)
    if layout == "soa":
        return 192 * n + out
    verts, idx = arrays
    return 32 * n + 24 * verts.shape[0] + out


def run_ours(args, world, rank, local):
    import torch

    import paper_1706_01613_b200 as hv

    torch.cuda.set_device(local)
    cfg = args.config
    desc = CONFIG_DESC[cfg]
    layout, n, host = make_inputs(cfg, rank, args.workers)
    dev = [torch.from_numpy(a).cuda() for a in host]
    flags = torch.empty(n, dtype=torch.uint8, device="cuda")
    coeffs = torch.empty((27, n), dtype=torch.float64, device="cuda") if args.coeffs else None
    stream = torch.cuda.current_stream()

    def step(profile=None, stats=None):
        if layout == "soa":
            hv.check_soa(dev[0], flags=flags, coeffs=coeffs, profile=profile, stats=stats)
        else:
            hv.check_indexed(dev[0], dev[1], flags=flags, coeffs=coeffs, profile=profile, stats=stats)

    # untimed: verdict / subdivision statistics of this workload
    stats = hv.Stats()
    step(stats=stats)
    torch.cuda.synchronize()
    st = stats.read()
    if world > 1:                                                      # whole-job verdict counts
        from paper_1706_01613_b200 import shard
        md = st["max_depth"]
        st = dict(zip(st.keys(), shard.sum_over_ranks(list(st.values()))))
        st["max_depth"] = int(shard.max_over_ranks(md))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # timed region 1 (the headline): the product call exactly as a user makes it
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, args.clock_ms * 1e-3) as clk:
        barrier(world)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms_total = ev0.elapsed_time(ev1)
    ms_step = dist_max(ms_total / args.steps, world)
    flags_timed = flags.cpu().numpy() if rank == 0 and world == 1 and not args.no_cpu_baseline else None
    graph = None
    if args.graph:
        # the same call captured once in a CUDA graph and replayed K times
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            step()
        for _ in range(args.warmup):
            g.replay()
        barrier(world)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            g.replay()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        ms_g = dist_max(ev0.elapsed_time(ev1) / args.steps, world)
        graph = {"ms_per_step": ms_g, "value": world * n / (ms_g * 1e-3),
                 "timing": "torch.cuda.CUDAGraph of one call, K replays between two CUDA events"}
    # timed region 2: the same K steps with the library's per-kernel events
    # (hexval_profile) for the roofline and the phase split
    prof = hv.Profile()
    prof.read()                                                        # reset
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    phases = {}

    def drain():                                                       # the profile holds 256 calls
        for k, v in prof.read().items():
            acc = phases.setdefault(k, {"ms": 0.0, "launches": 0})
            acc["ms"] += v["ms"]
            acc["launches"] += v["launches"]

    ms_prof = 0.0
    done = 0
    while done < args.steps:
        chunk = min(200, args.steps - done)
        ev2.record(stream)
        for _ in range(chunk):
            step(profile=prof)
        ev3.record(stream)
        torch.cuda.synchronize()
        ms_prof += ev2.elapsed_time(ev3)
        drain()
        done += chunk
    barrier(world)
    ms_step_prof = dist_max(ms_prof / args.steps, world)
    if args.no_cupti:
        kern_us = {"skipped": "--no-cupti"}
    else:
        try:
            kern_us, _ = cupti_kernel_us(step, min(args.steps, 20))
        except Exception as exc:                                      # profiler unavailable: report without it
            kern_us = {"error": str(exc)[:200]}
    p1_names = ("soa_cp_kernel", "idx_cp_kernel", "plain_kernel", "pass1_soa_wtma_kernel")
    p1_us = next((v for k, v in kern_us.items() if k in p1_names), None)
    k4_us = kern_us.get("subdiv_kernel")
    # every rank joins both reductions (-1: not measured on this rank)
    p1_us = dist_max(p1_us if isinstance(p1_us, float) else -1.0, world)
    k4_us = dist_max(k4_us if isinstance(k4_us, float) else -1.0, world)
    p1_us = p1_us if p1_us > 0 else None
    k4_us = k4_us if k4_us > 0 else None
    per = {k: v["ms"] / max(1, v["launches"]) for k, v in phases.items()}
    pass1_ms = dist_max(per["pass1"], world)
    subdiv_ms = dist_max(per["subdiv"], world)
    if k4_us is not None:
        subdiv_ms = k4_us * 1e-3                                       # CUPTI kernel duration (see roofline.timing)

    value = world * n / (ms_step * 1e-3)
    peak, peak_src = measured_peaks()
    algo = algorithmic_bytes(layout, n, host, args.coeffs)
    achieved_ev = algo / (pass1_ms * 1e-3) / 1e9
    # the kernel's own duration: CUPTI activity records when available (an event
    # pair around a single kernel adds a launch bubble of 10-40 us here, see
    # profiles/r01/SUMMARY.md "Event bubbles"), else the event pair
    p1_s = p1_us * 1e-6 if p1_us else pass1_ms * 1e-3
    achieved = algo / p1_s / 1e9
    traffic = ncu_traffic()
    roofline = {
        "bound": "hbm", "kernel": "pass1 (K1 SoA cp.async double-buffered / K2 indexed cp.async gather)",
        "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "duration_source": "cupti" if p1_us else "events",
        "pass1_us": p1_s * 1e6,
        "achieved_events": achieved_ev, "frac_events": achieved_ev / peak,
        "peak_source": peak_src,
        "algorithmic_bytes_per_launch": algo,
        "traffic": (traffic["dram_bytes_per_hex"] * n if traffic and cfg == 1 and not args.coeffs else None),
        "traffic_source": (traffic.get("source") if traffic and cfg == 1 and not args.coeffs else None),
        "frac_of_8TBs_nominal": achieved / 8000.0,
        "pass1_share_of_step": p1_s * 1e3 / ms_step,
        "kernel_us_cupti": kern_us,
        "phase_ms_per_step_events": per,
        "ms_per_step_profiled": ms_step_prof,
        "pass1_only_hex_per_s": n / p1_s,
        "timing": ("pass1_us: mean kernel duration over min(K, 20) calls from CUPTI activity records (torch.profiler), "
                   "live on the timed stream; *_events: CUDA events recorded by the library around each kernel over a "
                   "second run of the K timed steps (ms_per_step_profiled is that run's step time)"),
    }
    subdivision = {
        "rate": st["n_subdivided"] / (world * n),
        "nodes_per_step": st["n_nodes"],
        "subdiv_kernel_ms": subdiv_ms,
        "nodes_per_s": (st["n_nodes"] / (subdiv_ms * 1e-3)) if subdiv_ms > 0 and st["n_nodes"] else None,
        "lane_use": (st["n_nodes"] / st["n_lane_steps"]) if st.get("n_lane_steps") else None,
        "fp64_ops_per_node": FP64_OPS_PER_NODE,
        "fp64_achieved_gops": (st["n_nodes"] * FP64_OPS_PER_NODE / (subdiv_ms * 1e-3) / 1e9) if subdiv_ms > 0 and st["n_nodes"] else None,
        "fp64_peak_gops_at_max_clock": FP64_PEAK_GOPS,
    }

    # end to end through the host API: pinned inputs, H2D + kernels + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        del dev
        torch.cuda.empty_cache()
        pins_ = [torch.from_numpy(a).pin_memory() for a in host]
        fl_h = torch.empty(n, dtype=torch.uint8).pin_memory()

        def host_step():
            if layout == "soa":
                hv.check_soa_host(pins_[0], fl_h)
            else:
                hv.check_indexed_host(pins_[0], pins_[1], fl_h)

        host_step()                                                    # warm
        torch.cuda.synchronize()
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            host_step()
        dt = time.perf_counter() - t0
        dt = dist_max(dt, world)
        h2d = sum(a.nbytes for a in host)
        # the link's own ceiling: best of 3 plain pinned -> device copies of the largest input array
        big = pins_[0]
        dst = torch.empty(big.shape, dtype=big.dtype, device="cuda")
        link = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(big, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            link = max(link, big.numel() * big.element_size() / (e0.elapsed_time(e1) * 1e-3) / 1e9)
        del dst
        e2e = {"value": world * n * args.e2e_steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": n,
               "h2d_gbs_achieved": h2d * args.e2e_steps / dt / 1e9,
               "h2d_gbs_link": link,
               "frac_of_link": (h2d * args.e2e_steps / dt / 1e9) / link if link else None,
               "timing": "host wall clock around the synchronous hexval_check_*_host call (H2D of pinned inputs, kernels, D2H of flags), max over ranks",
               "steps": args.e2e_steps}
        if not torch.equal(flags.cpu(), fl_h):
            e2e["warning"] = "host-path flags differ from device-path flags"

    secondary = None
    if world == 1 and not args.no_secondary:
        del flags
        torch.cuda.empty_cache()
        secondary = run_secondary(args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_rate(cfg, args.cpu_seconds, gpu_flags=flags_timed, workers=args.workers)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "n_hexes_per_rank": n, "global_hexes": world * n, "layout": layout,
                       "parallelism": (f"independent shards x{world} (weak scaling; multi-GPU unmeasured on hardware until a "
                            "driver SCALE run)") if world > 1 else "single GPU",
                       "l2": L2_NOTE[cfg],
                       "pass1_variant": os.environ.get("HEXVAL_PASS1", "default"),
                       "coefficients_written": bool(args.coeffs)},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": hv.kernel_launches_per_call() * args.steps,
            "clocks": clk.summary(),
            "subdivision": subdivision,
            **({"secondary": secondary} if secondary else {}),
            **({"graph": graph} if graph else {}),
            "subdivision_rate": st["n_subdivided"] / (world * n),
            "verdicts": {"valid": st["n_valid"], "invalid": st["n_invalid"],
                         "undetermined": st["n_undetermined"], "nonfinite": st["n_nonfinite"],
                         "subdivided": st["n_subdivided"], "exact_sign_hexes": st["n_exact"],
                         "subdivision_nodes": st["n_nodes"], "max_depth": st["max_depth"]},
            "context": "paper: ~6 M hex/s on one core of a 2016 MacBook Pro (PAPER.md:39-40), other machine",
        }
        print(json.dumps(line), flush=True)
    return 0


def run_secondary(args):
    """The FP64-bound kernels of the path against a MEASURED FP64 peak (DFMA probe, same process):
    the subdivision kernel on config 4 (4M adversarial hexes, ~5e9 nodes) and indexed pass 1 on
    config 3 (40M candidates).  Kernel durations from CUPTI activity records; algorithmic FP64
    operations per unit from SURVEY.md 8(d) (294 per subdivision node, 381 per pass-1 hex)."""
    import torch

    import paper_1706_01613_b200 as hv
    out = {}
    try:
        pk = hv.fp64_peak()
        peak, src = pk["dfma_per_s"], ("measured: hexval_diag_fp64_peak, DFMA-only kernel, 8 chains/thread, "
                                        "8x256 threads/SM, best of 5 launches, DFMA lane-instructions/s")
    except Exception as exc:                                          # probe unavailable: datasheet level
        peak, src = FP64_PEAK_GOPS * 1e9, f"fallback 148 SMs x 64 lanes x 1.965 GHz ({str(exc)[:80]})"
    out["fp64_peak"] = {"value": peak, "unit": "FP64 lane-instr/s", "source": src}
    # config 4: subdivision
    layout, n4, host4 = make_inputs(4, 0, args.workers)
    c4 = torch.from_numpy(host4[0]).cuda()
    fl4 = torch.empty(n4, dtype=torch.uint8, device="cuda")
    st = hv.Stats()
    hv.check_soa(c4, flags=fl4, stats=st)
    torch.cuda.synchronize()
    st = st.read()
    ksteps = 3
    kern, _ = cupti_kernel_us(lambda: hv.check_soa(c4, flags=fl4), ksteps)
    k4_s = kern.get("subdiv_kernel", float("nan")) * 1e-6
    out["config4_subdivision"] = {
        "workload": CONFIG_DESC[4], "kernel": "subdiv_kernel (K4)", "kernel_ms": k4_s * 1e3,
        "pass1_ms": kern.get("soa_cp_kernel", float("nan")) * 1e-3,
        "nodes": st["n_nodes"], "subdivided_hexes": st["n_subdivided"], "max_depth": st["max_depth"],
        "nodes_per_s": st["n_nodes"] / k4_s, "lane_use": st["n_nodes"] / max(1, st["n_lane_steps"]),
        "fp64_ops_per_node": FP64_OPS_PER_NODE,
        "fp64_achieved": st["n_nodes"] * FP64_OPS_PER_NODE / k4_s,
        "frac": st["n_nodes"] * FP64_OPS_PER_NODE / k4_s / peak,
        # the kernel's second roofline (K4): a node is written to the warp's stack
        # once and read back once, 2 x 224 B through the L1 data pipe, which moves these 256-bit
        # accesses at 64 B/clk/SM (ncu: l1tex__data_pipe_lsu_wavefronts 50.0% at 2 x 1.16 TB per call,
        # profiles/r02/s4/subdiv_c4_l1_metrics.txt); the peak is derived from that rate at 1965 MHz
        "lsu_roofline": {"bound": "l1 data pipe", "bytes_per_node": K4_L1_BYTES_PER_NODE,
                         "achieved": st["n_nodes"] * K4_L1_BYTES_PER_NODE / k4_s / 1e9,
                         "peak": K4_L1_PEAK_GBS, "unit": "GB/s",
                         "frac": st["n_nodes"] * K4_L1_BYTES_PER_NODE / k4_s / 1e9 / K4_L1_PEAK_GBS,
                         "peak_source": "derived: 148 SMs x 64 B/clk x 1.965 GHz (rate measured with ncu)"},
        "timing": f"mean CUPTI kernel duration over {ksteps} calls"}
    del c4, fl4
    torch.cuda.empty_cache()
    # config 3: indexed pass 1
    layout, n3, host3 = make_inputs(3, 0, args.workers)
    v3, i3 = (torch.from_numpy(a).cuda() for a in host3)
    fl3 = torch.empty(n3, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        hv.check_indexed(v3, i3, flags=fl3)
    ksteps = 10
    kern, _ = cupti_kernel_us(lambda: hv.check_indexed(v3, i3, flags=fl3), ksteps)
    p1_s = next((v for k, v in kern.items() if k in ("idx_cp_kernel", "plain_kernel")), float("nan")) * 1e-6
    out["config3_pass1"] = {
        "workload": CONFIG_DESC[3], "kernel": "idx_cp_kernel (K2)", "kernel_ms": p1_s * 1e3,
        "hexes_per_s": n3 / p1_s, "fp64_ops_per_hex": FP64_OPS_PER_HEX,
        "fp64_achieved": n3 * FP64_OPS_PER_HEX / p1_s, "frac": n3 * FP64_OPS_PER_HEX / p1_s / peak,
        "timing": f"mean CUPTI kernel duration over {ksteps} calls"}
    del v3, i3, fl3
    torch.cuda.empty_cache()
    return out


def run_op(args, world, rank, local):
    """Secondary measurements of the NEXT rows: one kernel per step,
    timed with CUDA events on the launching stream; roofline against HBM."""
    import torch

    import paper_1706_01613_b200 as hv

    torch.cuda.set_device(local)
    cfg = args.config
    if args.op == "quads":
        import hexgen
        from paper_1706_01613_b200 import shard
        start, n = shard.weak_shard(10_000_000, rank)
        layout, host = "quad-soa", (hexgen.quad_soa(n, 0.35, 5, start),)
    else:
        layout, n, host = make_inputs(cfg, rank, args.workers)
    dev = [torch.from_numpy(a).cuda() for a in host]
    stream = torch.cuda.current_stream()
    in_bytes = None
    if args.op == "quads":
        qf = torch.empty(n, dtype=torch.uint8, device="cuda")

        def step():
            hv.check_quad_soa(dev[0], qf)
        out_bytes, in_bytes = 1, 64 * n
        metric = "quadrangles validated/sec (fp64, 1 B200)"
    elif args.op == "select":
        flags = torch.empty(n, dtype=torch.uint8, device="cuda")
        if layout == "soa":
            hv.check_soa(dev[0], flags=flags)
        else:
            hv.check_indexed(dev[0], dev[1], flags=flags)
        groups = 99 ** 3 if cfg == 3 else 1000
        grp = (torch.arange(n, device="cuda", dtype=torch.int64) % groups).to(torch.int32)
        ids = torch.empty(n, dtype=torch.int32, device="cuda")
        gcount = torch.zeros(groups, dtype=torch.int32, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        lib = hv.lib()
        handle = stream.cuda_stream

        def step():                                   # the C ABI directly: no host read-back per step
            lib.hexval_select_valid(flags.data_ptr(), n, grp.data_ptr(), groups, ids.data_ptr(), cnt.data_ptr(),
                                    gcount.data_ptr(), handle)
        step()
        torch.cuda.synchronize()
        n_valid = int(cnt.item())
        in_bytes = 2 * n + 4 * n + 4 * n_valid        # flags read twice, group ids, scattered count updates
        out_bytes = 0
        extra_sel = {"n_valid": n_valid, "groups": groups}
        metric = "candidates filtered/sec (VALID ids + per-cell counts, 1 B200)"
    elif args.op == "screen":
        fl = torch.empty(n, dtype=torch.uint8, device="cuda")
        sj = torch.empty(n, dtype=torch.float64, device="cuda")
        t1 = torch.empty(n, dtype=torch.uint8, device="cuda")

        def step():
            if layout == "soa":
                hv.check_screen_soa(dev[0], fl, sj, t1)
            else:
                hv.check_screen_indexed(dev[0], dev[1], fl, sj, t1)
        out_bytes = 10
        metric = "hexahedra validated + screened/sec (flags, corner scaled Jacobian, Test 1 in one pass, fp64, 1 B200)"
    elif args.op == "quality":
        sj = torch.empty(n, dtype=torch.float64, device="cuda")
        t1 = torch.empty(n, dtype=torch.uint8, device="cuda")

        def step():
            if layout == "soa":
                hv.corner_quality_soa(dev[0], sj, t1)
            else:
                hv.corner_quality_indexed(dev[0], dev[1], sj, t1)
        out_bytes = 9
        metric = "hexahedra screened/sec (corner scaled Jacobian + Test 1, fp64, 1 B200)"
    elif args.op == "bounds":
        lo = torch.empty(n, dtype=torch.float64, device="cuda")
        up = torch.empty(n, dtype=torch.float64, device="cuda")
        stt = torch.empty(n, dtype=torch.uint8, device="cuda")
        nodes = torch.zeros(1, dtype=torch.int64, device="cuda")

        def step(count=None):
            if layout == "soa":
                hv.min_detj_bounds_soa(dev[0], args.rel_tol, lo, up, stt, nodes=count)
            else:
                hv.min_detj_bounds_indexed(dev[0], dev[1], args.rel_tol, lo, up, stt, nodes=count)
        step(nodes)
        torch.cuda.synchronize()
        extra = {"rel_tol": args.rel_tol, "nodes_per_step": int(nodes.item()),
                 "capped": int((stt & 1).sum().item())}
        out_bytes = 17
        metric = f"hexahedra bounded/sec (min det J to rel_tol {args.rel_tol:g}, fp64, 1 B200)"
    if args.op != "bounds":
        extra = extra_sel if args.op == "select" else {}
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local, args.clock_ms * 1e-3) as clk:
        barrier(world)
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    ms = dist_max(ev0.elapsed_time(ev1) / args.steps, world)
    kern_us, launches = {}, None
    if not args.no_cupti:
        try:
            ksteps = min(args.steps, 20)
            kern_us, kcount = cupti_kernel_us(step, ksteps)
            launches = sum(c for k, c in kcount.items() if not k.startswith("Memset")) // ksteps * args.steps
        except Exception as exc:                                      # profiler unavailable
            kern_us = {"error": str(exc)[:200]}
    if in_bytes is None:
        in_bytes = 192 * n if layout == "soa" else 32 * n + 24 * host[0].shape[0]
    algo = in_bytes + out_bytes * n + (4 * extra.get("n_valid", 0) if args.op == "select" else 0)
    peak, peak_src = measured_peaks()
    ach = algo / (ms * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({
            "op": args.op, "metric": metric, "value": world * n / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "ms_per_step": ms, "dtype": "f64", "data": "synthetic",
            "config": {"workload": ("10M linear quadrangles, unit square + U[-0.35,0.35]^2 noise, seed 5"
                                    if args.op == "quads" else CONFIG_DESC[cfg]),
                       "layout": layout, "n_per_rank": n},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "peak_source": peak_src, "algorithmic_bytes_per_launch": algo,
                         "kernel_us_cupti": kern_us},
            "gpu_launches": launches if launches is not None else args.steps,
            "clocks": clk.summary(), **extra}), flush=True)
    return 0


def run_dry(args, world, rank):
    """CPU-only check of the multi-rank plumbing (tests/test_shard.py): every rank reports its shard
    range and runs the oracle on the first hexes of its shard; the verdict counts are summed with the
    same collective the GPU run uses."""
    import numpy as np

    from paper_1706_01613_b200 import shard
    m = 2000
    ref = oracle_sample(args.config, m, 0, nthreads=1, rank=rank)()
    counts = np.bincount(ref["flags"] & 3, minlength=4).tolist()
    summed = shard.sum_over_ranks(counts)
    lo, hi = shard_range(args.config, rank)
    layout, *arrays = shard_inputs(args.config, rank, 0, 4)
    first = float(arrays[0].ravel()[0]) if layout == "soa" else float(arrays[0][arrays[1][0, 0], 2])
    ranges = [None] * world
    if world > 1:
        import torch.distributed as dist
        dist.all_gather_object(ranges, {"rank": rank, "range": [lo, hi], "first_coord": first})
    else:
        ranges = [{"rank": rank, "range": [lo, hi], "first_coord": first}]
    if rank == 0:
        print(json.dumps({"dry_run": True, "world": world, "config": args.config, "shards": ranges,
                          "sample_per_rank": m, "verdicts_summed": dict(zip(["invalid", "valid", "undetermined",
                                                                              "nonfinite"], summed))}), flush=True)
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)                 # one process per GPU, launched for the caller
    world, rank, local = dist_setup(args.gpus, args.dry_run)
    try:
        if args.dry_run:
            return run_dry(args, world, rank)
        if args.impl == "reference":
            return run_reference(args, world, rank)
        if args.op != "check":
            return run_op(args, world, rank, local)
        return run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
