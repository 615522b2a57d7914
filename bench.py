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

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "hexahedra validated/sec (fp64, 1 B200); % of HBM roofline; subdivision rate"
UNIT = "hex/s"
FALLBACK_HBM_GBS = 6650.0
# fp64 operations per subdivision node: 147 new de Casteljau values, one add and one
# multiply each; peak = 148 SMs x 64 FP64 lanes x 1.965 GHz
FP64_OPS_PER_NODE = 294
FP64_PEAK_GOPS = 148 * 64 * 1.965
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
    p.add_argument("--clock-ms", type=float, default=10.0,
                   help="NVML clock sampling period during the timed region (ms)")
    p.add_argument("--no-cupti", action="store_true",
                   help="skip the torch.profiler (CUPTI) kernel-duration pass (e.g. under ncu)")
    p.add_argument("--graph", action="store_true",
                   help="also time the call captured in a CUDA graph (launch-bound small batches)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=8.0, help="target wall time of the CPU baseline sample")
    p.add_argument("--coeffs", action="store_true",
                   help="also write the 27 Bezier coefficients per hex (409 B/hex, SURVEY.md 8(d))")
    p.add_argument("--op", choices=["check", "quality", "screen", "bounds", "select", "quads"], default="check",
                   help="check: the hot path (headline); quality: NEXT-2 corner screening kernel; "
                        "bounds: NEXT-1 certified min det J bounds; select: NEXT-3 candidate filtering "
                        "(on the config's flags); quads: NEXT-4 linear quadrangles (10M, noise 0.35)")
    p.add_argument("--rel-tol", type=float, default=1e-3, help="NEXT-1 tolerance (relative to max|b|)")
    p.add_argument("--variant", choices=["ldg", "wtma", "cp"], default=None,
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


def dist_setup(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
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
def oracle_sample(cfg: int, m: int, start: int = 0, nthreads: int = 0):
    import hexgen
    import oracle
    if cfg in (0, 1):
        coords = hexgen.soa_config(m, 0.25 if cfg == 0 else 0.35, cfg, start)
        return lambda: oracle.check_soa(coords, nthreads=nthreads)
    if cfg == 4:
        coords, _ = hexgen.adversarial_config(m, 4, start)
        return lambda: oracle.check_soa(coords, nthreads=nthreads)
    _, verts, idx = hexgen.make(cfg, start, m)
    return lambda: oracle.check_indexed(verts, idx, nthreads=nthreads)


def oracle_rate(cfg: int, seconds: float, start: int = 0):
    """Time the oracle, as it stands, on a bounded prefix sample of the workload (all host threads)."""
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
    run = oracle_sample(cfg, m, start)
    t0 = time.perf_counter()
    run()
    dt = time.perf_counter() - t0
    # one thread on a smaller slice of the same stream (per-core rate, the unit of the
    # paper's ~6 M hex/s on one core)
    m1 = max(1000, min(m, int(m / max(1, cores) / 4)))
    run1 = oracle_sample(cfg, m1, start, nthreads=1)
    t1 = time.perf_counter()
    run1()
    dt1 = time.perf_counter() - t1
    return {"value": m / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"hexes {start}..{start + m - 1} of {CONFIG_DESC[cfg]} ({m} hexes, {dt:.2f} s wall on {cores} threads)",
            "single_thread": {"value": m1 / dt1, "unit": UNIT, "sample": f"hexes {start}..{start + m1 - 1}, 1 thread"}}


def run_reference(args, world, rank):
    import hexgen
    if rank != 0:
        return 0
    n = hexgen.config_size(args.config)
    per_step = []
    for _ in range(args.warmup):
        oracle_rate(args.config, min(args.cpu_seconds, 2.0))
    last = None
    for _ in range(args.steps):
        last = oracle_rate(args.config, args.cpu_seconds / max(1, args.steps) + 0.5)
        per_step.append(last["value"])
    value = statistics.median(per_step)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * n / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": CONFIG_DESC[args.config], "n_hexes": n,
                   "layout": "indexed" if args.config in (2, 3) else "soa",
                   "note": "each step times the CPU oracle (oracle/, as it stands) on a bounded prefix sample; ms_per_step is extrapolated to the full batch"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "oracle",
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def make_inputs(cfg: int, rank: int):
    """Host arrays of this rank's shard (weak scaling: every rank its own n hexes)."""
    import hexgen
    from paper_1706_01613_b200 import shard
    start, n = shard.weak_shard(hexgen.config_size(cfg), rank)
    if cfg in (0, 1):
        return "soa", n, (hexgen.soa_config(n, 0.25 if cfg == 0 else 0.35, cfg, start=start),)
    if cfg == 4:
        coords, _ = hexgen.adversarial_config(n, 4, start=start)
        return "soa", n, (coords,)
    _, verts, idx = hexgen.make(cfg)
    return "indexed", n, (verts, idx)


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
    layout, n, host = make_inputs(cfg, rank)
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

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_rate(cfg, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "n_hexes_per_rank": n, "global_hexes": world * n, "layout": layout,
                       "parallelism": f"independent shards x{world}" if world > 1 else "single GPU",
                       "l2": L2_NOTE[cfg],
                       "pass1_variant": os.environ.get("HEXVAL_PASS1", "default"),
                       "coefficients_written": bool(args.coeffs)},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": hv.kernel_launches_per_call() * args.steps,
            "clocks": clk.summary(),
            "subdivision": subdivision,
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
        layout, n, host = make_inputs(cfg, rank)
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


def main():
    args = parse()
    world, rank, local = dist_setup(args.gpus)
    try:
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
