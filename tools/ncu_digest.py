#!/usr/bin/env python
"""Digest of an ncu --set full capture: the details page (section / metric / value) plus the
warp-stall breakdown and the top source lines by stall samples.  Usage:
    python tools/ncu_digest.py REPORT.ncu-rep [--source N]
Writes nothing; print and redirect into profiles/ to keep a text record of a capture."""
import csv
import io
import subprocess
import sys


def ncu(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True, timeout=600).stdout


def main():
    rep = sys.argv[1]
    nsrc = int(sys.argv[sys.argv.index("--source") + 1]) if "--source" in sys.argv else 0
    rows = list(csv.DictReader(io.StringIO(ncu([rep, "--page", "details", "--csv"]))))
    kernel = rows[0]["Kernel Name"] if rows else "?"
    print(f"kernel: {kernel[:160]}")
    for r in rows:
        if r.get("Metric Name"):
            print(f"{r['Section Name'][:30]:30} | {r['Metric Name'][:52]:52} | {r['Metric Value']} {r['Metric Unit']}")
    raw = list(csv.DictReader(io.StringIO(ncu([rep, "--page", "raw", "--csv"]))))
    if raw:
        r = raw[-1] if len(raw) > 1 else raw[0]
        keys = [k for k in r if k.startswith("smsp__average_warp_latency_issue_stalled") or
                k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
        stalls = []
        for k in keys:
            try:
                stalls.append((float(r[k].replace(",", "")), k))
            except ValueError:
                pass
        print("\nwarp stall cycles per issued instruction:")
        for v, k in sorted(stalls, reverse=True)[:14]:
            print(f"  {v:8.3f}  {k}")
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                  "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"):
            if k in r:
                print(f"  {k} = {r[k]}")
    if nsrc:
        # SASS view: row 0 names the kernel, row 1 is the header, then one row per instruction
        src = list(csv.reader(io.StringIO(ncu([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
        if len(src) > 2:
            hdr = src[1]
            ix = {h: i for i, h in enumerate(hdr)}
            stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
            rows, total = [], 0
            for r in src[2:]:
                try:
                    smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
                    ex = int(r[ix["Instructions Executed"]] or 0)
                except (ValueError, IndexError, KeyError):
                    continue
                total += smp
                top = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:2]
                rows.append((smp, ex, r[ix["Address"]][-5:], r[ix["Source"]].strip()[:64], top))
            print(f"\ntop {nsrc} SASS lines by stall samples (share of {total} samples; warp-level executions):")
            for smp, ex, addr, text, top in sorted(rows, reverse=True)[:nsrc]:
                why = " ".join(f"{c}:{v * 100 // max(smp, 1)}%" for v, c in top if v)
                print(f"  {100.0 * smp / max(total, 1):5.2f}%  {ex:>12d}  {addr}  {text:64s}  {why}")


if __name__ == "__main__":
    main()
