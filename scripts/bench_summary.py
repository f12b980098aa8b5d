"""Markdown table of a directory of bench.py JSON lines (one file per config).

    python scripts/bench_summary.py gpurun_out/final > profiles/r02_bench_summary.md
"""
import glob
import json
import os
import sys


def fmt(x, f="{:.3g}"):
    return "—" if x is None else f.format(x)


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/final"
    rows = ["| file | workload | SEPS | ms / step | e2e SEPS | hot kernel | frac (model) | f_dram | clocks (MHz, reasons) | "
            "cpu baseline (cores) | notes |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for path in sorted(glob.glob(os.path.join(src, "bench_*.json"))):
        lines = [l for l in open(path) if l.startswith("{")]
        if not lines:
            rows.append(f"| {os.path.basename(path)} | (no JSON line) | | | | | | | | | |")
            continue
        d = json.loads(lines[-1])
        r = d.get("roofline") or {}
        det = d.get("detail") or {}
        cache = det.get("cache") or {}
        notes = []
        if cache.get("build_ms"):
            notes.append(f"build {cache['build_ms']:.0f} ms, one-call {cache.get('one_call_seps', 0):.3g} SEPS")
        sp = det.get("scan_path")
        if sp and "ms_per_step" in sp:
            notes.append(f"scan path {sp['kernel']} {sp['ms_per_step']:.1f} ms (frac {fmt(sp.get('frac'))})")
        if r.get("frac_of_random_gather_peak") is not None:
            notes.append(f"{r['frac_of_random_gather_peak']:.2f} of the random-gather peak")
        if r.get("bound") not in (None, "hbm"):
            notes.append(f"{r['bound']}: {fmt(r.get('achieved'))} of {fmt(r.get('peak'))} GB/s")
        if d.get("impl") == "reference":
            notes.append("oracle on the host cores (reference arm)")
        clk = d.get("clocks") or {}
        cpu = d.get("cpu_baseline") or {}
        e2e = d.get("e2e") or {}
        rows.append(f"| {os.path.basename(path)} | {(d.get('config') or {}).get('workload', '')[:60]} | {fmt(d.get('value'))} | "
                    f"{fmt(d.get('ms_per_step'), '{:.3f}')} | {fmt(e2e.get('value'))} | `{r.get('kernel', '')}` | "
                    f"{fmt(r.get('frac'))} | {fmt(r.get('f_dram'))} | {clk.get('sm_mhz')} {clk.get('reasons')} | "
                    f"{fmt(cpu.get('value'))} ({cpu.get('cores')}) | {'; '.join(notes)} |")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
