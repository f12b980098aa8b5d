"""Summarise ncu `--page raw --csv` exports (one full capture per config) into a
markdown table and refresh profiles/ncu_traffic.json (DRAM bytes per launch of
each config's hot kernel, which bench.py reports as roofline.traffic).

    python scripts/ncu_summary.py gpurun_out/prof r01 > profiles/r01_ncu_summary.md
"""
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}

METRICS = [
    ("time", "gpu__time_duration.sum"),
    ("dram_rd", "dram__bytes_read.sum"),
    ("dram_wr", "dram__bytes_write.sum"),
    ("dram_pct", "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_hit", "lts__t_sector_hit_rate.pct"),
    ("l1_hit", "l1tex__t_sector_hit_rate.pct"),
    ("l2_rd_sectors", "lts__t_sectors_srcunit_tex_op_read.sum"),
    ("bytes_per_sector", "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio"),
    ("warps_active", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue_active", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("sm_thr", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("mem_thr", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
]


def load(path):
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        return None
    h, u, v = rows[0], rows[1], rows[2]
    d = {"kernel": v[h.index("Kernel Name")].split("(")[0]}
    for key, m in METRICS:
        if m in h:
            i = h.index(m)
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                continue
            d[key] = x * UNIT.get(u[i], 1.0) if u[i] in UNIT else x
    stalls = []
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v[i]), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    d["stalls"] = stalls[:3]
    return d


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof"
    rnd = sys.argv[2] if len(sys.argv) > 2 else "r02"
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)
    out = [f"# {rnd} — ncu `--set full` summary, one hot-kernel launch per config", "",
           "Each row: `ncu --set full --clock-control none --import-source on --nvtx --nvtx-include csaw_step/ "
           "-k regex:<kernel> -c 1` around `bench.py --config <cfg> --steps 1 --warmup 1` "
           "(`scripts/gpu_bench_all_r02.sh`; a @variant name adds the flags it names: cfg2@stream = --no-cache, "
           "cfg5@inmem = --in-memory), exported with `ncu -i --page raw --csv` (`scripts/ncu_summary.py`); a "
           "metrics-only pass (DRAM bytes + time) covers every launch of the timed step.  ncu times are cold-cache and serialised: "
           "the bench line's CUDA-event numbers are the measurement; these explain them.", "",
           f"DRAM GB/s is ncu DRAM bytes / ncu duration; fraction of the measured {peak:.1f} GB/s copy peak.", "",
           "| config | kernel | ncu ms | DRAM rd+wr | DRAM GB/s (frac) | L2 hit | L1 hit | B used/sector (ld) | warps active | issue active | regs | grid x block | top stalls (per issue) |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        traffic = json.load(open(traffic_path))
    except Exception:
        traffic = {}
    for path in sorted(glob.glob(os.path.join(src, "*_raw.csv"))):
        cfg = os.path.basename(path)[:-len("_raw.csv")]
        d = load(path)
        if not d or "time" not in d:
            continue
        dram = d.get("dram_rd", 0) + d.get("dram_wr", 0)
        gbs = dram / d["time"] / 1e9
        st = ", ".join(f"{n} {x:.1f}" for x, n in d["stalls"])
        out.append(f"| {cfg} | `{d['kernel']}` | {d['time'] * 1e3:.3f} | {dram / 1e9:.3f} GB | {gbs:.0f} ({gbs / peak:.3f}) | "
                   f"{d.get('l2_hit', 0):.1f} % | {d.get('l1_hit', 0):.1f} % | {d.get('bytes_per_sector', 0):.1f} | "
                   f"{d.get('warps_active', 0):.1f} % | {d.get('issue_active', 0):.1f} % | {d.get('regs', 0):.0f} | "
                   f"{d.get('grid', 0):.0f} x {d.get('block', 0):.0f} | {st} |")
        key = cfg.replace("@", "_")   # e.g. cfg5_inmem, cfg2_scan (bench.py picks the key of its variant)
        note = "per launch of the bench's hot kernel (1 bench step)"
        traffic[key] = {"kernel": d["kernel"], "dram_bytes_per_launch": int(dram), "ncu_ms": d["time"] * 1e3,
                        "f_dram": gbs / peak,
                        "l2_sector_eff": (d["bytes_per_sector"] / 32.0) if "bytes_per_sector" in d else None,
                        "l2_hit_pct": d.get("l2_hit"), "round": rnd, "note": note}
    # metrics-only launch lists with DRAM counters (cfg3: the full bench launch, too long for --set full)
    for path in sorted(glob.glob(os.path.join(src, "*_launches.csv"))):
        cfg = os.path.basename(path)[:-len("_launches.csv")]
        rows = [r for r in csv.reader(open(path)) if r]
        hi = [j for j, r in enumerate(rows) if r[0] == "ID"]
        if not hi:
            continue
        h = rows[hi[0]]
        per = {}
        for r in rows[hi[0] + 1:]:
            d = dict(zip(h, r))
            if d.get("Metric Name") in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
                k = (d.get("ID"), d.get("Kernel Name", "").split("(")[0])
                per.setdefault(k, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        # the hot kernel of the launch list = the longest launch (a list also holds the seed
        # check, the fused copy, ...): only it updates the traffic record
        hot = max(per.items(), key=lambda kv: kv[1].get("gpu__time_duration.sum", 0.0))[0] if per else None
        for (lid, kname), m in per.items():
            if "dram__bytes_read.sum" not in m:
                continue
            if (lid, kname) != hot:
                t = m.get("gpu__time_duration.sum", 0.0) * 1e-9
                dram = m["dram__bytes_read.sum"] + m.get("dram__bytes_write.sum", 0.0)
                if t > 0:
                    out.append(f"| {cfg} (metrics-only, full launch) | `{kname}` | {t * 1e3:.3f} | {dram / 1e9:.3f} GB | "
                               f"{dram / t / 1e9:.0f} ({dram / t / 1e9 / peak:.3f}) | | | | | | | | |")
                continue
            dram = m["dram__bytes_read.sum"] + m.get("dram__bytes_write.sum", 0.0)
            t = m.get("gpu__time_duration.sum", 0.0) * 1e-9
            key = cfg.replace("@", "_")
            prev = traffic.get(key, {}) if traffic.get(key, {}).get("round") == rnd else {}
            traffic[key] = {"kernel": kname, "dram_bytes_per_launch": int(dram), "ncu_ms": t * 1e3, "round": rnd,
                            "f_dram": (dram / t / 1e9 / peak) if t > 0 else None,
                            "l2_sector_eff": prev.get("l2_sector_eff"), "l2_hit_pct": prev.get("l2_hit_pct"),
                            "note": "metrics-only pass (dram__bytes_read/write.sum) over the bench's timed launch; "
                                    "sector efficiency from the --set full capture of the same round"}
            if t > 0:
                out.append(f"| {cfg} (metrics-only, full launch) | `{kname}` | {t * 1e3:.3f} | {dram / 1e9:.3f} GB | "
                           f"{dram / t / 1e9:.0f} ({dram / t / 1e9 / peak:.3f}) | | | | | | | | |")
    traffic["_source"] = ("ncu --set full --clock-control none (profiles/%s_ncu_summary.md); "
                          "dram__bytes_read.sum + dram__bytes_write.sum per launch of the hot kernel" % rnd)
    json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main()
