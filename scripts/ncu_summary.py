"""Summarise ncu outputs into profiles/ (committed evidence).

  python scripts/ncu_summary.py rep   <file.ncu-rep> <out.md> [--levels <json log with level rows>]
  python scripts/ncu_summary.py list  <launches.csv> <out.md>

`rep`: per profiled launch -- duration, DRAM read/write bytes, DRAM and L2 throughput, L2 hit
rate, issue activity, occupancy and the top stall reasons. With --levels (a sample_sweep.py
JSON line printed with --levels), the algorithmic bytes of the profiled expansion launches
are computed from the exact level counters and profiles/expand_traffic.json
is written for bench.py's roofline.traffic.
`list`: per kernel name -- launches, total and mean device time, share of the run.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "ncu"

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
         "msecond": 1e3, "s": 1e6}


def raw_rows(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, data = r[0], r[1], r[2:]
    return hdr, units, data


def summarise_rep(rep, out_md, levels_log=None):
    hdr, units, data = raw_rows(rep)
    ix = {h: i for i, h in enumerate(hdr)}
    launches = []
    for row in data:
        d = {"kernel": row[ix["Kernel Name"]].split("(")[0], "id": row[ix["ID"]]}
        for k in KEYS:
            if k in ix:
                v = row[ix[k]].replace(",", "")
                try:
                    d[k] = float(v) * SCALE.get(units[ix[k]], 1)
                except ValueError:
                    d[k] = v
        stalls = {}
        for h, i in ix.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(row[i])
                except ValueError:
                    pass
        d["stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        launches.append(d)
    lines = [f"# ncu --set full summary: `{os.path.basename(rep)}`", "",
             "| id | kernel | time (us) | DRAM read (MB) | DRAM write (MB) | DRAM GB/s | L2 hit % | issue active % | warps active % | inst (M) | top stalls (cycles/issue) |",
             "|---|---|---|---|---|---|---|---|---|---|---|"]
    for d in launches:
        st = ", ".join(f"{k} {v:.2f}" for k, v in d["stalls"].items())
        lines.append(f"| {d['id']} | {d['kernel']} | {d.get('gpu__time_duration.sum', 0):.1f} | "
                     f"{d.get('dram__bytes_read.sum', 0) / 1e6:.1f} | {d.get('dram__bytes_write.sum', 0) / 1e6:.1f} | "
                     f"{(d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)) / max(d.get('gpu__time_duration.sum', 1), 1e-9) / 1e3:.0f} | "
                     f"{d.get('lts__t_sector_hit_rate.pct', 0):.1f} | "
                     f"{d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                     f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                     f"{d.get('smsp__inst_executed.sum', 0) / 1e6:.1f} | {st} |")
    traffic = None
    if levels_log:
        rows = None
        for line in open(levels_log):
            line = line.strip()
            if line.startswith("{") and '"levels"' in line:
                rows = json.loads(line)["levels"]
                break
        if rows:
            # profiled launches: ncu -s S -c C over k_expand_ic launches; expansion launch i of
            # batch 0 expands level i. Algorithmic bytes per level.
            lines += ["", "Algorithmic bytes of the profiled expansion launches (level rows: batch, level, raw, kept, "
                      "edges, vc):", ""]
            b0 = [r for r in rows if r[0] == 0]
            skip = int(os.environ.get("NCU_SKIP", "4"))
            per = []
            for j, d in enumerate(launches):
                lvl = skip + j
                if lvl >= len(b0):
                    break
                r = b0[lvl]
                nxt_raw = b0[lvl + 1][2] if lvl + 1 < len(b0) else 0
                alg = 16.0 * r[4] + 24.0 * r[3] + 8.0 * nxt_raw  # + 8 B per atomicOr (not in level rows)
                dram = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
                per.append((alg, dram, r[4], d.get("gpu__time_duration.sum", 0)))
                lines.append(f"- level {lvl}: edges {r[4]:,}, entries {r[3]:,}; algorithmic >= {alg / 1e6:.1f} MB; "
                             f"DRAM {dram / 1e6:.1f} MB ({dram / alg:.2f}x); "
                             f"{r[4] / (d.get('gpu__time_duration.sum', 1) * 1e-6) / 1e9:.1f} G edges/s")
            if per:
                alg = sum(p[0] for p in per) / len(per)
                dram = sum(p[1] for p in per) / len(per)
                traffic = {"dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": alg,
                           "source": os.path.relpath(out_md, ROOT), "launches": len(per)}
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic:
        with open(os.path.join(ROOT, "profiles", "expand_traffic.json"), "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines))


def summarise_list(csv_path, out_md):
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 5]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].split("::")[-1]
        v = float(r[ix["Metric Value"]].replace(",", "")) * SCALE.get(r[ix["Metric Unit"]], 1)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`): `{os.path.basename(csv_path)}`",
             "", "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
             "| kernel | launches | total (us) | share | mean (us) |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {v[0]} | {v[1]:.1f} | {100 * v[1] / tot:.1f}% | {v[1] / v[0]:.2f} |")
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "rep":
        lv = sys.argv[sys.argv.index("--levels") + 1] if "--levels" in sys.argv else None
        summarise_rep(sys.argv[2], sys.argv[3], lv)
    else:
        summarise_list(sys.argv[2], sys.argv[3])
