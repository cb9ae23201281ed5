"""Like-for-like DRAM traffic of the IC expansion (roofline `traffic`), for bench.py.

Runs the bench's C2 sampling call (theta = 65,536, the bench's first sampling seed, sorted start
vertices, the automatic batch of 4 blocks exactly as bench.py launches it) through the host-driven
level loop, and writes batch 0's level counters to gpurun_out/traffic_levels.json. Run it under
  ncu --set full -k regex:k_expand_bm -c 16 -o gpurun_out/traffic_full python scripts/traffic_capture.py
then `python scripts/traffic_capture.py --summarize` (here, no GPU) pairs launch i with level i and
writes profiles/expand_traffic.json (per launch the DRAM bytes next to the algorithmic bytes of the
SAME launch, DESIGN.md §6 byte model, and their sums) and profiles/expand_ncu_summary.json
(instructions per edge read, issue / warps active, cache hit rates of the same launches)."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "gpurun_out")


def alg_bytes(rows, slots=4):
    """DESIGN.md §6 per-level byte model of the batch-wide frontier (same as
    bpt_samples_info.expand_bytes): 8 B record + 8 B x S of U[u] per reverse-edge read, 8 B per
    atomicOr, (4 + 8 S) B per frontier entry, 8 B per vertex discovered for the next level."""
    out = []
    for i, r in enumerate(rows):
        batch, level, raw, kept, work, vc, coins, atomics = r
        raw_next = rows[i + 1][2] if i + 1 < len(rows) and rows[i + 1][0] == batch else 0
        out.append((8.0 + 8.0 * slots) * work + 8.0 * atomics + (4.0 + 8.0 * slots) * kept + 8.0 * raw_next)
    return out


def capture():
    import torch
    import graphgen
    import paper_2311_10201_b200 as bpt
    cfg = graphgen.CONFIGS["C2"]
    torch.cuda.set_device(0)
    row_ptr, col, thr = graphgen.make_graph(cfg)
    g = bpt.Graph(row_ptr, col, w_q31=thr)
    # the whole bench sampling call (sorted start vertices over all theta samples), host-driven so
    # every expansion launch is a direct launch; ncu captures the first ones = batch 0's levels
    s = g.sample(cfg.theta, colors=64, seed=cfg.seed, profile=True, poll_levels=1)
    rows = [r for r in s.level_stats().tolist() if r[0] == 0]
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "traffic_levels.json"), "w") as f:
        json.dump({"rows": rows, "info": s.info}, f)
    print(json.dumps({"levels": len(rows), "e_phys": s.info["e_phys"]}))


def _ncu_rows(rep):
    import subprocess
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                d[h] = v
                continue
            d[h] = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                        "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(u, 1)
        out.append(d)
    return out


def summarize():
    """Pairs launch i of the ncu --set full report gpurun_out/traffic_full.ncu-rep (every expansion launch
    of the capture run) with level i of the same run."""
    lv = json.load(open(os.path.join(OUT, "traffic_levels.json")))
    rows = lv["rows"]
    alg = alg_bytes(rows)
    seq = _ncu_rows(os.path.join(OUT, "traffic_full.ncu-rep"))[:len(rows)]  # batch 0's levels
    per = []
    for i, d in enumerate(seq):
        a = alg[i] if i < len(alg) else 0.0  # launches after the last level are no-ops (pipelined polling)
        per.append({"level": i, "edges": rows[i][4] if i < len(rows) else 0, "algorithmic_bytes": a,
                    "dram_bytes": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0),
                    "us": d.get("gpu__time_duration.sum", 0) * 1e6, "inst": d.get("smsp__inst_executed.sum", 0),
                    "issue_active_pct": d.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "warps_active_pct": d.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                    "l2_hit_pct": d.get("lts__t_sector_hit_rate.pct"), "l1_hit_pct": d.get("l1tex__t_sector_hit_rate.pct")})
    n = len(per)
    dram = sum(p["dram_bytes"] for p in per)
    algs = sum(p["algorithmic_bytes"] for p in per)
    edges = sum(p["edges"] for p in per)
    us = sum(p["us"] for p in per) or 1.0
    wavg = lambda k: sum((p[k] or 0) * p["us"] for p in per) / us  # time-weighted
    src = ("ncu --set full of every k_expand_bm launch of batch 0 of the bench's sampling call (C2, theta 65,536, "
           "bench seed, sorted start vertices, 4 blocks per batch, host-driven level loop; scripts/traffic_capture.py)")
    res = {"source": src, "kernel": seq[0].get("Kernel Name") if seq else None, "launches": n,
           "dram_bytes_per_launch": dram / n if n else None, "algorithmic_bytes_per_launch": algs / n if n else None,
           "dram_over_algorithmic": dram / algs if algs else None, "per_launch": per}
    summ = {"source": src, "inst_per_edge_read": sum(p["inst"] for p in per) / edges if edges else None,
            "issue_active_pct": wavg("issue_active_pct"), "warps_active_pct": wavg("warps_active_pct"),
            "l2_hit_pct": wavg("l2_hit_pct"), "l1_hit_pct": wavg("l1_hit_pct"),
            "edges_per_s": edges / (us * 1e-6), "launches": n}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "expand_traffic.json"), "w") as f:
        json.dump(res, f, indent=1)
    with open(os.path.join(ROOT, "profiles", "expand_ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "per_launch"}, indent=1))
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    summarize() if "--summarize" in sys.argv else capture()
