#!/usr/bin/env python
"""bench.py -- RRR sets/s and edges visited/s of the 64-colour fused BPT hot path on B200.

One step = the whole hot path over one batch of synthetic input:
  bpt_graph_load (validate + reverse-CSR build from the device-resident forward CSR)
  -> bpt_sample (theta RRR sets, 64 fused colours, sizes + digests)
  -> bpt_rrr_extract (the first 64-sample block of this rank, mask -> lists)
  -> bpt_select_seeds (k rounds of greedy max-cover, NCCL collectives when N > 1)
Workload: BASELINE.json configs[1] (C2, soc-LiveJournal1-shaped R-MAT). theta is fixed
(strong scaling): each of N ranks samples theta/N. Inputs (0.59 GB forward CSR) and the
39.7 GB RRR store exceed the 126 MB L2, so no L2 flush is needed between steps.

`--impl reference` times the CPU oracle (oracle/, unfused one-BPT-at-a-time) on the host
cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import graphgen  # noqa: E402

METRIC = "RRR sets/sec (64-color fused BPT, IC, LiveJournal-shaped R-MAT)"
METRICS = {  # per config (the default C2 line keeps the name above)
    "C1": "RRR sets/sec (64-color fused BPT, IC, R-MAT scale 10)",
    "C2": METRIC,
    "C3": "RRR sets/sec (64-color fused BPT, LT, Orkut-shaped R-MAT)",
    "C4": "RRR sets/sec (64-color fused BPT, IC, Friendster-shaped R-MAT)",
    "C5": METRIC,
}
UNIT = "RRR sets/s"
CFG = graphgen.CONFIGS["C2"]
EXTRACT_SAMPLES = 64
PER_MEMBER_BYTES_LT = "24 B per RRR member (8 B row bounds + 8 B chosen in-edge record + 8 B visited-set insertion)"
PER_EDGE_BYTES = ("per reverse-edge read of a frontier vertex: 8 B {src,thr} record + 8 B x S of U[u] (= V|N of the "
                  "S = 4 slots of the batch-wide frontier, one 32-B sector); + 8 B per atomicOr + (4 + 8 S) B per "
                  "frontier entry + 8 B per vertex discovered for the next level")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--batch-groups", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-wide", action="store_true", help="skip the wide-fusion (128-colour) side measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-samples", type=int, default=0, help="oracle sample size (0 = auto)")
    return ap.parse_args()


def workload_desc(cfg) -> str:
    return (f"{cfg.name}: R-MAT n={cfg.n} m={cfg.m} {cfg.model} weights={cfg.weights}, "
            f"C={cfg.colors}, theta={cfg.theta}, k={cfg.k}")


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first(self, timeout: float = 5.0):
        """Block until nvidia-smi has produced its first sample (so short timed regions are covered)."""
        t_end = time.time() + timeout
        while self.proc and not self.lines and time.time() < t_end:
            time.sleep(0.01)

    def mark(self):
        """Start of the timed region: samples before it are dropped."""
        self.first = len(self.lines)

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        first = getattr(self, "first", 0)
        if len(self.lines) <= first:  # region shorter than one sampling period: keep the sample after it
            first = max(0, first - 1)
        for line in self.lines[first:]:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic(name: str) -> dict:
    """DRAM read+write bytes per launch of the dominant kernel from a committed ncu capture, with the
    algorithmic bytes of the SAME launches (scripts/traffic_capture.py)."""
    p = os.path.join(ROOT, "profiles", name)
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------ CPU oracle baseline
def cpu_baseline(cfg, row_ptr, col, thr, nsamples: int | None = None, budget_s: float = 15.0) -> dict:
    import oracle
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.IC if cfg.model == "IC" else oracle.LT)
    threads = oracle.default_threads()
    # calibrate: a small probe, then size the sample for ~budget_s of wall time
    probe = max(threads, 8)
    t0 = time.perf_counter()
    g.sample_many(cfg.seed, np.arange(probe, dtype=np.uint64), threads)
    dt = max(time.perf_counter() - t0, 1e-3)
    if not nsamples:
        nsamples = int(min(cfg.theta, max(probe, probe * budget_s / dt)))
    ids = np.arange(nsamples, dtype=np.uint64)
    t0 = time.perf_counter()
    sizes, _, elog = g.sample_many(cfg.seed, ids, threads)
    dt = time.perf_counter() - t0
    # single-thread rate on a small slice of the same ids (SURVEY §8(d) oracle timing)
    n1 = max(1, min(nsamples, int(nsamples / max(threads, 1) / 2)))
    t1 = time.perf_counter()
    g.sample_many(cfg.seed, ids[:n1], 1)
    dt1 = max(time.perf_counter() - t1, 1e-6)
    return {"value": nsamples / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{nsamples} of {cfg.theta} samples (ids 0..{nsamples - 1}) of {cfg.name}, unfused "
                      f"one-BPT-at-a-time oracle, {threads} threads, {dt:.1f} s",
            "e_logical_per_s": float(elog.sum()) / dt, "seconds": dt,
            "single_thread_value": n1 / dt1, "single_thread_sample": f"ids 0..{n1 - 1}, 1 thread, {dt1:.1f} s"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    cfg = graphgen.CONFIGS[args.config]
    row_ptr, col, thr = graphgen.make_graph(cfg)
    import oracle
    g = oracle.Graph(row_ptr, col, w_q31=thr, model=oracle.IC if cfg.model == "IC" else oracle.LT)
    threads = oracle.default_threads()
    # per step: a bounded sample sized so that warmup + steps finish within ~3 minutes
    t0 = time.perf_counter()
    g.sample_many(cfg.seed, np.arange(threads, dtype=np.uint64), threads)
    per = max(time.perf_counter() - t0, 1e-3) / threads  # wall seconds per sample with all threads busy
    nsteps = args.steps + args.warmup
    per_step = int(max(threads, min(cfg.theta, 150.0 / nsteps / per)))
    times = []
    for i in range(nsteps):
        ids = np.arange(i * per_step, (i + 1) * per_step, dtype=np.uint64) % cfg.theta
        t0 = time.perf_counter()
        g.sample_many(cfg.seed, ids, threads)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    ms = 1000.0 * sum(times) / len(times)
    value = per_step / (ms / 1000.0)
    line = {"impl": "reference", "metric": METRICS.get(cfg.name, METRIC), "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg), "step": f"{per_step} samples of the workload (bounded)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{per_step} samples per step of {cfg.name}, unfused oracle, {threads} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist
    import paper_2311_10201_b200 as bpt

    cfg = graphgen.CONFIGS[args.config]
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    comm = None
    if world > 1:
        uid = [bpt.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = bpt.Comm(world, rank, local_rank, uid[0])
    else:
        comm = bpt.Comm(1, 0, local_rank)

    row_ptr, col, thr = graphgen.make_graph(cfg)
    model = bpt.IC if cfg.model == "IC" else bpt.LT
    # (the generator's arrays are cached read-only; torch wants writable host arrays)
    d_row = torch.from_numpy(row_ptr.view(np.int64).copy()).to(dev)
    d_col = torch.from_numpy(col.view(np.int32).copy()).to(dev)
    d_thr = torch.from_numpy(thr.view(np.int32).copy()).to(dev)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            dist.barrier()

    step_no = [0]  # sampling seeds rotate over cfg.seed + {0, 1, 2} (SURVEY §8(d) throughput protocol)

    def step(profile: bool, host: dict | None = None, wide: bool = False):
        seed = cfg.seed + step_no[0] % 3
        step_no[0] += 1
        if host is None:
            g = bpt.Graph(d_row, d_col, w_q31=d_thr, model=model, comm=comm, n=cfg.n, m=cfg.m, stream=stream)
        elif world > 1:  # end to end: rank 0 copies the input once, the reverse CSR goes over NVLink
            g = bpt.Graph(host["row"] if rank == 0 else None, host["col"] if rank == 0 else None,
                          w_q31=host["thr"] if rank == 0 else None, model=model, comm=comm, n=cfg.n, m=cfg.m,
                          stream=stream, bcast_root=0)
        else:
            g = bpt.Graph(host["row"], host["col"], w_q31=host["thr"], model=model, comm=comm, n=cfg.n, m=cfg.m,
                          stream=stream)
        s = g.sample(cfg.theta, colors=cfg.colors, seed=seed, stream=stream, batch_groups=args.batch_groups,
                     profile=profile, wide=wide)
        first = s.s0
        cnt = min(EXTRACT_SAMPLES, s.s1 - s.s0)
        d2h = 0
        if cnt > 0:
            if host is None:
                sz = int(s.sizes(first, cnt).astype(np.uint64).sum())
                off = torch.empty(cnt + 1, dtype=torch.int64, device=dev)
                mem = torch.empty(max(sz, 1), dtype=torch.int32, device=dev)
                s.extract(first, cnt, offsets=off, members=mem, capacity=sz)
            else:  # into reused pinned host buffers (grown with headroom in the untimed warm-up step)
                sz = int(s.sizes(first, cnt).astype(np.uint64).sum())
                if host.get("mem") is None or host["mem"].numel() < sz:
                    host["mem"] = torch.empty(max(sz + sz // 2, 1), dtype=torch.int32).pin_memory()
                if host.get("off") is None or host["off"].numel() < cnt + 1:
                    host["off"] = torch.empty(cnt + 1, dtype=torch.int64).pin_memory()
                s.extract(first, cnt, offsets=host["off"], members=host["mem"], capacity=host["mem"].numel())
                d2h += (cnt + 1) * 8 + sz * 4
        seeds, gains, sigma = s.select_seeds(cfg.k)
        d2h += seeds.nbytes + gains.nbytes + 8
        info = s.info
        s.close()
        g.close()
        return info, sigma, d2h

    # warmup
    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    clocks.wait_first()
    launches0 = bpt.kernel_launch_count()
    graph0 = bpt.graph_kernel_count()
    barrier()
    torch.cuda.synchronize()
    clocks.mark()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    infos = []
    for _ in range(args.steps):
        info, sigma, _ = step(False)  # production path: device-resident graph loop
        infos.append(info)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    host_launches = bpt.kernel_launch_count() - launches0
    graph_kernels = bpt.graph_kernel_count() - graph0
    launches = host_launches + graph_kernels
    ms = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    # aggregate work counters over ranks (per step)
    e_phys = float(np.mean([i["e_phys"] for i in infos]))
    e_log = float(np.mean([i["e_logical"] for i in infos]))
    ms_expand_timed = float(np.mean([i["ms_expand"] for i in infos]))  # device %globaltimer spans
    ms_sample = float(np.mean([i["ms_total"] for i in infos]))
    # one more step with a CUDA event pair around every expansion launch on the launching
    # stream (host-driven loop, same kernels): the roofline's per-launch durations
    pinfo, _, _ = step(True)
    torch.cuda.synchronize()
    ms_expand = float(pinfo["ms_expand"])
    expand_bytes = float(pinfo["expand_bytes"])
    expand_launches = float(pinfo["expand_launches"])
    agg = torch.tensor([e_phys, e_log], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(agg, op=dist.ReduceOp.SUM)
    e_phys_all, e_log_all = agg.tolist()

    # end-to-end through the C-ABI with pinned HOST buffers (H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        host = {"row": torch.from_numpy(row_ptr.view(np.int64).copy()).pin_memory(),
                "col": torch.from_numpy(col.view(np.int32).copy()).pin_memory(),
                "thr": torch.from_numpy(thr.view(np.int32).copy()).pin_memory()}
        h2d = row_ptr.nbytes + col.nbytes + thr.nbytes  # copied once per step (rank 0 when world > 1)
        step(False, host)
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        d2h = 0
        n_e2e = max(1, min(args.steps, 3))
        for _ in range(n_e2e):
            _, _, d2h = step(False, host)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1) / n_e2e
        et = torch.tensor([ems], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": cfg.theta / (float(et.item()) / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": float(et.item())}

    # wide fusion (BPT_FLAG_WIDE: 128 colours per frontier entry), the same
    # step with two 64-sample blocks sharing one frontier; reported beside the 64-colour headline
    wide = None
    if cfg.model == "IC" and cfg.colors == 64 and not args.batch_groups and not args.no_wide:
        step(False, wide=True)
        barrier()
        torch.cuda.synchronize()
        w0 = torch.cuda.Event(enable_timing=True)
        w1 = torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        n_w = max(1, min(args.steps, 3))
        winfos = []
        for _ in range(n_w):
            wi, _, _ = step(False, wide=True)
            winfos.append(wi)
        w1.record(stream)
        torch.cuda.synchronize()
        barrier()
        wt = torch.tensor([w0.elapsed_time(w1) / n_w], dtype=torch.float64)
        wa = torch.tensor([float(np.mean([i["e_phys"] for i in winfos]))], dtype=torch.float64)
        if world > 1:
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
            dist.all_reduce(wa, op=dist.ReduceOp.SUM)
        wms = float(wt.item())
        wide = {"value": cfg.theta / (wms / 1000.0), "unit": UNIT, "ms_per_step": wms, "steps": n_w,
                "colors_per_frontier_entry": 128, "edges_visited_per_step": float(wa.item()),
                "fusion_factor": e_log_all / float(wa.item()) if wa.item() else None,
                "note": "same step and RRR sets; two 64-sample blocks share one frontier (vertex-major masks)"}

    if rank != 0:
        return
    peak, peak_src = measured_peak_hbm()
    # the co-binding integer-ALU roof of the coins: Philox2x32-10 evaluations per second
    # measured on this device, against the coins the expansion evaluated per step
    pc, pms = bpt.bench_philox(256)
    coins = float(pinfo["coins"])
    alu = {"philox_calls_per_s": pc / (pms / 1000.0), "coins_per_step": coins,
           "coins_per_edge_read": coins / float(pinfo["e_phys"]) if pinfo["e_phys"] else None,
           "coin_roof_ms_per_step": 1000.0 * coins / (pc / (pms / 1000.0)),
           "coin_roof_share_of_expansion": (1000.0 * coins / (pc / (pms / 1000.0))) / ms_expand if ms_expand else None}
    prof = ncu_traffic("expand_ncu_summary.json") if cfg.model == "IC" else {}
    for key in ("inst_per_edge_read", "issue_active_pct", "warps_active_pct", "l2_hit_pct", "source"):
        if key in prof:
            alu["ncu_" + key] = prof[key]
    achieved = expand_bytes / (ms_expand / 1000.0) / 1e9 if ms_expand > 0 else None
    if cfg.model == "IC":
        tr = ncu_traffic("expand_traffic.json")
        kernel, per_unit = "k_expand_bm (A3 fused frontier expansion)", PER_EDGE_BYTES
    else:  # LT: one reverse walk per sample into the sparse member-list store
        tr = ncu_traffic("walk_lt_traffic.json")
        kernel, per_unit = "k_walk_lt_sparse (A3' LT reverse walks, sparse store)", PER_MEMBER_BYTES_LT
    traffic = tr.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "kernel": kernel,
                "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "traffic_algorithmic_per_launch": tr.get("algorithmic_bytes_per_launch"),
                "traffic_over_algorithmic": tr.get("dram_over_algorithmic"),
                "traffic_launches": tr.get("launches"),
                "algorithmic_bytes_per_launch": expand_bytes / expand_launches if expand_launches else None,
                "launches_per_step": expand_launches, "ms_expand_per_step": ms_expand,
                "ms_expand_per_step_timed_region": ms_expand_timed,
                "achieved_timed_region": expand_bytes / (ms_expand_timed / 1000.0) / 1e9 if ms_expand_timed else None,
                "share_of_step": ms_expand_timed / ms if ms else None,
                "timing": "CUDA events around every expansion launch of one extra step run right after the "
                          "timed region (host-driven loop); the timed steps themselves run the graph loop and "
                          "report the device %globaltimer span of every launch (achieved_timed_region)",
                "peak_source": peak_src, "per_unit": per_unit, "traffic_source": tr.get("source"),
                "alu": alu}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, row_ptr, col, thr, args.cpu_samples or None)
    entry_colours = 64.0 * (infos[0]["batch_groups"] if cfg.model == "IC" and cfg.colors == 64 and infos
                            and infos[0]["batch_groups"] <= 4 else 1)
    line = {
        "metric": METRICS.get(cfg.name, METRIC), "value": cfg.theta / (ms_max / 1000.0), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": workload_desc(cfg), "theta": cfg.theta, "colors": cfg.colors, "k": cfg.k,
                   "step": f"graph_load + sample + extract({EXTRACT_SAMPLES}/rank) + select_seeds(k={cfg.k})",
                   "seeds": f"sampling seed rotates over {cfg.seed:#x} + (0, 1, 2) across steps",
                   "l2": (f"graph input {(row_ptr.nbytes + col.nbytes + thr.nbytes) / 1e6:.0f} MB and "
                          f"{float(np.mean([i['store_bytes'] for i in infos])) / 1e9:.1f} GB store per rank, "
                          "written each step; the graph input alone exceeds the 126 MB L2 (no flush needed)"),
                   "parallelism": f"sample-sharded x{world} (NCCL in selection only)"},
        "edges_visited_per_s": e_phys_all / (ms_max / 1000.0),
        "unfused_equiv_edges_per_s": e_log_all / (ms_max / 1000.0),
        "fusion_factor": e_log_all / e_phys_all if e_phys_all else None,
        # live colours per frontier entry / the colours an entry carries (64 per block; the default
        # IC 64-colour form shares one frontier entry between the <= 4 blocks of a batch)
        "frontier_occupancy": (float(np.mean([i["members"] for i in infos])) /
                               (entry_colours * float(np.mean([i["frontier_entries"] for i in infos])))
                               if infos and infos[0]["frontier_entries"] else None),
        "frontier_entry_colours": entry_colours,
        "ms_sample_per_step": ms_sample,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "wide_fusion": wide,
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
        "gpu_launches_breakdown": {"host_launches": int(host_launches), "graph_kernel_executions": int(graph_kernels),
                                   "note": "graph kernels count themselves on the device (Ctl::kernels_run)"},
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on this node and wait for them; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
