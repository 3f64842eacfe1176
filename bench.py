#!/usr/bin/env python3
"""Benchmark: single-source matrix-scan Dijkstra solve at n=32768 (dense).

Metric (BASELINE.json): single-source solve ms and achieved HBM GB/s at
n=32768 dense, 1/2/4/8 B200 vs CPU.  Workload = BASELINE config 3:
graph_from_edges(generate_dense(32768, 32768), undirected), source 0.

* one step = one full solve (all n rounds) of the persistent kernel with the
  matrix resident in HBM; `value` = device ms per solve (CUDA events on the
  library's launch stream), max over ranks.
* `e2e` = the same solve through the reference-facing call
  dijkstra(G, s) with the uint64 host matrix: narrow + H2D + permute,
  solve, D2H of dist/pred, every step.
* N > 1 (torchrun): the matrix is column-partitioned (partition.hpp:31-41);
  each rank owns one shard and the per-round argmin is exchanged by device
  P2P stores over NVLink (CUDA IPC); scaling "strong".
* `--impl reference`: the reference's own CPU code (oracle/_ref, compiled
  from /root/reference headers) on the box's host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEFAULT = 32768
SEED_DEFAULT = 32768
METRIC = "single-source solve ms and achieved HBM GB/s at n=32768 dense, 1/2/4/8 B200 vs CPU"


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    smax.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, val in zip(names, parts[5:9]):
                    if val.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def build_graph(n, seed, kind, cols=None):
    import paper_2504_03667_b200 as P
    if kind == "dense":
        return P.generate_dense(n, seed, cols=cols)
    if kind == "bernoulli":
        return P.generate_bernoulli(n, 0.5, seed, cols=cols)
    raise ValueError(kind)


def host_info() -> dict:
    """The host the CPU baseline ran on (lscpu model, nproc, free -g)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
            elif line.startswith("Socket(s):"):
                info["sockets"] = int(line.split(":", 1)[1])
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            kb = int(f.readline().split()[1])
        info["mem_total_gb"] = round(kb / 2**20, 1)
    except Exception:
        pass
    return info


def rotating_sources(n: int, first: int, k: int) -> list:
    """k distinct-ish sources, `first` first: consecutive timed solves read
    different rows of a matrix larger than L2 (the L2 rule of the timing contract)."""
    return [(first + 7919 * i) % n for i in range(k)]


def self_launch(nproc: int) -> int:
    """Re-runs this command under torch.distributed.run with nproc ranks on
    127.0.0.1 (a free port); returns the launcher's exit code."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_reference(args, rank, world):
    """The reference's own CPU implementation (oracle/_ref), rank 0 only."""
    if rank != 0:
        return
    import ctypes

    import oracle
    C, R = oracle.C(), oracle.REF()
    n = args.n
    adj = C.dense(n, args.seed) if args.graph == "dense" else C.bernoulli(n, 0.5, args.seed)
    h = R.lib.ref_graph_new(adj.ctypes.data_as(oracle._u64p), n, 0)
    del adj
    dist = np.empty(n, np.uint64)
    pred = np.empty(n, np.uint64)
    nproc = os.cpu_count() or 1
    ph = (ctypes.c_double * 3)()

    def serial():
        t = time.perf_counter()
        assert R.lib.ref_graph_serial(h, args.source, oracle._p(dist), oracle._p(pred)) == 0
        return time.perf_counter() - t

    def partitioned():
        t = time.perf_counter()
        assert R.lib.ref_graph_partitioned(h, args.source, nproc, oracle._p(dist), oracle._p(pred),
                                           ph) == 0
        return time.perf_counter() - t

    engines = {"serial": (serial, 1), f"partitioned(p={nproc})": (partitioned, nproc)}
    probe = {}
    for name, (fn, _) in engines.items():  # the first warm-up pass picks the faster engine
        if name.startswith("partitioned") and args.ref_skip_partitioned:
            continue
        probe[name] = fn()
    best = min(probe, key=probe.get)
    fn, cores = engines[best]
    for _ in range(max(0, args.warmup - 1)):
        fn()
    times = [fn() for _ in range(args.steps)]
    ms = 1e3 * float(np.mean(times))
    R.lib.ref_graph_free(h)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(ms, 3), "unit": "ms",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": {"workload": f"generate_dense({n},{args.seed}) undirected, "
                                                    f"source {args.source}", "n": n},
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": cores, "kind": "reference",
                         "sample": f"full {best} solve per step (reference dijkstra_* from "
                                   f"/root/reference/proj/include compiled into oracle/_ref)",
                         "engine_probe_ms": {k: round(v * 1e3, 1) for k, v in probe.items()},
                         "host": host_info()},
        "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_configs(P, torch, peak, args) -> dict:
    """BASELINE configs 1 (sparse + dense), 2 and 4 on one GPU: device ms per
    solve (back to back, rotating sources, CUDA events), rows streamed, HBM
    fraction, the reference's serial CPU solve of source 0 on this host as the
    baseline AND the parity gate (bit-exact dist + pred, serial.hpp:26-68)."""
    import oracle
    R = oracle.REF()
    ENG = P.ENGINE_NAMES
    specs = [("1-sparse", "generate_sparse(1000,42) undirected",
              lambda: P.generate_sparse(1000, 42)),
             ("1-dense", "generate_dense(1000,42) undirected", lambda: P.generate_dense(1000, 42)),
             ("2", "Bernoulli(16384, p=0.5, seed 16384) undirected",
              lambda: P.generate_bernoulli(16384, 0.5, 16384)),
             ("4", "Bernoulli(65536, p=0.001, seed 65536) DIRECTED (-w), 1 GPU here (8 in BASELINE)",
              lambda: P.generate_bernoulli(65536, 0.001, 65536, directed=True))]
    out = {}
    for name, wl, build in specs:
        t0 = time.perf_counter()
        g = build()
        t_build = time.perf_counter() - t0
        hg = R.graph(g.adj, g.n, int(g.directed))
        d, p, cpu_s = R.graph_serial(hg, g.n, 0)
        R.graph_free(hg)
        k = 10 if g.n > 20000 else 20
        srcs = rotating_sources(g.n, 0, k)
        with P.DeviceGraph(g) as dg:
            r0 = dg.solve(0)
            same = bool(np.array_equal(r0.dist, d) and np.array_equal(r0.pred, p))
            if not same:
                raise SystemExit(f"PARITY FAILURE: config {name} != reference dijkstra_serial")
            invalid = sum(int(dg.validate(dg.solve(s)) != 0) for s in srcs)
            if invalid:
                raise SystemExit(f"VALIDATION FAILURE: config {name}: {invalid} sources")
            stream = torch.cuda.ExternalStream(dg.stream_ptr())
            for s in srcs[:3]:
                dg.enqueue([s])
                dg.finish()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):  # launches queued ahead of the timed region
                torch.cuda._sleep(int(k * 100_000))
            e0.record(stream)
            for s in srcs:
                dg.enqueue([s])
            e1.record(stream)
            st = dg.finish()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / k
            rows = nb = 0
            for s in srcs:
                dg.enqueue([s])
                x = dg.finish()
                rows += x["rows_read"]
                nb += x["bytes_read"]
            rows /= k
            nb /= k
            info = dg.info()
            lat = None
            if ENG[st["engine"]] == "bucket":  # the sync skeleton bound (as the headline's)
                nbar = int(st["barriers"])
                t_skel = dg.probe_skeleton(nbar, 100) * 1e3
                t_hbm = nb / (peak * 1e9) * 1e3
                lat = {"bound": "sync+hbm", "barriers": nbar, "t_skeleton_ms": round(t_skel, 5),
                       "t_hbm_ms": round(t_hbm, 5), "frac": round((t_skel + t_hbm) / ms, 4)}
        out[name] = {"workload": wl, "n": g.n, "engine": ENG[st["engine"]],
                     "ms_per_solve": round(ms, 4), "kernel_ms": round(st["rounds_s"] * 1e3, 4),
                     "sources": f"{k} rotating (0, 7919, ...)", "classes": st["classes"],
                     "rows_read_mean": round(rows, 1), "bytes_read_mean": int(nb),
                     "weight_bytes": info["weight_bytes"],
                     "roofline": {"bound": "hbm", "achieved_gbs": round(nb / (ms * 1e-3) / 1e9, 1),
                                  "frac": round(nb / (ms * 1e-3) / 1e9 / peak, 4)},
                     "latency_roofline": lat,
                     "parity": "source 0 dist and pred bit-identical to dijkstra_serial; all %d "
                               "timed sources validate_result-valid" % k,
                     "cpu_baseline": {"value": round(cpu_s * 1e3, 2), "unit": "ms", "cores": 1,
                                      "kind": "reference",
                                      "sample": "dijkstra_serial (oracle/_ref) from source 0"},
                     "speedup_vs_cpu": round(cpu_s * 1e3 / ms, 1), "build_s": round(t_build, 1)}
        print(f"config {name}: {json.dumps(out[name])}", file=sys.stderr, flush=True)
        del g
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--vertices", dest="n", type=int, default=N_DEFAULT)
    ap.add_argument("--seed", type=int, default=SEED_DEFAULT)
    ap.add_argument("--graph", default="dense", choices=["dense", "bernoulli"])
    ap.add_argument("--source", type=int, default=0)
    ap.add_argument("--flags", type=int, default=None)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--engine", default="auto", choices=["auto", "cluster", "grid", "bucket"])
    ap.add_argument("--warps", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batch", action="store_true", help="skip the config-5 batch object")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config objects (BASELINE configs 1, 2, 4, 5)")
    ap.add_argument("--ref-skip-partitioned", action="store_true")
    ap.add_argument("--no-host-driven", action="store_true",
                    help="skip the host-driven per-round allreduce comparison (SURVEY §8e)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: start the N ranks
        # (one process per GPU) ourselves, exactly as the driver's torchrun does
        raise SystemExit(self_launch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import paper_2504_03667_b200 as P

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (there is no CPU path)")
    # test knobs: run all ranks on one GPU over gloo (the 1-GPU multi-process check)
    if os.environ.get("SSSP_BENCH_ONE_GPU"):
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if os.environ.get("SSSP_BENCH_ONE_GPU"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    n = args.n
    # ---- input (untimed, as in the reference: PAPER.md:35, bench.hpp:43-44)
    t0 = time.perf_counter()
    if world == 1:
        g = build_graph(n, args.seed, args.graph)
        block = None
    else:
        loc_n = P.pad_vertex_count(n, world) // world
        cb = rank * loc_n
        cc = max(0, min(loc_n, n - cb))
        block = build_graph(n, args.seed, args.graph, cols=(cb, cc))
        g = None
    t_build = time.perf_counter() - t0

    def open_graph(engine):
        if world == 1:
            return P.DeviceGraph(g, (local_rank,), flags=args.flags, ctas=args.ctas, engine=engine,
                                 warps=args.warps)
        from paper_2504_03667_b200 import distributed as D
        return D.open_shard(block, n, max_weight=100, device=local_rank, flags=args.flags,
                            ctas=args.ctas, engine=engine)

    def time_engine(dg, steps, warmup, sample_clocks=False, sources=None):
        """W untimed + K timed solves queued back to back, CUDA events on the
        library's launch stream, barrier + synchronize on both sides, max over
        ranks.  `sources` rotate (default: args.source only)."""
        stream = torch.cuda.ExternalStream(dg.stream_ptr())
        srcs = sources or [args.source]
        for i in range(warmup):
            dg.enqueue([srcs[(i + 1) % len(srcs)]])
            dg.finish()
        sampler = ClockSampler(local_rank) if sample_clocks else None
        if sampler:
            sampler.start()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        ev_s = torch.cuda.Event(enable_timing=True)
        ev_e = torch.cuda.Event(enable_timing=True)
        # The K launches are queued behind a device-side sleep so that the
        # timed region holds exactly the K back-to-back solves: the host's
        # launch cost (~11 us per enqueue, 20-25 us while nvidia-smi samples
        # the clocks) is then not device idle time inside the region.  The
        # host cost of a call is what `e2e` measures.
        with torch.cuda.stream(stream):
            torch.cuda._sleep(int(steps * 100_000))  # ~50 us of GPU clock per queued solve
        ev_s.record(stream)
        t_h0 = time.perf_counter()
        for i in range(steps):  # queued back to back in stream order
            dg.enqueue([srcs[i % len(srcs)]])
        t_h1 = time.perf_counter()
        ev_e.record(stream)
        if os.environ.get("SSSP_BENCH_DEBUG"):
            print(f"time_engine: host enqueue {1e6 * (t_h1 - t_h0) / steps:.2f} us/solve", file=sys.stderr)
        st = dg.finish()
        kern = [st["rounds_s"]]
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        clocks = sampler.stop() if sampler else None
        ms = ev_s.elapsed_time(ev_e) / steps
        kms = 1e3 * float(np.mean(kern))
        if dist is not None:
            t = torch.tensor([ms, kms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, kms = float(t[0]), float(t[1])
        return ms, kms, st, clocks

    def time_cold(dg, sources, reps):
        """Per-solve CUDA events with a 256 MiB write (> 126 MB L2) before every
        solve: each solve starts with a cold L2 (and pays its own launch)."""
        stream = torch.cuda.ExternalStream(dg.stream_ptr())
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        ts = []
        for i in range(reps + 2):
            with torch.cuda.stream(stream):
                flush.fill_(i & 0xFF)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            dg.enqueue([sources[i % len(sources)]])
            e1.record(stream)
            dg.finish()
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        del flush
        return float(np.mean(ts)), float(np.min(ts))

    peak, peak_src = measured_peaks()
    loc_cols = n if world == 1 else P.pad_vertex_count(n, world) // world
    ENG = {1: "grid", 2: "cluster", 3: "bucket"}

    # ---- the default engine (what dijkstra(G, s) runs) -> `value`: K solves
    # from K different sources back to back (each reads different rows of the
    # 1 GiB matrix, > 126 MB L2), then every timed source's result validated
    dg = open_graph(args.engine)
    info = dg.info()
    wb = info["weight_bytes"]
    srcs = rotating_sources(n, args.source, args.steps) if world == 1 else [args.source]
    ms, kern_ms, st, clocks = time_engine(dg, args.steps, args.warmup, sample_clocks=True,
                                          sources=srcs)
    engine = ENG[st["engine"]]
    res0 = dg.solve(args.source) if world == 1 else None
    validated = None
    if world == 1:
        bad = 0
        for s in sorted(set(srcs)):
            bad += dg.validate(dg.solve(s)) != 0
        validated = {"sources": len(set(srcs)), "invalid": int(bad),
                     "check": "validate_result (oracle.hpp:51-120) on the device for every timed "
                              "source; source %d also bit-exact vs the reference's dijkstra_serial "
                              "(cpu_baseline.parity)" % args.source}
        if bad:
            raise SystemExit(f"VALIDATION FAILURE: {bad} timed sources invalid")
    rows, alg_bytes = st["rows_read"], st["bytes_read"]  # of the last timed solve
    # matrix bytes per solve, averaged over the timed sources (each solve reads
    # only what its distance classes need; the kernel counts every load)
    if world == 1:
        rsum = bsum = 0
        for s in srcs:
            dg.enqueue([s])
            x = dg.finish()
            rsum += x["rows_read"]
            bsum += x["bytes_read"]
        rows, alg_bytes = rsum / len(srcs), bsum / len(srcs)
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    cold = time_cold(dg, srcs, 10) if world == 1 else None
    skel = None
    if world == 1 and engine == "bucket":
        nbar = int(st["barriers"])
        t_skel = dg.probe_skeleton(nbar, 100) * 1e3  # ms per launch, same shape, no data
        t_hbm = alg_bytes / (peak * 1e9) * 1e3
        skel = {"bound": "sync+hbm", "barriers": nbar, "t_skeleton_ms": round(t_skel, 5),
                "t_hbm_ms": round(t_hbm, 5), "t_roof_ms": round(t_skel + t_hbm, 5),
                "frac": round((t_skel + t_hbm) / ms, 4),
                "note": "floor of a solve with this many grid barriers: the same cooperative "
                        "launch doing only the barriers, back to back (sssp_probe_skeleton, "
                        "this run), plus its algorithmic bytes at the measured HBM peak; "
                        "frac = t_roof / ms_per_step"}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            with open(tpath) as f:
                traffic = json.load(f).get(f"{engine}:{n}")
        except Exception:
            traffic = None
    transfer_in_s = info["transfer_in_s"]
    # ---- the paper's data-parallel engine on the same resident graph (one
    # shard): rounds to the fixpoint + reconstruct_predecessors, timed beside
    dp = None
    if world == 1:
        best_dp = None
        for _ in range(4):
            x = dg.solve_dataparallel(args.source)
            best_dp = x if best_dp is None or x.stats["rounds_s"] < best_dp.stats["rounds_s"] else best_dp
        dst = best_dp.stats
        dp_ms = dst["rounds_s"] * 1e3
        dp_bytes = dst["rows_read"] * loc_cols * wb
        dp = {"engine": "dataparallel (dijkstra_dataparallel: relax rounds + reconstruct_predecessors)",
              "ms": round(dp_ms, 4), "rounds": dst["rounds"], "rows_read": dst["rows_read"],
              "achieved_gbs": round(dp_bytes / (dp_ms * 1e-3) / 1e9, 1),
              "frac_hbm": round(dp_bytes / (dp_ms * 1e-3) / 1e9 / peak, 4),
              "dist_equals_serial": bool(np.array_equal(best_dp.dist, res0.dist))}
    dg.close()

    # ---- the north-star n-round persistent scan kernel, timed beside it
    scan = None
    if engine == "bucket" or args.engine == "auto":
        sdg = open_graph("cluster")
        t_sync = sdg.probe_sync(rounds=min(n, 20000))
        k2 = max(3, args.steps // 4)
        sms, skms, sst, _ = time_engine(sdg, k2, 3)
        rounds = sst["iterations"]
        t_hbm_ms = n * loc_cols * wb / (peak * 1e9) * 1e3
        t_sync_ms = rounds * t_sync * 1e3
        scan = {"engine": "cluster (n-round persistent kernel, DSMEM exchange)", "ms": round(sms, 4),
                "kernel_ms": round(skms, 4), "steps": k2, "rounds": rounds,
                "mispredicts": sst["mispredicts"],
                "achieved_gbs": round(n * loc_cols * wb / (skms * 1e-3) / 1e9, 2),
                "latency_roofline": {"t_hbm_ms": round(t_hbm_ms, 4),
                                     "t_sync_round_us": round(t_sync * 1e6, 4),
                                     "t_sync_ms": round(t_sync_ms, 3),
                                     "t_roof_ms": round(max(t_hbm_ms, t_sync_ms), 3),
                                     "frac": round(max(t_hbm_ms, t_sync_ms) / skms, 4),
                                     "note": "max(n*n_local*wbytes / HBM, rounds * t_sync_min); "
                                             "t_sync_min measured by sssp_probe_sync in this run"}}
        if world == 1:
            r1 = sdg.solve(args.source)
            assert r1 == res0, "scan engine != default engine"
        # SURVEY §8e comparison: the same rounds with a HOST-driven per-round
        # all_reduce(MIN) of the 8-byte key (NCCL at N > 1) between a
        # local_min and a relax launch, padded_n rounds like the reference
        if not args.no_host_driven:
            from paper_2504_03667_b200 import distributed as D
            hd = []
            for _ in range(2):  # warm-up + timed
                if dist is not None:
                    dist.barrier()
                dl, pl, secs = D.solve_host_driven(sdg, n, args.source)
                hd.append(secs)
            t = hd[-1]
            if dist is not None:
                tt = torch.tensor([t], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                t = float(tt[0])
            same = None
            if world == 1:
                same = bool(np.array_equal(dl, res0.dist) and np.array_equal(pl, res0.pred))
                if not same:
                    raise SystemExit("PARITY FAILURE: host-driven rounds != device engine")
            rounds_hd = P.pad_vertex_count(n, world)
            scan["host_driven"] = {
                "ms": round(t * 1e3, 3), "rounds": rounds_hd,
                "us_per_round": round(t * 1e6 / rounds_hd, 3),
                "collective": ("torch.distributed all_reduce(int64 MIN) per round, NCCL "
                               if world > 1 else "none (one rank): ") + "between 2 launches",
                "equals_device_engine": same,
                "note": "host-driven local_min -> allreduce -> relax per round (sssp_nccl_*), "
                        "the comparison for the device-initiated per-round exchange above"}
        sdg.close()
        # per-round latency histogram (%globaltimer at every round end; one
        # extra traced solve, outside the timed region)
        if world == 1:
            with P.DeviceGraph(g, (local_rank,), flags=args.flags, engine="cluster",
                               round_times=True) as tdg:
                tdg.solve(args.source)
                d = np.diff(tdg.round_times().astype(np.int64)) / 1e3  # us
            edges = [0, 0.3, 0.4, 0.5, 0.6, 0.8, 1.0, 2.0, 5.0, float("inf")]
            hist, _ = np.histogram(d, bins=edges)
            scan["round_latency_us"] = {
                "rounds": int(d.size + 1), "p50": round(float(np.percentile(d, 50)), 4),
                "p90": round(float(np.percentile(d, 90)), 4),
                "p99": round(float(np.percentile(d, 99)), 4), "max": round(float(d.max()), 3),
                "mean": round(float(d.mean()), 4),
                "histogram": {f"{a}-{b}": int(c) for a, b, c in zip(edges[:-1], edges[1:], hist)},
                "note": "%globaltimer deltas between consecutive round ends (CTA 0 of the cluster)"}

    # ---- BASELINE config 5 beside it: 64 sources 256*k on the config-2 graph
    # (n=16384 Bernoulli 0.5), sources split across ranks, one full replica
    # per GPU, no cross-GPU traffic; device ms for all 64 (max over ranks)
    batch = None
    if not args.no_batch:
        gb = P.generate_bernoulli(16384, 0.5, 16384)
        bsrcs = [256 * k for k in range(64)][rank::world]
        with P.DeviceGraph(gb, (local_rank,)) as bdg:
            bstream = torch.cuda.ExternalStream(bdg.stream_ptr())
            for _ in range(2):
                bdg.enqueue(bsrcs)
                bdg.finish()
            if dist is not None:
                dist.barrier()
            torch.cuda.synchronize()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b0.record(bstream)
            bdg.enqueue(bsrcs)
            b1.record(bstream)
            bst = bdg.finish()
            torch.cuda.synchronize()
            bms = b0.elapsed_time(b1)
            # parity: every source validated on the device (validate_result),
            # the first two bit-exact against the reference's dijkstra_serial
            bres = bdg.solve_batch(bsrcs)
            binvalid = sum(int(bdg.validate(r) != 0) for r in bres)
        bpar = None
        if rank == 0 and not args.no_cpu_baseline:
            import oracle
            R = oracle.REF()
            hg = R.graph(gb.adj, gb.n)
            cpu_s, same = [], True
            for r in bres[:2]:
                d, p, t = R.graph_serial(hg, gb.n, r.source)
                cpu_s.append(t)
                same &= bool(np.array_equal(d, r.dist) and np.array_equal(p, r.pred))
            R.graph_free(hg)
            if not same or binvalid:
                raise SystemExit("PARITY FAILURE: config-5 batch != reference dijkstra_serial")
            bpar = {"value": round(1e3 * float(np.mean(cpu_s)), 1), "unit": "ms per source",
                    "cores": 1, "kind": "reference",
                    "sample": f"dijkstra_serial (oracle/_ref) from sources {bsrcs[0]}, {bsrcs[1]}"}
        if dist is not None:
            t = torch.tensor([bms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            bms = float(t[0])
        batch = {"workload": "config 5: 64 sources 256*k, generate_bernoulli(16384, 0.5, 16384), "
                             "sources split over the GPUs, one replica each",
                 "ms_all_sources": round(bms, 4), "ms_per_source": round(bms / 64, 5),
                 "sources_per_gpu": len(bsrcs), "engine": ENG[bst["engine"]],
                 "rows_read": bst["rows_read"], "bytes_read": bst["bytes_read"] * len(bsrcs),
                 "achieved_gbs": round(bst["bytes_read"] * len(bsrcs) / (bms * 1e-3) / 1e9, 1),
                 "parity": ("all %d sources validate_result-valid on the device; sources %d, %d "
                            "bit-identical to dijkstra_serial" % (len(bres), bsrcs[0], bsrcs[1]))
                           if bpar else "device validate_result only",
                 "cpu_baseline": bpar,
                 "scaling": "strong (64 sources in total)"}
        del gb

    # context for the per-round exchange: a host-driven NCCL
    # 8-byte min-allreduce, the comparison path the device-initiated P2P
    # exchange replaces (N > 1 only)
    nccl_us = None
    if dist is not None and not os.environ.get("SSSP_BENCH_ONE_GPU"):
        x = torch.zeros(1, dtype=torch.int64, device="cuda")
        for _ in range(20):
            dist.all_reduce(x, op=dist.ReduceOp.MIN)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            dist.all_reduce(x, op=dist.ReduceOp.MIN)
        e1.record()
        torch.cuda.synchronize()
        nccl_us = e0.elapsed_time(e1) / 200 * 1e3
        if scan is not None:
            scan["nccl_allreduce_8b_us"] = round(nccl_us, 2)

    line = {
        "metric": METRIC, "value": round(ms, 4), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": {1: "u8", 2: "u16", 4: "u32"}[wb] + " weights / u32 dist",
        "data": "synthetic",
        "config": {"workload": f"graph_from_edges(generate_dense({n},{args.seed})) undirected, "
                               f"single source {args.source}",
                   "n": n, "parallelism": f"column-partitioned x{world}" if world > 1 else "1 GPU",
                   "engine": engine, "weight_bytes": wb,
                   "l2": (f"matrix {info['matrix_bytes'] / 2**20:.0f} MiB per GPU > 126 MB L2; the "
                          f"{len(set(srcs))} timed solves start from different sources "
                          f"({srcs[0]}, {srcs[1 % len(srcs)]}, ...: 7919-strided), so each reads "
                          f"different rows; ms_cold = the same solves each after a 256 MiB "
                          f"L2 flush, per-solve events (launch included)"),
                   "sources": "rotating" if world == 1 else "single",
                   "timing": "K solves queued back to back behind a device sleep (host launch "
                             "cost outside the device-timed region; it is in e2e), CUDA events "
                             "on the launch stream bracketing exactly the K solves"},
        "kernel_ms": round(kern_ms, 4),
        "ms_cold": round(cold[0], 4) if cold else None,
        "solve": {"vertices_settled": st["iterations"], "classes": st["classes"],
                  "rows_read_mean": round(float(rows), 1), "barriers": st["barriers"],
                  "mispredicts": st["mispredicts"], "validated": validated},
        "gpu_launches": args.steps,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 5), "traffic": traffic,
                     "peak_source": peak_src, "bytes_per_launch": int(alg_bytes),
                     "note": "algorithmic bytes = matrix bytes the solve kernel loads, counted "
                             "by the kernel (stats.bytes_read; bucket: per class the tile slices "
                             "of the class rows (push), or the still-improvable columns' "
                             "transposed rows read in vertex-id order up to the first "
                             "min-weight hit (pull); columns whose dist <= next class + min "
                             "weight are final and never read; scan: n rows), mean over the "
                             "timed sources, / kernel_ms; ncu DRAM bytes in `traffic`"},
        "latency_roofline": skel,
        "scan_engine": scan,
        "dataparallel_engine": dp,
        "batch": batch,
        "clocks": clocks,
        "build_s": round(t_build, 2), "transfer_in_s": round(transfer_in_s, 4),
    }

    if world == 1:
        # ---- e2e: dijkstra(G, s) through the public API with host buffers
        e2e = []
        r = None
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = P.dijkstra(g, args.source, device=local_rank)
            e2e.append(time.perf_counter() - t)
        e2e_ms = 1e3 * float(np.mean(e2e[1:])) if len(e2e) > 1 else 1e3 * e2e[0]
        line["e2e"] = {"value": round(e2e_ms, 3), "unit": "ms",
                       "h2d_bytes_per_step": int(n * n * wb + 8), "d2h_bytes_per_step": int(16 * n),
                       "note": "uint64 host matrix narrowed on host threads, pinned H2D, device "
                               "permute (+ transpose/symmetry check), solve, D2H; graph handle "
                               "created per call"}
        assert r == res0
        # ---- CPU baseline + parity gate (reference serial, 1 core)
        if not args.no_cpu_baseline:
            import oracle
            R = oracle.REF()
            hg = R.graph(g.adj, n)
            d, p, cpu_s = R.graph_serial(hg, n, args.source)
            R.graph_free(hg)
            ok = np.array_equal(d, res0.dist) and np.array_equal(p, res0.pred)
            if not ok:
                raise SystemExit("PARITY FAILURE: GPU result != reference dijkstra_serial")
            line["cpu_baseline"] = {"value": round(cpu_s * 1e3, 1), "unit": "ms", "cores": 1,
                                    "kind": "reference",
                                    "sample": "one full dijkstra_serial solve of the same graph "
                                              "(oracle/_ref, reference headers), source %d; timing "
                                              "scope {algorithm} as timed_run (bench.hpp:114-180), "
                                              "graph build excluded (PAPER.md:35)" % args.source,
                                    "parity": "dist and pred bit-identical",
                                    "host": host_info()}
        # ---- BASELINE configs 1, 2 and 4 beside the headline (config 5 is
        # `batch`), each parity-gated against the reference's dijkstra_serial
        if not args.no_configs:
            del g
            line["configs"] = run_configs(P, torch, peak, args)
    else:
        # ---- e2e at N GPUs: the collective dijkstra_distributed call -- every
        # rank uploads its host column block (narrow + H2D + permute), the
        # shards connect (IPC handles), solve, owned slices gathered to every
        # rank; wall time per call, max over ranks
        from paper_2504_03667_b200 import distributed as D
        e2e = []
        for i in range(args.e2e_steps + 1):
            dist.barrier()
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = D.dijkstra_distributed(block, n, args.source, 100, local_rank)
            torch.cuda.synchronize()
            dt = torch.tensor([time.perf_counter() - t], dtype=torch.float64)
            if dist.get_backend() == "nccl":
                dt = dt.cuda()
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            e2e.append(float(dt.item()))
        e2e_ms = 1e3 * float(np.mean(e2e[1:])) if len(e2e) > 1 else 1e3 * e2e[0]
        line["e2e"] = {"value": round(e2e_ms, 3), "unit": "ms",
                       "h2d_bytes_per_step": int(n * loc_cols * wb * world),
                       "d2h_bytes_per_step": int(16 * n),
                       "note": "collective dijkstra_distributed: every rank narrows and uploads its "
                               "uint64 column block, connects, solves, gathers the owned slices; "
                               "max over ranks"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
