#!/usr/bin/env python
"""Benchmark of the B200 community-detection hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl b200|reference]

One "step" = one complete detector run (the reference's RunReport.total_ms
region, H/plp.hpp:70-142, H/louvain.hpp:277-279) over one synthetic graph
resident in HBM.  Metric: edges/s = m (undirected edges, the reference CLI
bench's edge_count(), P/tools/commdet.cpp:241-245) / step time.  Default
workload = the largest single-GPU config, BASELINE.json configs[2] (C3):
PLP on R-MAT scale 24 (520.8M CSR entries); c3_rmat24_plm is the same graph
under PLM.

value      device time (CUDA events on the library stream), graph + output in HBM,
           L2 flushed (256 MiB write) before every timed step.
e2e        the same metric through the public C ABI with HOST buffers: pinned
           host CSR -> cd_graph_from_csr (H2D + validation + finalize) ->
           cd_plp_run / cd_louvain_run with a host output (D2H of the labels).
roofline   the dominant kernel family (the sweep: every tier kernel of a
           sub-sweep, run as concurrent branches exactly as in the timed step,
           timed as one unit with CUDA events around the group, so family time
           <= step time), algorithmic bytes per DESIGN.md's byte model vs
           MEASURED_PEAKS.json hbm_gbs; "kernels" = each tier kernel timed
           alone on a serialised pass (diagnostic).
quality    modularity / communities of the device run vs the reference: the
           live CPU baseline run (default order, all threads) and, for PLP, the
           named parity setting (randomize_order, seed 1, 1 worker; SURVEY.md
           8(c)) cached by tests/golden/make_ref_quality.py on the same bytes.
cpu_baseline  the unmodified reference (oracle/_ref) on identical bytes (the C
           port of the generator), all host threads, rank 0 at N=1.
--impl reference  the reference arm: the same metric from oracle/_ref only.
--gpus N   without a torchrun environment, re-launches itself under
           torch.distributed.run with N ranks (127.0.0.1).
Multi-GPU (torchrun), --parallel:
  replicas   one independent graph per rank, no collective (weak scaling);
             value = all ranks' edges / max-over-ranks time.  Default for the
             graphs that fit one GPU's work (C1, C2, C4).
  rows       one graph sharded by rows across the ranks:
             every rank evaluates its own nodes, move lists are allgathered
             over NCCL after each sub-sweep, coarse levels replicated (strong
             scaling); value = m / max-over-ranks time.  Default for C3 / C5.
  replicated the same with the whole graph on every rank.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PLP/PLM edges/sec at 1/2/4/8 B200, % HBM roofline; modularity vs CPU ref"

LFR_C2 = dict(n=1_000_000, tau1=2.0, avg_degree=20.0, max_degree=200, tau2=1.0, min_community=20,
              max_community=1000, mu=0.3)

WORKLOADS = {
    # BASELINE.json configs[1] -- the headline (fits one GPU)
    "c2_lfr_plm": dict(gen="lfr", algo="plm", seed=1,
                       desc="PLM gamma=1 on LFR-shaped n=1e6 (tau1=2, mean 20, max 200, tau2=1, [20,1000], mu=0.3)"),
    "c1_planted_plp": dict(gen="planted", algo="plp", seed=1,
                           desc="PLP on planted partition n=1e5, k=1000, p_in=0.1, p_out=2/99900"),
    "c1_planted_plm": dict(gen="planted", algo="plm", seed=1, desc="PLM on config-1 planted graph"),
    # a seconds-sized planted graph for the contract tests (not a bench config)
    "t0_planted_plp": dict(gen="planted", algo="plp", seed=3, n=2000, k=8, p_in=0.05, p_out=0.002,
                           desc="PLP on a planted partition n=2000, k=8 (test workload)"),
    "c3_rmat24_plp": dict(gen="rmat", scale=24, weighted=False, algo="plp", seed=1,
                          desc="PLP on R-MAT scale 24 ef 16 (0.57,0.19,0.19,0.05)"),
    "c3_rmat24_plm": dict(gen="rmat", scale=24, weighted=False, algo="plm", seed=1,
                          desc="PLM on R-MAT scale 24 ef 16"),
    "c4_rmat22w_plmr": dict(gen="rmat", scale=22, weighted=True, algo="plmr", seed=1,
                            desc="PLMR on weighted R-MAT scale 22 ef 16"),
    "c4_rmat22w_epp": dict(gen="rmat", scale=22, weighted=True, algo="epp", seed=1,
                           desc="EPP(4,PLP,PLMR) on weighted R-MAT scale 22 ef 16"),
    # BASELINE.json configs[4]: 8.5e9 entries; fits one B200 through the
    # chunked builder / batched contraction, row shards built per rank at N > 1
    "c5_rmat28_plm": dict(gen="rmat", scale=28, weighted=False, algo="plm", seed=1, cpu=False,
                          desc="PLM on R-MAT scale 28 ef 16 (0.57,0.19,0.19,0.05), int64 offsets"),
    "c5_rmat28_plp": dict(gen="rmat", scale=28, weighted=False, algo="plp", seed=1, cpu=False,
                          desc="PLP on R-MAT scale 28 ef 16"),
}
# graphs whose multi-GPU mode is one sharded graph rather than replicas
SHARDED_BY_DEFAULT = {"c3_rmat24_plp", "c3_rmat24_plm", "c5_rmat28_plm", "c5_rmat28_plp"}
# the reference is infeasible there (~240 GB RAM, hours)
NO_CPU_REASON = "reference infeasible at R-MAT scale 28 (SURVEY.md 8(d): ~240 GB host RAM, hours per run)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3_rmat24_plp", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--parallel", default=None, choices=["replicas", "rows", "replicated"],
                    help="multi-GPU mode (default: rows for C3, replicas otherwise)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=15.0, help="bound on the cpu_baseline sample")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class NvmlClockSampler:
    """SM clocks and clock-event (throttle) reasons during the timed region,
    read through NVML by the bench loop itself between timed steps (outside
    each step's CUDA events), at most every 200 ms (the recipe's interval) and
    at both ends of the region.  NVML queries taken concurrently with a step
    stalled it: an `nvidia-smi -lms 200` process gave C3 PLM timed steps of
    253 / 306 ms among 198 ms ones, a sampling thread a C2 step of 22 ms among
    6.8 ms ones; between steps they cannot touch a measurement."""

    NAMES = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
             ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
             ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
             ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = None
        try:  # the CUDA device's own NVML handle (indices may differ)
            import torch
            pr = torch.cuda.get_device_properties(device)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        self.samples = []
        self.window = None
        self.last = 0.0

    def _sample(self):
        import datetime
        nv = self.nv
        try:
            sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append((datetime.datetime.now(), float(sm), float(mx), int(rs)))
        except Exception:
            pass

    def start(self):
        # the first queries initialise NVML's per-device state (it stalled a
        # timed step by 45 ms): done here, before the warm-up
        for _ in range(3):
            self._sample()
        self.samples.clear()
        self.last = 0.0

    def between_steps(self):
        """Called by the timed loop after a step's closing event has completed."""
        if time.perf_counter() - self.last >= 0.2:
            self._sample()
            self.last = time.perf_counter()

    def mark_begin(self):
        import datetime
        self.window = [datetime.datetime.now(), None]
        self._sample()
        self.last = time.perf_counter()

    def mark_end(self):
        import datetime
        self._sample()
        if self.window:
            self.window[1] = datetime.datetime.now()

    def stop(self):
        import datetime
        rows = self.samples
        if self.window and self.window[1]:
            inside = [r for r in rows if self.window[0] <= r[0] <= self.window[1]]
            rows = inside or rows
        if not rows:
            return None
        reasons = sorted({name for r in rows for name, attr in self.NAMES
                          if r[3] & getattr(self.nv, attr, 0)})
        return {"sm_mhz": statistics.median(r[1] for r in rows), "sm_max_mhz": max(r[2] for r in rows),
                "reasons": reasons, "samples": len(rows), "source": "nvml, between timed steps"}


def clock_sampler(device):
    """NVML in-process when pynvml works, else the nvidia-smi process."""
    try:
        return NvmlClockSampler(device)
    except Exception:
        return ClockSampler(device)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region.  Started
    before the warm-up (nvidia-smi's start-up -- NVML initialisation -- then
    never overlaps the timed steps); only the samples stamped inside the timed
    window (mark_begin / mark_end) are reported."""

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None
        self.window = None

    def mark_begin(self):
        import datetime
        self.window = [datetime.datetime.now(), None]

    def mark_end(self):
        import datetime
        if self.window:
            self.window[1] = datetime.datetime.now()

    def start(self):
        if os.environ.get("CD_BENCH_NO_CLOCKS"):  # diagnostics only: the JSON line then has no clocks
            return
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        # (no power.draw: its query stalled the GPU's work for 50-240 ms now and
        # then -- C3 PLM timed steps of 253 / 266 ms among 199 ms ones)
        q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.device)], stdout=open(self.path, "w"),
                                         stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        # nvidia-smi's start-up (NVML initialisation) stalls the GPU's work for
        # tens of ms: wait for its first sample, so that it is over before the
        # warm-up (a short warm-up alone did not cover it: C3 PLP's first timed
        # step took 39 ms against 19.6 ms for the others)
        t0 = time.time()
        while time.time() - t0 < 10.0 and self.proc.poll() is None:
            if os.path.getsize(self.path) > 0:
                break
            time.sleep(0.02)
        time.sleep(0.3)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        import datetime
        rows = []
        with open(self.path) as f:
            for line in f:
                p = [x.strip() for x in line.split(",")]
                if len(p) >= 8:
                    try:
                        ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f")
                        rows.append((ts, float(p[1]), float(p[2]), p[4:8]))
                    except ValueError:
                        pass
        os.unlink(self.path)
        if self.window and self.window[1]:
            pad = datetime.timedelta(milliseconds=250)  # one sampling interval either side
            inside = [r for r in rows if self.window[0] - pad <= r[0] <= self.window[1] + pad]
            rows = inside or rows
        rows = [r[1:] for r in rows]
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[2]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def planted_args(wl):
    return (wl.get("n", 100000), wl.get("k", 1000), wl.get("p_in", 0.1), wl.get("p_out", 2 / 99900), wl["seed"])


def make_device_graph(P, ctx, wl, shard=False):
    """shard: this rank's row shard (R-MAT shards are generated directly,
    never holding the whole graph; other graphs are cut from the whole)."""
    if shard and wl["gen"] == "rmat":
        return P.generate_rmat(wl["scale"], 16, 0.57, 0.19, 0.19, weighted=wl["weighted"], seed=wl["seed"], ctx=ctx,
                               shard=True)
    if shard:
        return make_device_graph(P, ctx, wl).shard(ctx)
    if wl["gen"] == "lfr":
        g, _ = P.generate_lfr(seed=wl["seed"], ctx=ctx, **LFR_C2)
    elif wl["gen"] == "planted":
        g, _ = P.generate_planted(*planted_args(wl), ctx=ctx)
    else:
        g = P.generate_rmat(wl["scale"], 16, 0.57, 0.19, 0.19, weighted=wl["weighted"], seed=wl["seed"], ctx=ctx)
    return g


def make_oracle_graph(O, wl):
    """The identical graph through the C port / the reference generator."""
    if wl["gen"] == "lfr":
        return O.generate_lfr(seed=wl["seed"], **LFR_C2)[0]
    if wl["gen"] == "planted":
        rg, _ = O.RefGraph.planted(*planted_args(wl), workers=0)
        return rg.csr()
    return O.generate_rmat(wl["scale"], 16, 0.57, 0.19, 0.19, weighted=wl["weighted"], seed=wl["seed"])


def run_device(P, g, algo, out, report=False):
    if algo == "plp":
        return P.run_plp(g, P.PlpConfig(), out=out, report=report)
    if algo == "plm":
        return P.run_louvain(g, P.LouvainConfig(refine=False), out=out, report=report)
    if algo == "plmr":
        return P.run_louvain(g, P.LouvainConfig(refine=True), out=out, report=report)
    return P.run_epp(g, P.EnsembleConfig(), out=out)


def run_reference(O, rg, algo, workers):
    if algo == "plp":
        return rg.run_plp(workers=workers)[1]
    if algo == "plm":
        return rg.run_louvain(refine=False, workers=workers)[1]
    if algo == "plmr":
        return rg.run_louvain(refine=True, workers=workers)[1]
    return rg.run_epp(workers=workers)[1]


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# shared pieces of both arms' lines
# ---------------------------------------------------------------------------
def workload_config(args, wl, n, m, entries):
    """The workload-identifying config: identical keys and values in both arms."""
    return {"workload": args.workload, "desc": wl["desc"], "algo": wl["algo"], "seed": wl["seed"], "n": int(n),
            "m": int(m), "entries": int(entries)}


def cached_reference_quality(workload, digest=None):
    """tests/golden/ref_quality.json: the reference's results on the same bytes
    (tests/golden/make_ref_quality.py), keyed by workload/setting."""
    path = os.path.join(ROOT, "tests", "golden", "ref_quality.json")
    if not os.path.exists(path):
        return {}
    with open(path) as f:
        cache = json.load(f)
    out = {}
    for key, v in cache.items():
        wk, setting = key.split("/")
        if wk == workload and (digest is None or v["graph"]["digest"] == digest):
            out[setting] = {"modularity": v["modularity"], "communities": v["communities"], "workers": v["workers"],
                            "randomize_order": v["randomize_order"], "runs": v["runs"], "total_ms": v["total_ms"],
                            "host": v["host"]}
    return out


def graph_digest(off, col):
    import hashlib

    import numpy as np
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(off, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(col, dtype=np.int32).tobytes())
    return h.hexdigest()[:16]


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def bench_reference(args, wl):
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    if not O.ref_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libcommdet_ref.so not built"})
        return 0
    if wl.get("cpu") is False:
        emit({"impl": "reference", "unavailable": NO_CPU_REASON})
        return 0
    og = make_oracle_graph(O, wl)
    rg = O.RefGraph.from_csr(og)
    threads = cpu_threads()
    for _ in range(args.warmup):
        run_reference(O, rg, wl["algo"], threads)
    times, qs, ks = [], [], []
    for _ in range(args.steps):
        rep = run_reference(O, rg, wl["algo"], threads)
        times.append(rep["total_ms"] / 1e3)
        qs.append(rep["modularity"])
        ks.append(rep["community_count"])
    total = sum(times)
    value = og.m * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, wl, og.n, og.m, og.D),
        "parallelism": f"openmp x{threads}",
        "quality": {"modularity": statistics.median(qs), "communities": int(statistics.median(ks)),
                    "setting": f"reference defaults (ascending order), OMP workers={threads}"},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": threads, "kind": "reference",
                         "sample": f"{args.steps} complete runs of the reference {wl['algo']} (oracle/_ref, "
                                   f"OMP workers={threads}) on the identical graph"},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
SWEEP_FAMILY = {"plp": "plp_sweep", "plm": "plm_move", "plmr": "plm_move", "epp": "plp_sweep"}


def profile_pass(P, ctx, step, flush, mode, reps):
    """`reps` profiled runs (ctx profiling mode 1: every launch timed, sweep
    tiers serialised; 2: tiers concurrent as in the timed run, each
    sub-sweep's group timed as one unit).  Returns (kernel stats, total
    device ms of the profiled runs measured around each run)."""
    import torch
    stream = torch.cuda.ExternalStream(ctx.stream)
    ctx.reset_stats()
    ctx.set_profiling(mode)
    tot = 0.0
    for _ in range(reps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    ctx.set_profiling(0)
    return ctx.kernel_stats(), tot


def bench_b200(args, wl):
    import numpy as np
    import torch

    import paper_1304_4453_b200 as P

    world, rank, local = dist_env()
    dist = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) on stderr
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    ctx = P.Context(local)
    mode = "1gpu"
    if world > 1:
        mode = args.parallel or ("rows" if args.workload in SHARDED_BY_DEFAULT else "replicas")
    elif args.parallel in ("rows", "replicated"):
        mode = args.parallel  # world size 1 through the same NCCL exchange path
    sharded = mode in ("rows", "replicated")
    if sharded:
        # the library's own NCCL communicator (torch only carries the unique id)
        uid = [P.nccl_unique_id() if rank == 0 else None]
        if dist:
            dist.broadcast_object_list(uid, src=0)
        ctx.attach_nccl(world, rank, uid[0])
    g = make_device_graph(P, ctx, wl, shard=mode == "rows")
    n, m = g.node_count(), g.edge_count()
    entries = g.entries if mode != "rows" else g._info.D_global
    units = 1 if sharded else world  # graphs processed per step, all ranks
    out = torch.empty(max(n, 1), dtype=torch.int32, device=f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")

    def step():
        run_device(P, g, wl["algo"], out, report=False)

    clocks = clock_sampler(local)
    clocks.start()  # before the warm-up: its start-up must not overlap the timed steps
    warm_ms = []
    for _ in range(args.warmup):
        h0 = time.perf_counter()
        step()
        ctx.synchronize()
        warm_ms.append(1e3 * (time.perf_counter() - h0))
    print("warm-up steps, host wall (ms):", " ".join(f"{t:.2f}" for t in warm_ms), file=sys.stderr)
    # ---- timed region ------------------------------------------------------------
    import gc
    gc.collect()
    gc.disable()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_begin()
    launches0 = ctx.launch_count()
    total_ms = 0.0
    step_ms, host_ms = [], []
    for _ in range(args.steps):
        flush.fill_(1.0)  # evict L2 (256 MiB > 126 MB) outside the timed step
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record(stream)
        step()
        e1.record(stream)
        e1.synchronize()
        host_ms.append(1e3 * (time.perf_counter() - h0))
        step_ms.append(e0.elapsed_time(e1))
        total_ms += step_ms[-1]
        if hasattr(clocks, "between_steps"):  # outside the step's events
            clocks.between_steps()
    torch.cuda.synchronize()
    clocks.mark_end()
    gc.enable()
    print("timed steps (ms):", " ".join(f"{t:.2f}" for t in step_ms), file=sys.stderr)
    print("host wall (ms):", " ".join(f"{t:.2f}" for t in host_ms), file=sys.stderr)
    launches = ctx.launch_count() - launches0
    if dist:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{local}")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = units * m * args.steps / (total_ms / 1e3)

    # ---- quality of the run (modularity vs the CPU reference below) --------------
    z, rep = run_device(P, g, wl["algo"], None, report=True)
    quality = {"modularity": rep.modularity, "communities": rep.community_count,
               "levels": [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in l.items()}
                          for l in rep.levels],
               "iterations": len(rep.iterations), "run_ms": rep.total_ms}

    # ---- roofline: profiled passes of the same workload ---------------------------
    peak, peak_kind = measured_peak()
    fam = SWEEP_FAMILY[wl["algo"]]
    prof_steps = max(1, min(3, args.steps))
    # (a) the sweep family as it runs in the timed step: tier kernels concurrent,
    #     each sub-sweep's group timed as one unit (+ the one-kernel phases)
    gst, gstep_ms = profile_pass(P, ctx, step, flush, 2, prof_steps)
    # (b) every kernel timed alone (tiers serialised): per-tier diagnostics
    sst, sstep_ms = profile_pass(P, ctx, step, flush, 1, prof_steps)
    s = gst.get(fam) or {"total_ms": 0.0, "bytes": 0.0, "launches": 0}
    achieved = s["bytes"] / (s["total_ms"] / 1e3) / 1e9 if s["total_ms"] > 0 and s["bytes"] > 0 else None
    roofline = {"bound": "hbm", "kernel": fam, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": None, "peak_kind": peak_kind,
                "unit_of_launch": "one sub-sweep: its tier kernels as concurrent branches (as timed), "
                                  "or one cooperative phase kernel",
                "bytes_per_launch": s["bytes"] / max(s["launches"], 1),
                "avg_launch_ms": s["total_ms"] / max(s["launches"], 1), "launches": s["launches"] // prof_steps,
                "family_ms_per_step": s["total_ms"] / prof_steps,
                "profiled_step_ms": gstep_ms / prof_steps,
                "share_of_step": s["total_ms"] / gstep_ms if gstep_ms else None,
                "families_ms_per_step": {k: round(v["total_ms"] / prof_steps, 4) for k, v in
                                         sorted(gst.items(), key=lambda kv: -kv[1]["total_ms"])[:10]},
                # every sweep tier kernel timed alone (serialised pass) against the roofline
                "kernels_serialised_step_ms": sstep_ms / prof_steps,
                "kernels": {k: {"ms_per_step": round(v["total_ms"] / prof_steps, 4),
                                "achieved": round(v["bytes"] / (v["total_ms"] / 1e3) / 1e9, 2),
                                "frac": round(v["bytes"] / (v["total_ms"] / 1e3) / 1e9 / peak, 5)}
                            for k, v in sorted(sst.items(), key=lambda kv: -kv[1]["total_ms"])
                            if "." in k and v["bytes"] > 0 and v["total_ms"] > 0}}
    cs = gst.get("coarsen")
    if cs and cs["total_ms"] > 0 and cs["bytes"] > 0:
        # contraction (PLM / PLMR / EPP): the SURVEY.md 8(d) byte model per coarsening
        # over the coarsen kernels' time (they run on the library stream, serially)
        ca = cs["bytes"] / (cs["total_ms"] / 1e3) / 1e9
        roofline["contraction"] = {"achieved": ca, "frac": ca / peak, "ms_per_step": cs["total_ms"] / prof_steps,
                                   "bytes_per_step": cs["bytes"] / prof_steps,
                                   "share_of_step": cs["total_ms"] / gstep_ms if gstep_ms else None}
    prof_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof_path):
        with open(prof_path) as f:
            ps = json.load(f).get(args.workload, {}).get(fam)
        if ps and ps.get("dram_bytes_per_step"):
            # ncu DRAM bytes of the family's kernels per step, over the sub-sweeps
            roofline["traffic"] = ps["dram_bytes_per_step"] / max(roofline["launches"], 1)
            roofline["traffic_source"] = ps.get("source")

    # ---- end to end through the C ABI with host buffers ----------------------------
    # (rows mode: every rank uploads the offsets and only its own rows)
    c = (make_device_graph(P, ctx, wl) if mode == "rows" else g).csr()
    bounds = P.shard_bounds(c["off"], world) if mode == "rows" else None
    if entries >= 1 << 31:  # C5: room on the device for the uploaded copy
        g = None
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    h_off = pin(c["off"])
    if mode == "rows":
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        e0_, e1_ = int(c["off"][lo]), int(c["off"][hi])
        h_col = pin(c["col"][e0_:e1_])
        h_w = pin(c["w"][e0_:e1_]) if c["w"] is not None else None
    else:
        h_col = pin(c["col"])
        h_w = pin(c["w"]) if c["w"] is not None else None
    digest = graph_digest(c["off"], c["col"]) if mode != "rows" else None
    h_out = torch.empty(max(n, 1), dtype=torch.int32).pin_memory().numpy()
    e2e_ms = 0.0
    e2e_steps = max(1, min(args.steps, 5))
    e2e_step_ms = []
    for i in range(e2e_steps + 1):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if mode == "rows":
            gh = P.Graph.from_csr_rows(n, h_off, lo, hi, h_col, h_w, ctx=ctx)
        else:
            gh = P.Graph.from_csr(n, h_off, h_col, h_w, ctx=ctx)
        run_device(P, gh, wl["algo"], h_out, report=False)
        e1.record(stream)
        e1.synchronize()
        if i > 0:  # first iteration is a warm-up
            e2e_step_ms.append(e0.elapsed_time(e1))
            e2e_ms += e2e_step_ms[-1]
        del gh
    e2e_ms /= e2e_steps
    print("e2e steps (ms):", " ".join(f"{t:.2f}" for t in e2e_step_ms), file=sys.stderr)
    h2d = h_off.nbytes + h_col.nbytes + (h_w.nbytes if h_w is not None else 0)
    if dist:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = {"value": units * m / (e2e_ms / 1e3), "unit": "edges/s", "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(4 * n), "ms_per_step": e2e_ms,
           "steps_ms": [round(t, 3) for t in e2e_step_ms],
           "path": "pinned host CSR -> cd_graph_from_csr" + ("_rows (own rows)" if mode == "rows" else "")
                   + " -> detector -> host labels"}

    # ---- the reference on the same bytes: cached parity setting + live baseline ----
    cached = cached_reference_quality(args.workload, digest)
    if cached:
        quality["reference_cached"] = cached
        for setting, v in cached.items():
            quality[f"abs_diff_{setting}"] = abs(quality["modularity"] - v["modularity"])
    cpu = None
    if wl.get("cpu") is False:
        cpu = {"value": None, "unit": "edges/s", "cores": cpu_threads(), "kind": "reference",
               "sample": "skipped: " + NO_CPU_REASON}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import oracle as O
            if O.ref_available():
                if cached:
                    # these bytes' digest equals the one the C port of the
                    # generator produced for the cached reference runs
                    og = O.from_csr(n, c["off"], c["col"], None if c["w"] is None else c["w"].astype(np.float64))
                else:
                    og = make_oracle_graph(O, wl)
                assert og.m == m and graph_digest(og.off, og.col) == digest, "oracle graph differs from device graph"
                rg = O.RefGraph.from_csr(og)
                del og
                threads = cpu_threads()
                ts, qs = [], []
                t0 = time.time()
                while len(ts) < 3 and (not ts or time.time() - t0 < args.cpu_sample_s):
                    r = run_reference(O, rg, wl["algo"], threads)
                    ts.append(r["total_ms"] / 1e3)
                    qs.append(r["modularity"])
                cpu = {"value": m / statistics.median(ts), "unit": "edges/s", "cores": threads, "kind": "reference",
                       "sample": f"{len(ts)} complete reference {wl['algo']} runs (oracle/_ref, OMP workers="
                                 f"{threads}, default order) on the identical graph, median total_ms"}
                quality["ref_modularity"] = statistics.median(qs)
                quality["abs_diff"] = abs(quality["modularity"] - quality["ref_modularity"])
        except Exception as exc:  # the baseline is reported, never the target
            cpu = {"value": None, "unit": "edges/s", "cores": cpu_threads(), "kind": "reference",
                   "sample": f"failed: {exc}"}

    del c
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "steps_ms": [round(t, 3) for t in step_ms], "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "int32+f64",
            "data": "synthetic",
            "config": workload_config(args, wl, n, m, entries),
            "parallelism": f"{mode} x{world}" if mode != "1gpu" else "1gpu",
            "l2": "flushed (256 MiB write) before every timed step",
            "quality": quality,
            "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu, "clocks": clk,
        }
        emit(line)
    if dist:
        dist.destroy_process_group()
    return 0


_OUT = None  # the JSON line's stream (the original stdout)


def emit(line):
    print(json.dumps(line), file=_OUT or sys.stdout, flush=True)


def spawn_ranks(n):
    """--gpus N outside torchrun: re-launch this command with N ranks (one per
    GPU) under torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) on stderr
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env, stdout=_OUT, stderr=sys.stderr)


def main():
    global _OUT
    # Libraries (NCCL's version banner, ...) may write to fd 1; keep stdout
    # for the one JSON line and send everything else to stderr.
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse()
    wl = WORKLOADS[args.workload]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    if args.impl == "reference":
        return bench_reference(args, wl)
    return bench_b200(args, wl)


if __name__ == "__main__":
    sys.exit(main())
