"""bench.py -- adaptive k-NN (arXiv 1902.09465) hot path on B200: queries/s and
sampled coordinate evaluations/s, with the dominant kernel against its roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--alpha theory]
    python bench.py --impl reference ...        # the CPU oracle, timed the same way

One step = one call of aknn_query (the whole batched round loop, SURVEY.md §8(a)
rows a2-a9) over the config's query batch, inputs resident in HBM.  At N=1 the
workload is the largest single-GPU config, BASELINE.json configs[2] (C3,
Tiny-ImageNet-shaped: n=100,000, d=12,288, q=256, k=h=10, delta=0.05; X = 1.23 GB,
larger than L2); --config 2 / 4 select the other single-GPU configs.  With N>1
(one process per GPU; `--gpus N` re-executes itself under torchrun when needed) the
default is configs[4] (C5): the point set is sharded 1,000,000 rows per GPU and every
rank runs the same 1,024-query batch with one ncclAllGather of the round summaries
per round ("scaling": "weak": the point set grows with N).

Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events on
the stream the library launches on; L2 (126 MB) is flushed by a 512 MiB write
before every step (outside the events), the whole timed region is bracketed by
a barrier and torch.cuda.synchronize(), and the time is the max over ranks.

The oracle (oracle/) is used only by the cpu_baseline leg and --impl reference.
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
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402  (input generator only; no method arithmetic)

METRIC = "adaptive k-NN queries/s (+ sampled coord-evals/s; % of HBM roofline)"
UNIT = "queries/s"
L2_FLUSH_BYTES = 512 << 20
SHARD_ROWS = 1_000_000  # C5: points per GPU (BASELINE.json configs[4])


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=None,
                    help="BASELINE.json config (1-based; default 2, or 1 with --schedule a1)")
    ap.add_argument("--schedule", choices=("br", "a1"), default="br",
                    help="batched round rule (default) or the literal Algorithm 1 "
                         "(SURVEY §8(f) row 2, aknn_query_a1)")
    ap.add_argument("--alpha", default="theory",
                    help="'theory' (footnote 2, P:132-138) or 'exp:<C_alpha>' (§5, P:349)")
    ap.add_argument("--q", type=int, default=0, help="override queries per rank (0 = config)")
    ap.add_argument("--draws", choices=("per-query", "shared"), default="per-query",
                    help="per-query Philox streams (default, DESIGN.md R19) or query-independent "
                         "draws (SURVEY §8(f1), AKNN_FLAG_SHARED_DRAWS)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-variant", action="store_true", help="skip the shared-draw variant timing")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exact", action="store_true")
    ap.add_argument("--workload", choices=("config", "sec5"), default="config",
                    help="sec5: the paper's §5 sweep (recall / fraction vs C_alpha, sec5.py)")
    ap.add_argument("--trials", type=int, default=20, help="sec5: trials per (workload, C_alpha)")
    ap.add_argument("--c-alpha", default="1e-5,1e-4,1e-3,1e-2", help="sec5: C_alpha values")
    ap.add_argument("--sec5-schedules", default="a1,br,br_lead3,br_g2",
                    help="sec5: a1, br, br_lead<L> (close-side lead L), br_g2[_lead<L>] (growth < 2), br_wor")
    ap.add_argument("--sec5-workloads", default="p10,p100,p1000,images")
    ap.add_argument("--sec5-threads", type=int, default=80, help="sec5: trials in flight")
    ap.add_argument("--sec5-a1-max-iters", type=int, default=0,
                    help="sec5: cap on Algorithm-1 iterations per query (0: none; capped trials are counted)")
    ap.add_argument("--lead", type=int, default=1,
                    help="close-side lead L of the batched rule (aknn_opts.lead, DESIGN.md §16)")
    ap.add_argument("--clock-sampler", choices=("nvml", "smi", "none"), default="nvml")
    a = ap.parse_args()
    if a.config is None:
        # N = 1: the largest single-GPU config (C3, 1.23 GB of X, not L2-resident);
        # N > 1: the point-sharded C5 (1M rows per GPU, one allgather per round)
        a.config = 1 if a.schedule == "a1" else (5 if a.gpus > 1 else 3)
    return a


def _relaunch_under_torchrun(args) -> None:
    """`python bench.py --gpus N` (N > 1) outside torchrun re-executes itself as N ranks
    (one process per GPU) so that N always means N processes; under torchrun the world
    size must equal --gpus."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        port = os.environ.get("MASTER_PORT", "29533")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
               os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    if ws is not None and int(ws) != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={ws} but --gpus {args.gpus}")


def _alpha_desc(a: str) -> str:
    return "footnote-2 theory table (P:132-138)" if a == "theory" else \
        f"section-5 experimental table, C_alpha={a.split(':', 1)[1]} (P:349)"


# ----------------------------------------------------------------------------- dist
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, v: float) -> float:
        if not self.pg:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: float) -> float:
        if not self.pg:
            return v
        import torch
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock, max clock, power and throttle reasons sampled during the timed region.

    mode "nvml" (default): in-process NVML queries every 200 ms from a thread (the
    same counters the nvidia-smi recipe line reads); mode "smi": an nvidia-smi
    -lms 200 subprocess (the recipe line itself); "none": no sampling."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu: int, mode: str = "nvml", period_s: float = 0.2):
        self.gpu, self.mode, self.period = gpu, mode, period_s
        self.proc = None
        self.samples = []  # (sm, smax, power_w, set(reasons))
        self.t = None
        self.stop_evt = threading.Event()

    def start(self):
        if self.mode == "none":
            return
        if self.mode == "smi":
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits", "-lms", str(int(self.period * 1000))],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except Exception:
                self.proc = None
                return
            self.t = threading.Thread(target=self._read_smi, daemon=True)
        else:
            try:
                import pynvml
                pynvml.nvmlInit()
                self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
                self.nv = pynvml
            except Exception:
                self.mode = "none"
                return
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
        self.t.start()

    def _read_smi(self):
        for ln in self.proc.stdout:
            f = [x.strip() for x in ln.strip().split(",")]
            if len(f) < 9:
                continue
            try:
                rs = {nm for nm, v in zip(self.NAMES, f[5:9]) if v.lower().startswith("active")}
                self.samples.append((float(f[1]), float(f[2]), float(f[3]), rs))
            except ValueError:
                continue

    def _poll_nvml(self):
        nv, h = self.nv, self.h
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        while not self.stop_evt.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(smax), pw,
                                     {k for k, b in bits.items() if r & b}))
            except Exception:
                pass
            self.stop_evt.wait(self.period)

    def stop(self) -> dict:
        if self.mode == "none":
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "source": "not sampled"}
        self.stop_evt.set()
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm = [s[0] for s in self.samples]
        reasons = set().union(*[s[3] for s in self.samples]) if self.samples else set()
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(s[1] for s in self.samples) if sm else None,
                "power_w_max": max(s[2] for s in self.samples) if sm else None,
                "samples": len(sm), "reasons": sorted(reasons),
                "source": "NVML every 200 ms" if self.mode == "nvml" else "nvidia-smi -lms 200"}


# ----------------------------------------------------------------------------- peaks
def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy, read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def _bf16_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["bf16_tflops"]), "measured (MEASURED_PEAKS.json bf16_tflops, cuBLAS 8192^3)"
    except Exception:
        return 2250.0, "fallback (nominal 2.25 PFLOP/s bf16 dense)"


def _traffic_from_profiles(kernel: str, workload: str):
    """(dram bytes per launch, source) of `kernel` on `workload` from the committed ncu
    summary profiles/ncu_traffic.json (keys "<workload>/<kernel>"), if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            j = json.load(f)
        v = j.get(f"{workload}/{kernel}")
        return (None, None) if v is None else (v.get("dram_bytes_per_launch"), v.get("source"))
    except Exception:
        return None, None


# Algorithmic bytes per unit of each kernel class:
#   init     per pair: one 32-B sector of X (the one used byte) + S(4) + level(1) + action(1)
#   select   per evaluated query: n x (S 4 B + level 1 B), one read of the arm state
#   filter   per blocked query: n x (S 4 + level 1) read + n action bytes written
#   compact  per blocked query: n action bytes read + 4 B per listed pair written
#   advance  per sampled draw: one 32-B sector of X; per exact fallback: d bytes of X;
#            per advanced pair: list entry 4 + S read 4 + S write 4 + level 1
SECTOR = 32
L2_BYTES = 126 << 20


def _measure_probes(d: int, x_bytes: int) -> dict:
    """Roofline denominators measured on this GPU now (tools/probes.cu)."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import run_probes as rp
        L = rp.load()
        pb = rp.philox_blocks_per_s(L, d=d)
        gl, fb = rp.gather_sectors_per_s(L, x_bytes)
        sd = rp.shared_draws_per_s(L)
        return {"philox_blocks_per_s": pb, "gather_loads_per_s": gl, "gather_footprint_bytes": fb,
                "shared_draws_per_s": sd}
    except Exception as e:  # the probes are evidence, never a reason to fail the bench
        return {"error": repr(e)}


def _algorithmic_bytes(st: dict, n: int, d: int, q: int) -> dict:
    init_draws = q * n
    return {
        "init": init_draws * (SECTOR + 6),
        "select": st["query_rounds"] * n * 5,
        "filter": st["blocked_query_rounds"] * n * 6,
        "compact": st["blocked_query_rounds"] * n + st["active_pair_rounds"] * 4,
        # list path + exact fallbacks: sampled draws outside the tiles at one sector each
        "advance": max(0, st["draws"] - init_draws - st["tile_draws"]) * SECTOR + st["exact_fallbacks"] * d,
        # tiles stage rows (R + P) * pitch per dense tile: ALU-bound, no byte model here
        "tiles": 0,
    }


KERNEL_OF = {"init": "k_init", "select": "k_select_pivot", "filter": "k_filter",
             "compact": "k_scatter", "advance": "k_advance", "tiles": "k_advance_tiles",
             "output": "k_output"}
KERNEL_OF_SHARED = dict(KERNEL_OF, tiles="k_level_mma")


# ----------------------------------------------------------------------------- oracle legs
_ORC = {}


def _orc_worker(i):
    import oracle.oracle as orc
    X, Q, cfg, al = _ORC["X"], _ORC["Q"], _ORC["cfg"], _ORC["alpha"]
    r = orc.query_br(X, Q[i:i + 1], cfg.k, cfg.h, cfg.seed, al,
                     qids=np.array([i], np.int32), want_counts=False,
                     shared_draws=_ORC.get("shared", False), lead=_ORC.get("lead", 1))
    return int(r["evals"][0])


def _oracle_time(X, Q, cfg, alpha, nq: int, cores: int, shared: bool = False, lead: int = 1):
    """Wall time of the oracle (as it stands, single-threaded C) on nq queries spread
    over `cores` worker processes (one query per task)."""
    import multiprocessing as mp
    import oracle.oracle as orc
    orc.lib()  # build/load before forking
    _ORC.update(X=X, Q=Q, cfg=cfg, alpha=alpha, shared=shared, lead=lead)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        evals = pool.map(_orc_worker, range(nq), chunksize=1)
    return time.perf_counter() - t0, sum(evals)


def _oracle_alpha(cfg, alpha_arg):
    import oracle.oracle as orc
    if alpha_arg == "theory":
        return orc.alpha_theory(cfg.n, cfg.delta, cfg.d)
    return orc.alpha_experimental(cfg.n, cfg.delta, cfg.d, float(alpha_arg.split(":", 1)[1]))


def _cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, dist: Dist):
    """--impl reference: the CPU oracle timed on the box's host cores (rank 0 only)."""
    if dist.rank != 0:
        return
    cfg = synth.config(args.config)
    if args.q:
        cfg = synth.config(args.config, q=args.q)
    Q = synth.queries(cfg)
    if cfg.shards > 1:  # C5: the same N * SHARD_ROWS points as our arm
        X = synth.points(cfg, 0, SHARD_ROWS * args.gpus)
        cfg = synth.config(args.config, q=cfg.q, n=SHARD_ROWS * args.gpus)
    else:
        X = synth.points(cfg)
    al = _oracle_alpha(cfg, args.alpha)
    cores = max(1, min(_cpu_cores(), 16))
    nq = min(cores, cfg.q)  # one query per core per step
    times = []
    # CPU timing needs no GPU-style warm-up beyond one step (page-in, fork); the run is
    # capped at ~4 min of oracle work (at least one timed step): a C3/C5 oracle query
    # takes 10-100+ s, and the run must end within minutes
    warm = min(args.warmup, 1)
    t_start = time.perf_counter()
    for it in range(warm + args.steps):
        off = (it * nq) % max(1, cfg.q - nq + 1)
        dt, _ = _oracle_time(X, Q[off:off + nq], cfg, al, nq, cores, args.draws == "shared", args.lead)
        if it >= warm:
            times.append(dt)
            if time.perf_counter() - t_start > 240.0:
                break
    ms = 1e3 * sum(times) / len(times)
    value = nq / (ms / 1e3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "config": _config_desc(cfg, args, extra={"sample_queries_per_step": nq}),
        "steps_timed": len(times), "warmup_steps_run": warm,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{nq} queries of {cfg.name} per step (full n={cfg.n}), "
                                   f"one single-threaded oracle process per core"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_desc(cfg, args, extra=None):
    d = {"workload": cfg.name + ("_shared_draws" if getattr(args, "draws", "per-query") == "shared" else ""),
         "n": cfg.n, "d": cfg.d, "q_per_rank": cfg.q, "k": cfg.k,
         "h": cfg.h, "delta": cfg.delta, "seed": cfg.seed, "alpha": _alpha_desc(args.alpha),
         "lead": getattr(args, "lead", 1),
         "parallelism": f"query-parallel x{args.gpus} (X replicated)" if args.gpus > 1 else "1 GPU",
         "l2": "flushed before every step (512 MiB write, outside the timed events)"}
    if extra:
        d.update(extra)
    return d


# ----------------------------------------------------------------------------- ours
def run_ours(args, dist: Dist):
    import torch
    import paper_1902_09465_b200 as ak

    torch.cuda.set_device(dist.local)
    dev = torch.device("cuda", dist.local)
    base = synth.config(args.config)
    qpr = args.q or base.q
    sharded = base.shards > 1  # C5: point-sharded, SHARD_ROWS per GPU (weak scaling)
    if sharded:
        # rank r holds rows [r * SHARD_ROWS, (r+1) * SHARD_ROWS) of the C5 point set; the
        # job answers ONE batch of q queries against all N * SHARD_ROWS points, with one
        # ncclAllGather of the round summaries per round
        n_global = SHARD_ROWS * dist.world
        row0 = SHARD_ROWS * dist.rank
        cfg = synth.config(args.config, q=qpr, n=n_global)
        Qh = synth.queries(synth.config(args.config, q=qpr))
        X = synth.points(base, row0, row0 + SHARD_ROWS)
    else:
        cfg = synth.config(args.config, q=qpr)
        # every rank: the same X, its own slice of a (world * q)-query batch of the mixture
        allq = synth.queries(synth.config(args.config, q=qpr * dist.world)) if dist.world > 1 \
            else synth.queries(cfg)
        Qh = np.ascontiguousarray(allq[dist.rank * qpr:(dist.rank + 1) * qpr])
        X = synth.points(cfg)
    n, d, k, h = cfg.n, cfg.d, cfg.k, cfg.h
    n_loc = X.shape[0]  # points on this GPU
    if args.alpha == "theory":
        alpha = ak.alpha_table(n, cfg.delta, d, "theory")
    else:
        alpha = ak.alpha_table(n, cfg.delta, d, "experimental", float(args.alpha.split(":", 1)[1]))
    if sharded and dist.world > 1:
        nid = [ak.nccl_unique_id() if dist.rank == 0 else None]
        dist.pg.broadcast_object_list(nid, src=0)
        ix = ak.Index(X, n_global=n_global, offset=row0, nccl_id=nid[0], rank=dist.rank, world=dist.world)
        args.no_exact = True  # the exact pass is per shard: no global recall here
    else:
        ix = ak.Index(torch.from_numpy(X).to(dev))
    Qd = torch.from_numpy(Qh).to(dev)
    alpha_d = torch.from_numpy(alpha).to(dev)
    stream = torch.cuda.Stream(device=dev)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    kh = k + h
    out = dict(sets=torch.empty((qpr, kh), dtype=torch.int32, device=dev),
               dhat=torch.empty((qpr, kh), dtype=torch.float64, device=dev), counts=None,
               sums=None, evals=torch.empty(qpr, dtype=torch.int64, device=dev),
               draws=torch.empty(qpr, dtype=torch.int64, device=dev),
               rounds=torch.empty(qpr, dtype=torch.int32, device=dev))
    qi_off = 0 if sharded else dist.rank * qpr
    qflags = ak.FLAG_SHARED_DRAWS if args.draws == "shared" else 0

    def step(timing: bool, flags=None):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ix.query_device(Qd, k, h, cfg.delta, cfg.seed, alpha_d, qi_offset=qi_off, timing=timing,
                        stream=stream, out=out, flags=qflags if flags is None else flags, lead=args.lead)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), ix.stats()

    def timed(timing: bool, flags=None):
        """W warm-up steps, then K steps bracketed by barrier + synchronize; per-step CUDA
        events on the library's stream (L2 flushed before each step, outside the events)."""
        for _ in range(args.warmup):
            step(timing, flags)
        clocks = ClockSampler(dist.local, args.clock_sampler)
        dist.barrier()
        torch.cuda.synchronize()
        clocks.start()
        times, stats = [], []
        for _ in range(args.steps):
            ms, st = step(timing, flags)
            times.append(ms)
            stats.append(st)
        dist.barrier()
        torch.cuda.synchronize()
        return times, stats, clocks.stop()

    # (1) the product path: device-driven round loop (one CUDA graph launch per batch)
    times, gstats, clk = timed(False)
    ms_local = sum(times)
    ms_max = dist.max(ms_local)
    total_q = qpr * args.steps if sharded else dist.sum(qpr * args.steps)
    value = total_q / (ms_max / 1e3)
    ms_per_step = ms_max / args.steps
    # (1b) the query-independent-draw variant on the same workload:
    # reported beside the headline, which keeps the per-query streams (R19)
    variant = None
    variants = {}
    if args.draws == "per-query" and not args.no_variant:
        for vname, vflag, vdesc in (
                ("shared_draws", ak.FLAG_SHARED_DRAWS, "query-independent draws (AKNN_FLAG_SHARED_DRAWS, DESIGN.md §12)"),
                ("without_replacement", ak.FLAG_WITHOUT_REPLACEMENT,
                 "per-query draws without replacement (AKNN_FLAG_WITHOUT_REPLACEMENT, DESIGN.md §15)")):
            vtimes, _, vclk = timed(False, vflag)
            vms = dist.max(sum(vtimes))
            vev = int(out["evals"].sum().item())  # sharded: already summed over the shards
            frac = vev / (qpr * cfg.n * d) if sharded else dist.sum(vev) / (dist.world * qpr * n_loc * d)
            variants[vname] = {"what": vdesc, "value": total_q / (vms / 1e3), "unit": UNIT,
                               "ms_per_step": vms / args.steps, "step_ms": [round(t, 3) for t in vtimes],
                               "sample_fraction": frac, "clocks": vclk}
        variant = dict(variants["shared_draws"], draws="shared (AKNN_FLAG_SHARED_DRAWS, DESIGN.md §12)")
    # (2) the same steps with per-launch CUDA events (host-driven loop) for the roofline
    itimes, stats, _ = timed(True)
    ms_local_instr = sum(itimes)

    # per-class device time and algorithmic bytes over the timed region (this rank)
    agg = {key: sum(s[key] for s in stats) for key in stats[0]}
    draws = agg["draws"]
    evals_total = int(out["evals"].sum().item()) * args.steps
    classes = ["init", "select", "filter", "compact", "advance", "tiles", "output"]
    ms_cls = {c: agg[f"ms_{c}"] for c in classes}
    launches = {c: agg[f"launches_{c}"] for c in classes}
    abytes = {c: 0 for c in classes}
    for s in stats:
        for c, b in _algorithmic_bytes(s, n_loc, d, qpr).items():
            abytes[c] += b
    dom = max(classes, key=lambda c: ms_cls[c])
    peak, peak_src = _peaks()
    probes = _measure_probes(d, n_loc * cfg.d)
    blocks = agg.get("philox_blocks", 0)
    # list-path level-gather draws: all sampled draws minus initialisation minus the tiles'
    adv_draws = max(0, agg["draws"] - args.steps * qpr * n_loc - agg.get("tile_draws", 0))
    x_in_l2 = n_loc * d <= L2_BYTES * 0.8
    kof = KERNEL_OF_SHARED if (args.draws == "shared" and agg.get("level_mma_tiles", 0) > 0) else KERNEL_OF
    if d > 8192 and kof is KERNEL_OF:  # rows wider than 8 KB: the grouped tile kernel
        kof = dict(KERNEL_OF, tiles="k_advance_tiles_grp")
    common = {"kernel": kof[dom], "launches": launches[dom],
              "avg_launch_ms": ms_cls[dom] / max(1, launches[dom]),
              "share_of_step": ms_cls[dom] / ms_local_instr,
              "timing": "CUDA events around every launch on the library stream, K instrumented "
                        "steps (host-driven loop) right after the K graph-launched timed steps",
              "ms_per_step_instrumented": dist.max(ms_local_instr) / args.steps,
              "traffic": _traffic_from_profiles(kof[dom], cfg.name)[0],
              "per_class": {c: {"ms": ms_cls[c], "launches": launches[c],
                                "GBps_algorithmic": (abytes[c] / (ms_cls[c] / 1e3) / 1e9)
                                if c in abytes and ms_cls[c] > 0 else None}
                            for c in classes},
              "probes": probes}
    adv_s = ms_cls["advance"] / 1e3
    sector_view = {
        "draws_per_s": adv_draws / adv_s if adv_s > 0 else None,
        "sector_GBps": adv_draws * SECTOR / adv_s / 1e9 if adv_s > 0 else None,
        "frac_of_measured_random_sector_rate": (adv_draws / adv_s) / probes["gather_loads_per_s"]
        if adv_s > 0 and probes.get("gather_loads_per_s") else None,
        "x_footprint_bytes": n_loc * d, "x_l2_resident": x_in_l2}
    tile_blocks = agg.get("tile_blocks", 0)
    lm_tiles = agg.get("level_mma_tiles", 0)
    if dom == "tiles" and args.draws == "shared" and lm_tiles > 0:
        # shared draws, dominant level as 4 integer GEMMs (u8 x u8 -> s32) per 128 x 128
        # (query x point) tile over K = d: tensor-bound; int8 dense peak = 2 x the measured
        # bf16 dense peak (B200 nominal ratio 4.5 / 2.25 PFLOP/s)
        ts = ms_cls["tiles"] / 1e3
        ops = lm_tiles * 128 * 128 * d * 2 * 4
        pk_bf16, pk_src = _bf16_peak()
        roofline = {"bound": "tensor", "achieved": ops / ts / 1e12, "peak": 2 * pk_bf16,
                    "unit": "TOP/s (int8)", "frac": ops / ts / 1e12 / (2 * pk_bf16),
                    "peak_source": pk_src + " x 2 (int8 : bf16 dense, B200_PROFILING.md nominal)",
                    "algorithmic_units_per_launch": ops / max(1, launches[dom]),
                    "level_mma_tiles": lm_tiles, "sector_view": sector_view, **common}
    elif dom == "tiles" and args.draws == "shared" and probes.get("shared_draws_per_s"):
        # shared draws: Philox runs once per point column; the tile gathers are bound by
        # the byte gathers + multiply-adds of the (query, point) draws: measured ceiling of
        # that instruction mix in tools/probes.cu k_probe_shared
        ts = ms_cls["tiles"] / 1e3
        ach = agg.get("tile_draws", 0) / ts / 1e9
        pk = probes["shared_draws_per_s"] / 1e9
        roofline = {"bound": "alu", "achieved": ach, "peak": pk, "unit": "G pair-draws/s",
                    "frac": ach / pk,
                    "peak_source": "measured in this run: tools/probes.cu k_probe_shared (the "
                                   "shared-draw gather loop alone, full occupancy)",
                    "algorithmic_units_per_launch": agg.get("tile_draws", 0) / max(1, launches[dom]),
                    "sector_view": sector_view, **common}
    elif dom == "tiles" and probes.get("philox_blocks_per_s"):
        # dense tiles gather from shared memory: the sampled draws are bound by the
        # integer pipes running Philox4x32-10 (ncu: fma-heavy + LDS wavefronts), not by
        # memory
        ts = ms_cls["tiles"] / 1e3
        ach = tile_blocks / ts / 1e9
        pk = probes["philox_blocks_per_s"] / 1e9
        roofline = {"bound": "alu", "achieved": ach, "peak": pk, "unit": "G Philox blocks/s",
                    "frac": ach / pk,
                    "peak_source": "measured in this run: tools/probes.cu k_probe_philox "
                                   "(Philox4x32-10 + multiply-high map, no memory)",
                    "algorithmic_units_per_launch": tile_blocks / max(1, launches[dom]),
                    "sector_view": sector_view, **common}
    elif dom == "advance" and x_in_l2 and probes.get("philox_blocks_per_s"):
        # X fits the 126 MB L2: the list-path levels are bound by the integer pipe
        ach = (blocks - tile_blocks) / adv_s / 1e9
        pk = probes["philox_blocks_per_s"] / 1e9
        roofline = {"bound": "alu", "achieved": ach, "peak": pk, "unit": "G Philox blocks/s",
                    "frac": ach / pk,
                    "peak_source": "measured in this run: tools/probes.cu k_probe_philox "
                                   "(Philox4x32-10 + multiply-high map, no memory)",
                    "algorithmic_units_per_launch": (blocks - tile_blocks) / max(1, launches[dom]),
                    "sector_view": sector_view, **common}
    else:
        achieved = abytes.get(dom, 0) / (ms_cls[dom] / 1e3) / 1e9 if ms_cls[dom] > 0 else 0.0
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": abytes[dom] / max(1, launches[dom]),
                    "sector_view": sector_view, **common}

    # the same kernel against the HBM roofline (BASELINE.json metric: "% of HBM roofline"):
    # the DRAM bytes it moves per launch (ncu dram__bytes_read + write, committed summary
    # of this workload) over its live average launch time
    tb, tsrc = _traffic_from_profiles(kof[dom], cfg.name)
    avg_s = ms_cls[dom] / max(1, launches[dom]) / 1e3
    roofline["hbm_view"] = {
        "dram_bytes_per_launch": tb, "GBps": tb / avg_s / 1e9 if tb and avg_s > 0 else None,
        "peak": peak, "unit": "GB/s", "frac": tb / avg_s / 1e9 / peak if tb and avg_s > 0 else None,
        "peak_source": peak_src, "bytes_source": tsrc or "no committed ncu capture of this kernel on this workload"}

    extra = {
        "draws_per_s": dist.sum(draws) / (ms_max / 1e3),
        # sharded: the library already sums evals over the ranks (ncclAllReduce)
        "evals_per_s": (evals_total if sharded else dist.sum(evals_total)) / (ms_max / 1e3),
        "sample_fraction": evals_total / (args.steps * qpr * n * d),
        "rounds_max": int(out["rounds"].max().item()),
        "exact_fallbacks_per_query": agg["exact_fallbacks"] / (args.steps * qpr),
        # G2 (k_init): one random 32-byte sector of X + 6 B of state per pair, served from
        # L2 when X fits it (then the rate can exceed the HBM peak) else from HBM
        "init_sector_GBps": (qpr * n_loc * (SECTOR + 6)) / (ms_cls["init"] / args.steps / 1e3) / 1e9
        if ms_cls["init"] > 0 else None,
        "init_sector_source": "L2 (X fits the 126 MB L2)" if x_in_l2 else "HBM",
    }

    # exact comparison pass on the same queries: time + recall of the adaptive sets
    if not args.no_exact:
        ex_idx = torch.empty((qpr, k), dtype=torch.int32, device=dev)
        ex_d = torch.empty((qpr, k), dtype=torch.int32, device=dev)
        ets = []
        for it in range(2 + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ix.exact_device(Qd, k, stream=stream, out=(ex_idx, ex_d))
            e1.record(stream)
            torch.cuda.synchronize()
            if it >= 2:
                ets.append(e0.elapsed_time(e1))
        ex_ms = dist.max(sum(ets) / len(ets))
        sets = out["sets"].cpu().numpy()
        exi = ex_idx.cpu().numpy()
        exd = ex_d.cpu().numpy()
        ok = 0
        for a in range(qpr):
            # tie-aware containment (reading R16): every strictly-closer point, and
            # enough of the points tied at the k-th distance
            kth = exd[a, -1]
            strict = set(exi[a][exd[a] < kth].tolist())
            s = set(sets[a].tolist())
            ok += strict <= s
        extra.update({"exact_pass_ms": ex_ms, "speedup_vs_exact": ex_ms / ms_per_step,
                      "recall_contains_knn": dist.sum(ok) / (qpr * dist.world),
                      "exact_pass_kernel": "k_exact_fused (persistent tcgen05 kind::i8, running top-k epilogue) + k_exact_merge" if k <= 128 else "tcgen05 kind::i8 tiles (k_mma_tiles) + block top-k",
                      # 2 q n d int8 ops (u8 x u8 -> s32 MACs) over the whole pass incl. top-k
                      "exact_pass_tops": 2.0 * qpr * n_loc * d / (ex_ms / 1e3) / 1e12,
                      "exact_pass_x_GBps": n_loc * d / (ex_ms / 1e3) / 1e9})

    # end to end through the host API (pinned host buffers, H2D + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        Qpin = torch.from_numpy(Qh).pin_memory()
        hout = dict(sets=torch.empty((qpr, kh), dtype=torch.int32).pin_memory().numpy(),
                    dhat=torch.empty((qpr, kh), dtype=torch.float64).pin_memory().numpy(),
                    counts=None, sums=None,
                    evals=torch.empty(qpr, dtype=torch.int64).pin_memory().numpy(),
                    draws=torch.empty(qpr, dtype=torch.int64).pin_memory().numpy(),
                    rounds=torch.empty(qpr, dtype=torch.int32).pin_memory().numpy())
        Qpin_np = Qpin.numpy()
        for _ in range(1):
            ix.query(Qpin_np, k, h, cfg.delta, cfg.seed, alpha, qi_offset=qi_off, out=hout, flags=qflags,
                     lead=args.lead)
        dist.barrier()
        wall = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ix.query(Qpin_np, k, h, cfg.delta, cfg.seed, alpha, qi_offset=qi_off, out=hout, flags=qflags,
                     lead=args.lead)
            wall.append(time.perf_counter() - t0)
        e2e_s = dist.max(sum(wall))
        h2d = Qh.nbytes + alpha.nbytes
        d2h = sum(v.nbytes for key, v in hout.items() if key != "status" and v is not None)
        e2e = {"value": (qpr * args.steps if sharded else dist.sum(qpr * args.steps)) / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": "aknn_query (host pointers, pinned), wall clock incl. copies"}
        if not np.array_equal(hout["sets"], out["sets"].cpu().numpy()):
            raise RuntimeError("host API and device API disagree on the candidate sets")

    cpu = None
    if not args.no_cpu_baseline and dist.rank == 0 and dist.world == 1:
        # a bounded sample of the same workload: ~10-30 s of oracle work on the host cores
        cores = max(1, min(_cpu_cores(), 16))
        nq = min(qpr, 8 * cores if n * d <= 100_000_000 else cores)
        dt, _ = _oracle_time(X, Qh, cfg, _oracle_alpha(cfg, args.alpha), nq, cores, args.draws == "shared",
                             args.lead)
        cpu = {"value": nq / dt, "unit": UNIT, "cores": min(cores, nq), "kind": "oracle",
               "sample": f"first {nq} queries of {cfg.name} (full n={n}, d={d}), one "
                         f"single-threaded oracle process per core, {dt:.1f} s wall"}

    gpu_launches = int(dist.sum(sum(st["kernel_launches"] for st in gstats)))
    ix.close()
    if dist.rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded; synth/ recipes, DESIGN.md §5)",
            "config": _config_desc(cfg, args, extra={
                "parallelism": f"point-sharded x{dist.world}: {SHARD_ROWS:,} rows per GPU, one "
                               f"ncclAllGather of the round summaries per round" if sharded and dist.world > 1
                else ("point set of 1 shard (the N=1 point of the weak-scaling series)" if sharded
                      else _config_desc(cfg, args)["parallelism"])}),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": gpu_launches, "gpu_launches_per_step": gpu_launches / args.steps,
            "step_ms": [round(t, 3) for t in times],
            "variant_shared_draws": variant,
            "variants": variants or None,
            **extra,
        }
        print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- Algorithm 1
def _a1_inputs(args):
    cfg = synth.config(args.config)
    if args.config == 1:
        X, Q, _ = synth.planted(cfg)
    else:
        if args.q:
            cfg = synth.config(args.config, q=args.q)
        X, Q = synth.points(cfg), synth.queries(cfg)
    return cfg, X, Q


def _a1_orc_worker(i):
    import oracle.oracle as orc
    X, Q, cfg, al = _ORC["X"], _ORC["Q"], _ORC["cfg"], _ORC["alpha"]
    return int(orc.query_a1(X, Q[i], cfg.k, cfg.h, cfg.seed, al, qi=i)["evals"])


def _a1_oracle_time(X, Q, cfg, alpha, nq: int, cores: int):
    import multiprocessing as mp
    import oracle.oracle as orc
    orc.lib()
    _ORC.update(X=X, Q=Q, cfg=cfg, alpha=alpha)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(min(cores, nq)) as pool:
        pool.map(_a1_orc_worker, range(nq), chunksize=1)
    return time.perf_counter() - t0


def _a1_desc(cfg, args):
    return {"workload": cfg.name + "_algorithm1", "schedule": "literal Algorithm 1 (P:159-191): "
            "{d1, b2} sampled once per iteration", "n": cfg.n, "d": cfg.d, "q_per_rank": cfg.q,
            "k": cfg.k, "h": cfg.h, "delta": cfg.delta, "seed": cfg.seed,
            "alpha": _alpha_desc(args.alpha), "parallelism": "1 GPU, one warp per query",
            "l2": "inputs smaller than L2; the iteration chain is latency-bound (no flush)"}


def run_reference_a1(args, dist: Dist):
    if dist.rank != 0:
        return
    cfg, X, Q = _a1_inputs(args)
    al = _oracle_alpha(cfg, args.alpha)
    cores = max(1, min(_cpu_cores(), 16))
    nq = min(cores, cfg.q)
    times = []
    for it in range(min(args.warmup, 1) + args.steps):  # each step ~ seconds: one warm-up
        dt = _a1_oracle_time(X, Q, cfg, al, nq, cores)
        if it >= min(args.warmup, 1):
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    value = nq / (ms / 1e3)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": _a1_desc(cfg, args),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(cores, nq), "kind": "oracle",
                         "sample": f"{nq} queries of {cfg.name} per step, oracle A1 mode "
                                   f"(one full sort per iteration), one process per query"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
        flush=True)


def run_a1(args, dist: Dist):
    """--schedule a1: the literal Algorithm 1 (aknn_query_a1_device) on the config's
    queries; one step = one call over all of them, inputs resident in HBM."""
    import torch
    import paper_1902_09465_b200 as ak

    torch.cuda.set_device(dist.local)
    dev = torch.device("cuda", dist.local)
    cfg, X, Qh = _a1_inputs(args)
    n, d, k, h, q = cfg.n, cfg.d, cfg.k, cfg.h, Qh.shape[0]
    alpha = ak.alpha_table(n, cfg.delta, d, "theory") if args.alpha == "theory" else \
        ak.alpha_table(n, cfg.delta, d, "experimental", float(args.alpha.split(":", 1)[1]))
    ix = ak.Index(torch.from_numpy(X).to(dev))
    Qd = torch.from_numpy(Qh).to(dev)
    alpha_d = torch.from_numpy(alpha).to(dev)
    stream = torch.cuda.Stream(device=dev)
    kh = k + h
    out = dict(sets=torch.empty((q, kh), dtype=torch.int32, device=dev),
               dhat=torch.empty((q, kh), dtype=torch.float64, device=dev), counts=None, sums=None,
               evals=torch.empty(q, dtype=torch.int64, device=dev),
               draws=torch.empty(q, dtype=torch.int64, device=dev),
               rounds=torch.empty(q, dtype=torch.int32, device=dev))

    def step():
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ix.query_device(Qd, k, h, cfg.delta, cfg.seed, alpha_d, stream=stream, out=out, schedule="a1")
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), ix.stats()

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(dist.local, args.clock_sampler)
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    times, stats = [], []
    for _ in range(args.steps):
        ms, st = step()
        times.append(ms)
        stats.append(st)
    dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_max = dist.max(sum(times))
    value = dist.sum(q * args.steps) / (ms_max / 1e3)
    draws = int(out["draws"].sum().item())
    evals = int(out["evals"].sum().item())
    iters = out["rounds"].cpu().numpy()
    probes = _measure_probes(d, n * d)
    s_step = ms_max / args.steps / 1e3
    pk = probes.get("philox_blocks_per_s")
    roofline = {
        "bound": "alu", "achieved": draws / s_step / 1e9, "peak": pk / 1e9 if pk else None,
        "unit": "G Philox blocks/s (one block per Algorithm-1 draw)",
        "frac": (draws / s_step) / pk if pk else None,
        "peak_source": "measured in this run: tools/probes.cu k_probe_philox",
        "kernel": "k_a1", "launches": args.steps, "avg_launch_ms": ms_max / args.steps,
        "share_of_step": 1.0,
        "note": "latency-bound by design: every query is one dependent chain of iterations "
                "(rank split, Eq. 2-5, two draws); the GPU runs one warp per query",
        "us_per_iteration": s_step * 1e6 / float(iters.max()), "traffic": None}
    # the batched rule on the same queries (untimed): sample efficiency of the schedules
    bout = ix.query(Qh, k, h, cfg.delta, cfg.seed, alpha, counts=False)
    e2e = None
    if not args.no_e2e:
        wall = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = ix.query(Qh, k, h, cfg.delta, cfg.seed, alpha, counts=False, schedule="a1")
            wall.append(time.perf_counter() - t0)
        e2e = {"value": q * args.steps / dist.max(sum(wall)), "unit": UNIT,
               "h2d_bytes_per_step": int(Qh.nbytes + alpha.nbytes),
               "d2h_bytes_per_step": int(sum(v.nbytes for key, v in r.items()
                                             if key != "status" and v is not None)),
               "api": "aknn_query_a1 (host pointers), wall clock incl. copies"}
    cpu = None
    if not args.no_cpu_baseline and dist.rank == 0 and dist.world == 1:
        cores = max(1, min(_cpu_cores(), 16))
        nq = min(q, cores)
        dt = _a1_oracle_time(X, Qh, cfg, _oracle_alpha(cfg, args.alpha), nq, cores)
        cpu = {"value": nq / dt, "unit": UNIT, "cores": min(cores, nq), "kind": "oracle",
               "sample": f"first {nq} queries of {cfg.name}, oracle A1 mode, {dt:.1f} s wall"}
    ix.close()
    if dist.rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": dist.world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded; synth/ recipes, DESIGN.md §5)", "config": _a1_desc(cfg, args),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
            "gpu_launches": int(sum(s["kernel_launches"] for s in stats)),
            "step_ms": [round(t, 3) for t in times],
            "iterations": iters.tolist() if q <= 16 else {"mean": float(iters.mean()), "max": int(iters.max())},
            "draws_per_s": draws / s_step, "evals_per_s": evals / s_step,
            "sample_fraction": evals / (q * n * d),
            "batched_rule_same_queries": {"sample_fraction": int(bout["evals"].sum()) / (q * n * d),
                                          "rounds_max": int(bout["rounds"].max())},
        }), flush=True)


def main():
    args = _args()
    _relaunch_under_torchrun(args)
    dist = Dist()
    try:
        if args.workload == "sec5":
            if args.impl == "reference":
                if dist.rank == 0:
                    print(json.dumps({"impl": "reference", "unavailable": "the §5 sweep has no "
                                      "reference arm (bench.py --workload config times the oracle)"}))
            else:
                import sec5
                sec5.run(args, dist)
        elif args.impl == "reference":
            (run_reference_a1 if args.schedule == "a1" else run_reference)(args, dist)
        elif args.schedule == "a1":
            run_a1(args, dist)
        else:
            run_ours(args, dist)
    finally:
        dist.close()


if __name__ == "__main__":
    main()
