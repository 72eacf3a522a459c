#!/usr/bin/env python
"""Benchmark of the GP-surrogate + EI hot path (BASELINE.json metric) on 1..8 B200s.

One step = one pass of the whole hot path over one batch: gp_fit (H1-H4) on the observed
configurations + ei_score_argmax (H6-H10: fast tensor/CUDA-core phase, float64 refine of the
candidates that can still win, per-search argmax, NCCL max-all-reduce across ranks).

Workload (N=1 line): BASELINE.json configs[1] -- one 20-parameter search, n = 200 observations,
M = 2^20 random candidates per GPU (weak scaling: each rank scores its own 2^20-candidate shard
of a pool of N * 2^20; the fit is replicated).  Inputs are seeded synthetic data shaped like the
paper's (workloads/gen.py), resident in HBM when timing starts; L2 is
flushed (256 MiB write) between timed steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C]

Prints ONE JSON line on rank 0.  `--impl reference` times the float64 CPU oracle (oracle/) on a
bounded sample of the same workload (rank 0 only; other ranks exit 0).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "GP-posterior+EI candidates scored/sec at 1/2/4/8 B200; % of roofline"
UNIT = "candidates/s"


def flops_per_candidate(n, d):
    """F_c = 2nd (distances) + n(n+1) (triangular V) + 4n (mu, sum v^2)."""
    return 2 * n * d + n * (n + 1) + 4 * n


def profiled_traffic(kernel, config):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes per launch) of `kernel` from the latest
    committed ncu --set full summary under profiles/ taken on the same bench config, else None."""
    import glob
    want = "--config 4" if config == 4 else ""
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_{kernel}_summary.txt"))):
        lines = open(f).read().splitlines()
        if not lines or ("--config" in lines[0]) != bool(want) or (want and want not in lines[0]):
            continue
        if config not in (2, 4):
            continue
        vals = {}
        for ln in lines:
            for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                if ln.startswith(key + ":"):
                    vals[key] = float(ln.split(":")[1])
        if len(vals) == 2:  # ncu reports MB
            best = ((vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]) * 1e6,
                    os.path.relpath(f, ROOT))
    return best


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return dict(hbm=j.get("hbm_gbs", 6650.0), bf16=j.get("bf16_tflops", 1590.0),
                    bf16_sus=j.get("bf16_tflops_sustained", 1400.0),
                    sm_mhz=j.get("sm_max_mhz", 1965.0), src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, sm_mhz=1965.0, src="fallback")


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region: NVML polled
    every ~0.5 ms in a thread (the timed region of a default run is ~10 ms, too short for
    nvidia-smi's 100 ms sampling, which remains the fallback when NVML is unavailable)."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, gpus):
        self.gpus = gpus
        self.sm, self.mx, self.reasons, self.n = [], [], set(), 0
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        if self.gpus <= 0:
            return self
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = [int(v) for v in vis.split(",")] if vis and vis[0].isdigit() else None
            self.handles = [pynvml.nvmlDeviceGetHandleByIndex(idx[g] if idx else g)
                            for g in range(self.gpus)]
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None
        return self

    def _poll(self):
        nv = self.nvml
        while not self.stop.is_set():
            for h in self.handles:
                try:
                    self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    self.mx.append(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for name, attr in self.REASONS:
                        if r & getattr(nv, attr, 0):
                            self.reasons.add(name)
                    self.n += 1
                except Exception:
                    pass
            time.sleep(0.0005)

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                "samples": self.n, "source": "nvml, 0.5 ms polling during the timed region"}


def cpu_oracle_rate(cfg, M_sample, threads=None, layout="uniform", want_results=False):
    """Time the float64 oracle on a bounded sample of the workload (host cores; `threads` BLAS
    threads, default all).  want_results: also return the oracle's ScoreResult per search."""
    from threadpoolctl import threadpool_limits
    from oracle import gp
    from workloads import gen
    cores = threads or os.cpu_count()
    w = gen.make(cfg, M=M_sample, layout=layout)
    res = []
    with threadpool_limits(limits=cores):
        t0 = time.perf_counter()
        for s, Xs in zip(w.searches, w.Xstar):
            m = gp.fit(s.X, s.y, s.lengthscale, s.sf2, s.sn2, w.kernel)
            res.append(gp.score(m, Xs))
        dt = time.perf_counter() - t0
    total = sum(x.shape[0] for x in w.Xstar)
    if want_results:
        return total / dt, cores, total, dt, res
    return total / dt, cores, total, dt


def cpu_model():
    """Host CPU model name (lscpu 'Model name', else /proc/cpuinfo)."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def spawn_ranks(ngpus):
    """`bench.py --gpus N` without a torchrun environment: re-exec under torch.distributed.run
    with N ranks on this node (127.0.0.1 rendezvous), as the driver launches it."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={ngpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def replay_raw(params, row):
    """raw values of one Table IV configuration from per-parameter value indices"""
    out = []
    for v, p in zip(row, params):
        out.append(float(p["values"][int(v)]) if p["kind"] == 2 else
                   float(p["lo"] + int(v)) if p["kind"] == 1 else float(v))
    return np.array(out)


def replay_vidx(params, raw):
    """value indices of one configuration from its raw values (inverse of replay_raw)"""
    out = []
    for v, p in zip(raw, params):
        out.append(int(np.argmin(np.abs(np.asarray(p["values"], float) - v))) if p["kind"] == 2
                   else int(round(v - p["lo"])) if p["kind"] == 1 else int(round(v)))
    return np.array(out, np.int64)


def bench_replay(args, world, rank, local):
    """Config 5 (BASELINE.json configs[4]): the tuning-campaign replay on the Table IV space.
    One step = one sequential BO iteration: the surrogate update with the new observation
    (gp_fit_append, O(n^2)) + bo_suggest_batch (M = 2^18 candidates generated
    on the device under the Table IV constraints, dedup against the history, scoring, argmax,
    decode).  W untimed iterations, then K timed ones continuing the same campaign (n grows from
    5 + W); the host objective (R18) runs between steps, outside the timed region.  e2e: the same
    steps timed with the host -> device copy of the new observation and the suggestion's read-back
    inside (the candidates never cross PCIe)."""
    import torch
    from paper_2403_08131_b200 import gpbo
    from workloads import rttddft
    dev = torch.device("cuda", local)
    torch.cuda.set_device(local)
    stream = torch.cuda.current_stream()
    ctx = gpbo.Context(device=local, stream=stream)
    params, blocks, _ = rttddft.table_iv()
    sp = gpbo.Space(ctx, params, blocks)
    d = sp.dim
    M = 1 << 18
    vidx = rttddft.initial_design(params, blocks, 5, 5)
    y = rttddft.objective(vidx, params)
    X = np.concatenate([sp.encode(replay_raw(params, r)[None, :]) for r in vidx]).astype(np.float32)
    ls = np.full(d, 0.4 * np.sqrt(d), np.float32)
    sf2 = np.ones(1, np.float32)
    sn2 = np.full(1, 1e-4, np.float32)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    m = ctx.fit([len(y)], [d], np.ascontiguousarray(X.ravel()), y, ls, sf2, sn2)
    xd = torch.empty(d, dtype=torch.float32, device=dev)
    yd = torch.empty(1, dtype=torch.float64, device=dev)
    xpin = torch.empty(d, dtype=torch.float32).pin_memory()
    ypin = torch.empty(1, dtype=torch.float64).pin_memory()
    dev_ms, e2e_ms, launches, impls, refined = [], [], 0, {}, 0
    ctx.set_profiling(True)
    for it in range(args.warmup + args.steps):
        timed = it >= args.warmup
        flush.zero_()
        l0 = ctx.launches
        if it > 0:  # the previous suggestion's observation: pinned host -> device inside e2e
            xpin.copy_(torch.from_numpy(X[-1]))
            ypin.copy_(torch.from_numpy(y[-1:]))
        stream.synchronize()
        e0.record(stream)
        if it > 0:
            xd.copy_(xpin, non_blocking=True)
            yd.copy_(ypin, non_blocking=True)
            m2 = ctx.fit_append(m, xd, yd)
            m.free()
            m = m2
        t0 = time.perf_counter()
        idx, xr, ei = gpbo.suggest(ctx, m, [sp], [M], 5, it, dedup=True)  # ends synchronised
        e1.record(stream)
        e1.synchronize()
        if timed:
            dev_ms.append(e0.elapsed_time(e1))
            launches += ctx.launches - l0
            impls[ctx.last_impl] = impls.get(ctx.last_impl, 0) + 1
            refined += ctx.last_refine_count
        del t0
        raw = np.asarray(xr[0], np.float64)
        vnew = replay_vidx(params, raw)
        X = np.concatenate([X, sp.encode(raw[None, :]).astype(np.float32)])
        y = np.concatenate([y, rttddft.objective(vnew[None, :], params)])
    kt = {k: ctx.kernel_time(k) for k in ctx.KERNELS}
    ctx.set_profiling(False)
    m.free()
    T = float(np.sum(dev_ms))
    value = M * args.steps / (T / 1e3)
    names = {1: "cuda-core", 2: "tcgen05", 3: "tcgen05-stream", 4: "fp64-direct"}
    fast_n, fast_ms = kt["fast"]
    return ctx, dict(value=value, T=T, launches=launches, kt=kt, refined=refined,
                     impls={names.get(k, str(k)): v for k, v in impls.items()},
                     n_first=5 + args.warmup, n_last=5 + args.warmup + args.steps - 1, d=d,
                     fast_ms=fast_ms / max(fast_n, 1), best_y=float(np.min(y)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--layout", default="uniform", choices=["uniform", "bo"])
    ap.add_argument("--score-impl", type=int, default=0, help="0 auto, 1 CUDA-core, 2 tcgen05")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=1 << 20,
                    help="candidates the CPU oracle scores for cpu_baseline (~10-15 s at config 2)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: fixed candidates per GPU; strong: the config's M split over N")
    ap.add_argument("--shard", default="candidates", choices=["candidates", "searches"],
                    help="candidates: every rank scores a slice of every search, one all-reduce "
                         "of the keys (H10); searches: rank r takes searches r, r + N, ... whole "
                         "(no collective; the SURVEY.md §8(e) ablation for config 3)")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the configs 1/3/4/5 sub-runs summarised in the config-2 line")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        spawn_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:  # the NCCL communicator init lines (stderr) document the H10 transport
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    from workloads import gen
    S0, n0, d0, M0 = gen.CONFIG_SHAPES[args.config]
    # weak scaling: configs 1-3 keep their M per GPU, config 4 its 2^19 per-GPU shard; strong
    # scaling: the config's whole pool split over the ranks
    per_gpu = M0 if args.config != 4 else M0 // 8
    if args.scaling == "strong":
        per_gpu = -(-M0 // world)

    if args.impl == "reference":
        if rank != 0:
            return
        # the oracle as it stands, each step a bounded sample of the same workload
        M_ref = max(4096, min(per_gpu, 1 << 14))
        times = []
        for i in range(args.warmup + args.steps):
            rate, cores, total, dt = cpu_oracle_rate(args.config, M_ref)
            if i >= args.warmup:
                times.append(dt)
        T = float(np.sum(times))
        value = total * args.steps / T
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": gen.CONFIG_NAMES[args.config], "S": S0, "n": n0,
                           "d": d0, "M_per_step_sample": M_ref},
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores,
                                 "kind": "oracle",
                                 "sample": f"{M_ref} candidates of {gen.CONFIG_NAMES[args.config]}"
                                           " per step (fit + score + argmax, float64 numpy)"},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if args.config == 5:
        return main_replay(args, world, rank, local)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2403_08131_b200 import gpbo

    nccl_id = None
    if world > 1 and args.shard == "candidates":
        obj = [gpbo.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    stream = torch.cuda.current_stream()
    shard_s = args.shard == "searches"
    ctx = gpbo.Context(device=local, stream=stream, nranks=1 if shard_s else world,
                       rank=0 if shard_s else rank, nccl_id=nccl_id)
    ctx.set_score_impl(args.score_impl)

    # ---- inputs (seeded, host -> HBM once, untimed)
    M_total = M0 if args.scaling == "strong" else per_gpu * world
    if shard_s:  # whole searches per rank: the config's full pool of each of its searches
        M_total = M0
        ids = list(range(rank, S0, world))
        if not ids:
            raise SystemExit(f"--shard searches: rank {rank} has no search (S = {S0} < N)")
        w = gen.make(args.config, M=M0, layout=args.layout, search_ids=ids)
    else:
        w = gen.make(args.config, M=M_total, rank=rank, world=world, layout=args.layout)
    S = w.S
    n = [s.X.shape[0] for s in w.searches]
    d = [s.X.shape[1] for s in w.searches]
    Xh = np.ascontiguousarray(np.concatenate([s.X.ravel() for s in w.searches]), np.float32)
    yh = np.ascontiguousarray(np.concatenate([s.y for s in w.searches]), np.float64)
    lsh = np.ascontiguousarray(np.concatenate([s.lengthscale for s in w.searches]), np.float32)
    sf2h = np.array([s.sf2 for s in w.searches], np.float32)
    sn2h = np.array([s.sn2 for s in w.searches], np.float32)
    Xsh = np.ascontiguousarray(np.concatenate([x.ravel() for x in w.Xstar]), np.float32)
    m_off = np.zeros(S + 1, np.int64)
    m_off[1:] = np.cumsum([x.shape[0] for x in w.Xstar])
    base = np.array(w.m_global_base, np.int64)
    t = lambda a: torch.from_numpy(a).to(dev)
    Xd, yd, lsd, sf2d, sn2d, Xsd = t(Xh), t(yh), t(lsh), t(sf2h), t(sn2h), t(Xsh)
    Xs_pin = torch.from_numpy(Xsh).pin_memory()
    local_cands = int(m_off[-1])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step_device():
        m = ctx.fit(n, d, Xd, yd, lsd, sf2d, sn2d, kernel=w.kernel, wait=False)
        idx, ei = ctx.score_argmax(m, Xsd, m_off, base)
        m.free()
        return idx, ei

    def step_host():
        m = ctx.fit(n, d, Xh, yh, lsh, sf2h, sn2h, kernel=w.kernel, wait=False)
        idx, ei = ctx.score_argmax(m, Xs_pin, m_off, base)
        m.free()
        return idx, ei

    def step_score(m):
        """score-only: the fitted model stays resident (SURVEY.md §8(d) primary scaling metric)"""
        return ctx.score_argmax(m, Xsd, m_off, base)

    def timed(step, K, W, profile=False):
        for _ in range(W):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        l0 = ctx.launches
        ctx.set_profiling(profile)
        tot = 0.0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        refined = 0
        for _ in range(K):
            flush.zero_()
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
            refined += ctx.last_refine_count
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        kt = {k: ctx.kernel_time(k) for k in ctx.KERNELS}
        ctx.set_profiling(False)
        return tot, ctx.launches - l0, kt, refined

    # ---- device-resident timing (the value) with clocks sampled during it.  No per-kernel events
    # here: timing events around each library launch cost ~6 % of the step on the device.
    with ClockSampler(world if rank == 0 else 0) as clk:
        T_dev, launches, _, refined = timed(step_device, args.steps, args.warmup)
    # ---- the same steps again with CUDA events around every library kernel (on the ctx stream):
    # the per-kernel breakdown and the fast-phase launch duration of the roofline
    _, _, kt, _ = timed(step_device, args.steps, args.warmup, profile=True)
    # ---- end-to-end through the C ABI with host buffers
    T_e2e, _, _, _ = timed(step_host, args.steps, args.warmup)
    # ---- end to end through bo_suggest_batch (the BO user's call): per step the observations
    # (host) go in, the suggestion comes out; the M candidates of each search are drawn on the
    # device from the search's parameter box (d REAL parameters in [0, 1], the workload's
    # uniform candidates; H5) -- no candidate crosses PCIe
    T_sug = None
    if world == 1 and args.layout == "uniform":
        spaces = [gpbo.Space(ctx, [{"kind": 0, "lo": 0.0, "hi": 1.0}] * dd) for dd in d]
        Msug = np.diff(m_off).astype(np.int64)
        it_ctr = [0]

        def step_suggest():
            m = ctx.fit(n, d, Xh, yh, lsh, sf2h, sn2h, kernel=w.kernel, wait=False)
            it_ctr[0] += 1
            out = gpbo.suggest(ctx, m, spaces, Msug, 1234, it_ctr[0], dedup=True)
            m.free()
            return out

        T_sug, _, _, _ = timed(step_suggest, args.steps, args.warmup)
        del spaces
    # ---- score-only (model resident, fit outside the timed region): H6-H10 alone
    m_res = ctx.fit(n, d, Xd, yd, lsd, sf2d, sn2d, kernel=w.kernel)
    T_score, _, _, _ = timed(lambda: step_score(m_res), args.steps, args.warmup)
    # ---- gp_posterior (H6-H8 raw mu / var / EI of every candidate, float64 on DMMA) of search 0
    T_post, M_post = None, 0
    if world == 1:
        M_post = int(m_off[1])
        Xs0 = Xsd[: M_post * d[0]].view(M_post, d[0])
        T_post, _, _, _ = timed(lambda: ctx.posterior(m_res, 0, Xs0), args.steps, args.warmup)
    m_res.free()

    def vmax(x):
        if world == 1:
            return x
        tt = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    T_dev, T_e2e, T_score = vmax(T_dev), vmax(T_e2e), vmax(T_score)
    fast_n, fast_ms = kt["fast"]
    fast_ms = vmax(fast_ms)
    # every rank scores its local shard of every search: the candidates of all ranks per step
    global_cands = local_cands
    if world > 1:
        tt = torch.tensor([local_cands], dtype=torch.int64, device=dev)
        dist.all_reduce(tt)
        global_cands = int(tt.item())
    total_cands = global_cands * args.steps
    value = total_cands / (T_dev / 1e3)
    e2e_value = total_cands / (T_e2e / 1e3)
    score_value = total_cands / (T_score / 1e3)
    idx, ei = step_device()
    if rank == 0:
        peaks = load_peaks()
        impl_used = {2: "tcgen05", 3: "tcgen05-stream", 4: "fp64-direct"}.get(ctx.last_impl,
                                                                             "cuda-core")
        Fc = sum(flops_per_candidate(nn, dd) * x.shape[0] for nn, dd, x in zip(n, d, w.Xstar))
        achieved = Fc / (fast_ms / fast_n / 1e3) / 1e12  # TFLOP/s of the fast-phase kernel
        clocks = clk.summary()
        # the burst peak applies when the clocks stayed at max with no cap during the timed
        # region (the kernel runs in ~0.1-3 ms bursts); else the sustained one
        capped = bool(clocks["reasons"]) or not (clocks["sm_mhz"] and clocks["sm_max_mhz"] and
                                                 clocks["sm_mhz"] >= 0.97 * clocks["sm_max_mhz"])
        if impl_used.startswith("tcgen05"):
            peak = peaks["bf16_sus"] if capped else peaks["bf16"]
            tr = profiled_traffic("score_tcs" if impl_used == "tcgen05-stream" else "score_tc",
                                  args.config)
            roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak,
                    "fp16x3_ceiling": {"peak": peak / 3, "frac": achieved / (peak / 3),
                                       "why": "every contraction runs as 3 fp16 MMAs (hi.hi + "
                                              "hi.lo + lo.hi: float32-level products for the "
                                              "1e-4 parity), so the algorithmic flops can reach "
                                              "at most 1/3 of the fp16 peak"},
                    "traffic": tr[0] if tr else None,
                    "traffic_src": tr[1] if tr else None,
                    "algorithmic_bytes": int(sum(4 * dd * x.shape[0] for dd, x in zip(d, w.Xstar))),
                    "peak_src": f"{peaks['src']} bf16 dense "
                                f"{'sustained' if capped else 'burst (clocks at max, no cap)'}"
                                " (fp16 same rate)"}
        elif impl_used == "fp64-direct":
            peak = 148 * 64 * 2 * peaks["sm_mhz"] * 1e6 / 1e12
            roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": None,
                    "peak_src": "FP64 DFMA: 148 SM x 64 lanes x 2 flop x max SM clock "
                                "(tools/micro: 58-64 DFMA/clk/SM); small problem: latency-bound"}
        else:
            peak = 148 * 128 * 2 * peaks["sm_mhz"] * 1e6 / 1e12
            roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": None,
                    "peak_src": "FP32 FFMA: 148 SM x 128 lanes x 2 flop x max SM clock"}
        cpu = None
        oracle_check = None
        if world == 1 and not args.no_cpu_baseline:
            rate, cores, tot_c, dt, ores = cpu_oracle_rate(args.config, args.cpu_sample,
                                                           layout=args.layout, want_results=True)
            # 1-thread figure on a smaller sample (SURVEY.md §8(d) oracle timing)
            m1 = max(4096, args.cpu_sample // 16)
            rate1, _, tot1, dt1 = cpu_oracle_rate(args.config, m1, threads=1, layout=args.layout)
            cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"{tot_c} candidates of {gen.CONFIG_NAMES[args.config]} "
                             f"(fit + score + argmax, float64 numpy, {dt:.1f} s)",
                   "cpu_model": cpu_model(),
                   "one_thread": {"value": rate1, "unit": UNIT, "cores": 1,
                                  "sample": f"{tot1} candidates ({dt1:.1f} s)"}}
            # the GPU's suggestion vs the oracle's argmax on the same candidates, where the
            # sample is the whole timed workload (reading R11: index parity where the gap is
            # decisive, else a pick within 1e-3 of the oracle's maximum)
            if tot_c == local_cands:
                ok, detail = True, []
                for si, r in enumerate(ores):
                    gi = int(idx[si])
                    top = float(r.ei_all.max())
                    exact = r.gap_rel > 1e-3 and top >= 1e-30
                    good = (gi == r.idx) if exact else (
                        0 <= gi < r.ei_all.size and (top < 1e-30 or r.ei_all[gi] >= top * (1 - 1e-3)))
                    ok = ok and good
                    if si < 4:
                        detail.append({"gpu_idx": gi, "oracle_idx": r.idx,
                                       "gap_rel": r.gap_rel, "decisive": exact})
                oracle_check = {"oracle_idx_match": ok, "searches": len(ores),
                                "first": detail}
        h2d = Xh.nbytes + yh.nbytes + lsh.nbytes + sf2h.nbytes + sn2h.nbytes + Xsh.nbytes
        d2h = 8 * S + 4 + 192 * S
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": T_dev / args.steps,
            "higher_is_better": True,
            "scaling": "strong" if shard_s else args.scaling, "vs_baseline": None,
            "dtype": ("f16x3+f32+f64" if impl_used.startswith("tcgen05") else
                      "f64" if impl_used == "fp64-direct" else "f32+f64"),
            "data": "synthetic",
            "config": {"workload": gen.CONFIG_NAMES[args.config], "S": S, "n": n0, "d": d0,
                       "M_per_gpu": per_gpu, "M_global": M_total, "shard": args.shard,
                       "candidates_per_step": global_cands,
                       "kernel": "matern52" if w.kernel == 1 else "rbf",
                       "layout": args.layout, "l2": "flushed between steps (256 MiB write)",
                       "scoring": impl_used},
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "e2e_suggest": None if T_sug is None else {
                "value": total_cands / (T_sug / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": int(Xh.nbytes + yh.nbytes + lsh.nbytes + sf2h.nbytes +
                                          sn2h.nbytes),
                "d2h_bytes_per_step": int(8 * S + 4 * S + 8 * sum(d)),
                "what": "gp_fit (host observations) + bo_suggest_batch (candidates drawn on the "
                        "device from the parameter box, H5) -> suggestion read back"},
            "posterior": None if T_post is None else {
                "value": M_post * args.steps / (T_post / 1e3), "unit": UNIT,
                "ms_per_call": T_post / args.steps, "candidates": M_post,
                "what": "gp_posterior of search 0 on a resident model: raw mu, var, EI of every "
                        "candidate in float64 (K* and V = L^-1 K*^T on the FP64 tensor cores)",
                "roofline": {"bound": "tensor-fp64",
                             "achieved": (n[0] * (n[0] + 1) + 2 * n[0] * d[0] + 2 * n[0]) *
                                         M_post * args.steps / (T_post / 1e3) / 1e12,
                             "peak": 45.0, "unit": "TFLOP/s",
                             "peak_src": "B200 FP64 tensor nominal (blackwell_cuda_programming.md)"}},
            "score_only": {"value": score_value, "unit": UNIT,
                           "ms_per_step": T_score / args.steps,
                           "what": "ei_score_argmax alone on a resident model (H6-H10)"},
            "clocks": clocks, "gpu_launches": int(launches),
            "breakdown_ms_per_step": {k: kt[k][1] / args.steps for k in kt},
            "breakdown_src": "second timed pass of the same steps with CUDA events around each "
                             "library kernel (events perturb the step by ~6 %, so the value's "
                             "pass runs without them)",
            "refined_per_step": refined / args.steps,
            "result": {"idx": int(idx[0]), "ei": float(ei[0])},
            "oracle_check": oracle_check,
            "collectives": ctx.collectives,
        }
        if line["posterior"]:
            pr = line["posterior"]["roofline"]
            pr["frac"] = pr["achieved"] / pr["peak"]
        if (args.config == 2 and world == 1 and args.layout == "uniform" and
                args.scaling == "weak" and not args.no_other_configs):
            line["other_configs"] = other_configs(args)
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def other_configs(args):
    """The other BASELINE configs measured in the same run (sub-processes of this script on the
    same GPU, after this run's own timing): per config the bench line's value, step time,
    breakdown, roofline fraction and clocks -- so the driver-run line covers configs 1-5."""
    import subprocess
    out = {}
    for c, extra in ((1, []), (3, []), (4, []), (5, ["--steps", "100"])):
        cmd = [sys.executable, os.path.abspath(__file__), "--config", str(c), "--warmup", "3",
               "--no-cpu-baseline", "--no-other-configs"]
        cmd += extra if extra else ["--steps", str(min(args.steps, 20))]
        env = {k: v for k, v in os.environ.items()
               if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
            j = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
        except Exception as e:  # a failed sub-run is reported, not fatal
            out[f"cfg{c}"] = {"error": f"{type(e).__name__}: {e}"[:200]}
            continue
        roof = j.get("roofline") or {}
        out[f"cfg{c}"] = {
            "workload": (j.get("config") or {}).get("workload"),
            "value": j.get("value"), "unit": j.get("unit"), "ms_per_step": j.get("ms_per_step"),
            "steps": j.get("steps"),
            "breakdown_ms_per_step": j.get("breakdown_ms_per_step"),
            "roofline_frac": roof.get("frac"), "roofline_bound": roof.get("bound"),
            "score_only": (j.get("score_only") or {}).get("value"),
            "e2e": (j.get("e2e") or {}).get("value"),
            "e2e_suggest": (j.get("e2e_suggest") or {}).get("value"),
            "refined_per_step": j.get("refined_per_step"),
            "clocks": j.get("clocks"), "gpu_launches": j.get("gpu_launches")}
    return out


def main_replay(args, world, rank, local):
    """bench.py --config 5: one JSON line for the replay (rank 0; replicas only for N > 1 --
    one BO campaign is sequential and does not shard)."""
    from workloads import gen
    with ClockSampler(1 if rank == 0 else 0) as clk:
        ctx, r = bench_replay(args, world, rank, local)
    if rank != 0:
        ctx.close()
        return
    peaks = load_peaks()
    n_mid = (r["n_first"] + r["n_last"]) / 2.0
    Fc = flops_per_candidate(n_mid, r["d"]) * (1 << 18)
    achieved = Fc / (r["fast_ms"] / 1e3) / 1e12
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["T"] / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f16x3+f32+f64", "data": "synthetic",
        "config": {"workload": gen.CONFIG_NAMES[5] + ", M=262,144 on-device candidates per "
                               "iteration, fit_append + bo_suggest_batch per step",
                   "n_range": [r["n_first"], r["n_last"]], "d": r["d"], "M_per_step": 1 << 18,
                   "l2": "flushed between steps (256 MiB write)", "scoring": r["impls"]},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16"],
                     "unit": "TFLOP/s", "frac": achieved / peaks["bf16"], "traffic": None,
                     "peak_src": f"{peaks['src']} bf16 dense burst (fp16 same rate); F_c at the "
                                 "mean n of the timed iterations"},
        "cpu_baseline": None,
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 4 * r["d"] + 8,
                "d2h_bytes_per_step": 8 + 8 * 20 + 4,
                "what": "the timed steps include the new observation's pinned host->device copy "
                        "and the suggestion's read-back; candidates are generated on the device"},
        "clocks": clocks, "gpu_launches": int(r["launches"]),
        "breakdown_ms_per_step": {k: v[1] / (args.warmup + args.steps) for k, v in r["kt"].items()},
        "refined_per_step": r["refined"] / args.steps,
        "result": {"best_y": r["best_y"]},
    }
    print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
