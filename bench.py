#!/usr/bin/env python
"""Benchmark of the NBM loss+grad training step (BASELINE.json metric: collocation-point
loss+grad evaluations/s and steps/s at 1/2/4/8 B200, % roofline).

One step = sample (interior + boundary, K1) -> nbm_loss_grad (K2 classify/assemble,
K3 fused MLP fwd/residual/bwd, K4r reduce) -> all-reduce of [grad, loss] (N > 1) ->
nbm_adam_step (K4a).  Default workload: BASELINE config 4 (configs[3], the north_star's
2^22 points/step): union of 32 spheres, two 3-256^4-1 tanh bf16 MLPs, 2^22 interior + 2^19
boundary points per GPU (weak scaling), h = 2/1023.  A `secondary` record times config 5 at
width 256 in fp32 (the paper's own arithmetic) on the same points.  Synthetic seeded data (the
paper's dragon scan is not available).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl reference]
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N ... (NCCL all-reduce).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2210_14907_b200 import dp, inputs  # noqa: E402

METRIC = "collocation-pt loss+grad evals/sec (full training step)"
FP32_FFMA_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4: SMs x FFMA lanes x 2 x max clock
# measured on this pool's B200 (scripts/ffma_peak.cu, 1965 MHz): FFMA with three register
# operands, the form a GEMM issues, reaches 57.0 TFLOP/s (the immediate form 71.0)
FP32_FFMA_3REG_MEASURED_TFLOPS = 57.0


def mlp_macs(sizes):
    """(forward MACs, forward+backward MACs) per evaluation, algorithmic."""
    fwd = sum(sizes[l - 1] * sizes[l] for l in range(1, len(sizes)))
    dh = sum(sizes[l - 1] * sizes[l] for l in range(2, len(sizes)))
    return fwd, 2 * fwd + dh


def kernel_name(cfg):
    w = cfg["sizes"][1]
    if cfg["prec"] == inputs.PREC_FP32:
        return "k_mlp_fp32w" if w >= 128 else "k_mlp_fp32"
    if cfg["prec"] == inputs.PREC_FP32X:
        return "k_mlp_tc<P=3> (tcgen05, 3-plane bf16 split)"
    if cfg.get("stencil", 0) == inputs.STENCIL_STABLE:
        return "k_mlp_tc<STAB> (tcgen05, difference propagation)"
    if w == 256:
        return "k_mlp_w256 (tcgen05 cta_group::2)"
    nh = len(cfg["sizes"]) - 2
    if w == 128 and cfg["act"] == inputs.ACT_TANH and 3 <= nh <= 4 and not os.environ.get("NBM_TCH_OFF"):
        return "k_mlp_tch (tcgen05, two 64-row half-tiles in flight)"
    return "k_mlp_tc (tcgen05)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg, levels=1):
    """The oracle as it stands (fp64 C, OpenMP with a fixed-order reduction) on a seeded
    subsample of the same workload: 2^12 interior + 2^9 boundary points on all
    host cores, 2^10 + 2^7 on one core.  Loss+grad cost is exactly linear in the point count,
    so pts/s carries over to the full N; the full-step time is extrapolated and marked so."""
    import oracle
    pb, ar = oracle.from_config(cfg)
    th = oracle.init_params(ar, 0)

    def run(n, threads):
        nb = max(1, n * cfg["Nb"] // cfg["N"])
        pts = oracle.sample(0, 0, 0, 0, n, cfg["H"])
        bpts = oracle.sample(1, 0, 0, 0, nb, cfg["H"])
        t0 = time.perf_counter()
        if levels == 1:
            oracle.loss_grad(pb, ar, th, pts, bpts, cfg["h"], n_glob=cfg["N"], nb_glob=cfg["Nb"], nthreads=threads)
        else:
            oracle.loss_grad_ml(pb, ar, th, pts, bpts, cfg["h"], levels, n_glob=cfg["N"], nb_glob=cfg["Nb"])
        return n, nb, time.perf_counter() - t0

    cores = oracle.num_threads()
    n, nb, dt = run(min(cfg["N"], 1 << 12), cores)
    n1, nb1, dt1 = run(min(cfg["N"], 1 << 10), 1)
    return {"value": n / dt, "unit": "pts/s", "cores": cores, "kind": "oracle",
            "sample": f"{n} interior + {nb} boundary points of {cfg['label']} (seeded subsample, fp64 loss+grad, "
                      f"{dt:.2f} s on {cores} threads); pts/s carries over linearly to N = {cfg['N']}",
            "extrapolated_step_s": dt * cfg["N"] / n, "extrapolated": True,
            "one_core": {"value": n1 / dt1, "unit": "pts/s", "cores": 1,
                         "sample": f"{n1} interior + {nb1} boundary points ({dt1:.2f} s)",
                         "extrapolated_step_s": dt1 * cfg["N"] / n1},
            "nproc": os.cpu_count(), "cpu_model": cpu_model()}


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle (CPU, fp64) as the reference arm, rank 0 only."""
    if rank != 0:
        return
    import oracle
    pb, ar = oracle.from_config(cfg)
    th = oracle.init_params(ar, 0).astype("float64")
    m = th * 0
    v = th * 0
    n = 1 << 12
    nb = max(1, n * cfg["Nb"] // cfg["N"])
    times = []
    for it in range(args.warmup + args.steps):
        pts = oracle.sample(0, 0, it, 0, n, cfg["H"])
        bpts = oracle.sample(1, 0, it, 0, nb, cfg["H"])
        t0 = time.perf_counter()
        if args.levels == 1:
            _, _, g, _ = oracle.loss_grad(pb, ar, th, pts, bpts, cfg["h"], n_glob=n, nb_glob=nb)
        else:
            _, g = oracle.loss_grad_ml(pb, ar, th, pts, bpts, cfg["h"], args.levels, n_glob=n, nb_glob=nb)
        th, m, v = oracle.adam(th, m, v, g, it + 1, lr=cfg["lr"])
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = n * len(times) / tot
    line = {"metric": METRIC, "value": val, "unit": "pts/s",
            "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["label"], "points_per_gpu": cfg["N"], "boundary_per_gpu": cfg["Nb"],
                       "mlp": "x".join(map(str, cfg["sizes"])), "n_nets": cfg["n_nets"], "h": cfg["h"],
                       "levels": args.levels, "parallelism": "host cores",
                       "sample_points_per_step": n, "sample_boundary_per_step": nb,
                       "note": "the fp64 oracle on a bounded sample of the workload per step (host cores)"},
            "cpu_baseline": {"value": val, "unit": "pts/s", "cores": oracle.num_threads(),
                             "kind": "oracle", "sample": f"{n} + {nb} points per step"},
            "e2e": {"value": val, "unit": "pts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_secondary(args):
    """config 5 at width 256 in IEEE fp32 (K3fw; the paper's own arithmetic) on
    2^22 + 2^19 points: graph-replayed steps timed with CUDA events, L2 flushed between steps,
    the fused kernel timed by the library's event hook (roofline: the fp32 FFMA peak)."""
    import torch
    from paper_2210_14907_b200 import nbm
    cfg = inputs.config("c5", width=256, prec=inputs.PREC_FP32)
    N, Nb = cfg["N"], cfg["Nb"]
    s = nbm.Solver(cfg, device=torch.cuda.current_device(), max_points=max(N, Nb))
    s.init_params(0)
    pts = torch.empty(N, 3, device="cuda")
    bpts = torch.empty(Nb, 3, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    steps, warm = 3, 3

    def step(it):
        s.sample(nbm.POINTS_INTERIOR, 0, it, 0, N, pts)
        s.sample(nbm.POINTS_BOUNDARY, 0, it, 0, Nb, bpts)
        s.loss_grad(pts, bpts)
        s.adam_step(lr=cfg["lr"])
    for it in range(warm):
        step(it)
    nbm.nbm_timing_enable(s.h, True)
    nbm.nbm_timing_read(s.h)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for k in range(steps):
        flush.zero_()
        ev[k][0].record(stream)
        step(warm + k)
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    mlp_ms, _, calls = nbm.nbm_timing_read(s.h)
    tot = sum(a.elapsed_time(b) for a, b in ev)
    st = s.status()
    s.close()
    _, fb = mlp_macs(cfg["sizes"])
    flop = 2.0 * fb * (7 * N + Nb)
    achieved = flop / (mlp_ms / max(calls, 1) / 1e3) / 1e12
    return {"workload": "c5-w256-fp32", "metric": METRIC, "value": N * steps / (tot / 1e3), "unit": "pts/s",
            "steps": steps, "warmup": warm, "ms_per_step": tot / steps, "dtype": "f32", "status": st,
            "launch_mode": "eager", "points_per_gpu": N, "boundary_per_gpu": Nb, "mlp": "3x256x256x256x256x1",
            "roofline": {"bound": "alu", "achieved": achieved, "peak": FP32_FFMA_TFLOPS, "unit": "TFLOP/s",
                         "frac": achieved / FP32_FFMA_TFLOPS, "kernel": "k_mlp_fp32w fused fwd/residual/bwd",
                         "avg_launch_ms": mlp_ms / max(calls, 1),
                         "peak_src": "fp32 FFMA: 148 SM x 128 lanes x 2 FLOP x 1965 MHz (derived, DESIGN.md)"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--no-secondary", action="store_true", help="skip the fp32 c5-w256 secondary record")
    ap.add_argument("--width", type=int, default=None)
    ap.add_argument("--prec", default=None, choices=["fp32", "bf16", "fp32x"], help="override the config's precision (c4/c5)")
    ap.add_argument("--impl", default="nbm", choices=["nbm", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA-graph replays")
    ap.add_argument("--eval", action="store_true", help="also time inference (nbm_eval) at the step's points")
    ap.add_argument("--grid", type=int, default=None,
                    help="replace the level set by its samples on an Nc^3 grid (S:82 Sampled variant, P:60)")
    ap.add_argument("--levels", type=int, default=1,
                    help="multi-resolution levels h0/2^l of the loss (S:348; the paper's scaling runs use 3)")
    ap.add_argument("--points", type=int, default=None, help="override interior points per GPU")
    ap.add_argument("--stencil", default="direct", choices=["direct", "stable"],
                    help="uncrossed stencil evaluation: 7 network values or difference propagation (G27; bf16 tanh)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local = dp.env_rank_world()
    prec = None if args.prec is None else {"fp32": inputs.PREC_FP32, "bf16": inputs.PREC_BF16,
                                            "fp32x": inputs.PREC_FP32X}[args.prec]
    cfg = inputs.config(args.config, width=args.width, prec=prec)
    if args.grid:
        cfg = inputs.with_grid(cfg, args.grid)
    cfg["stencil"] = inputs.STENCIL_STABLE if args.stencil == "stable" else inputs.STENCIL_DIRECT
    cfg["label"] = cfg["name"] + (f"-w{cfg['sizes'][1]}" if cfg["name"] == "c5" else "") + \
        ("" if prec is None else {inputs.PREC_FP32: "-fp32", inputs.PREC_BF16: "-bf16", inputs.PREC_FP32X: "-fp32x"}[prec]) + \
        (f"-grid{args.grid}" if args.grid else "") + ("-stable" if args.stencil == "stable" else "")
    if args.points:
        cfg["N"] = args.points
        cfg["Nb"] = max(1, args.points // 8)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as tdist

    from paper_2210_14907_b200 import nbm
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # NCCL logs its rank count / NVLS use to stderr
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    N, Nb = cfg["N"], cfg["Nb"]                 # per GPU (weak scaling)
    Ng, Nbg = N * world, Nb * world
    s = nbm.Solver(cfg, device=local, max_points=max(N, Nb))
    s.init_params(0)
    pts = torch.empty(N, 3, device="cuda")
    bpts = torch.empty(Nb, 3, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")   # > L2 (126 MB)
    stream = torch.cuda.current_stream()

    def step(it):
        s.sample(nbm.POINTS_INTERIOR, 0, it, rank * N, N, pts)
        s.sample(nbm.POINTS_BOUNDARY, 0, it, rank * Nb, Nb, bpts)
        s.loss_grad(pts, bpts, n_global=Ng, nb_global=Nbg, levels=args.levels)
        dp.allreduce_sum_(s.gbuf)
        s.adam_step(lr=cfg["lr"])

    for it in range(args.warmup):
        step(it)
    torch.cuda.synchronize()
    st = s.status()
    if st != 0:
        raise RuntimeError(f"device status {st} after warm-up")

    def barrier():
        if world > 1:
            tdist.barrier()
        torch.cuda.synchronize()

    def timed(fn, first_it):
        """K steps, CUDA events on the launching stream, L2 flushed between steps (untimed)"""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        barrier()
        with ClockSampler(local) as clk:
            for k in range(args.steps):
                flush.zero_()
                ev[k][0].record(stream)
                fn(first_it + k)
                ev[k][1].record(stream)
            barrier()
        return sum(a.elapsed_time(b) for a, b in ev), clk.summary()

    # eager pass: the library's event hook times the fused MLP kernel for the roofline
    nbm.nbm_timing_enable(s.h, True)
    nbm.nbm_timing_read(s.h)
    eager_ms, clk_eager = timed(step, args.warmup)
    launches_eager = nbm.nbm_last_launch_count(s.h) + 3          # + 2 samples + Adam
    mlp_ms, lg_ms, calls = nbm.nbm_timing_read(s.h)
    nbm.nbm_timing_enable(s.h, False)
    done = args.warmup + args.steps
    if args.no_graph:
        tot_ms, clocks, launches_per_step, mode = eager_ms, clk_eager, launches_eager, "eager"
    else:
        # the production step: one CUDA graph of [sample x2, loss_grad, Adam] on the device step
        # counter (two graphs around the NCCL all-reduce when N > 1), replayed per step
        s.t_dev.fill_(done)
        replay = s.capture_step(pts, bpts, first=rank * N, bfirst=rank * Nb, n_global=Ng, nb_global=Nbg,
                                lr=cfg["lr"], allreduce=dp.allreduce_sum_ if world > 1 else None, levels=args.levels)
        for _ in range(args.warmup):
            replay()
        tot_ms, clocks = timed(lambda it: replay(), 0)
        launches_per_step, mode = launches_eager + 1, "cuda-graph"   # Adam: prep + update
    if world > 1:
        t = torch.tensor([tot_ms, lg_ms, eager_ms], device="cuda", dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        tot_ms, lg_ms_max, eager_ms = t.tolist()
    else:
        lg_ms_max = lg_ms

    # ---- all-reduce time per step: the [grad, loss] collective alone,
    # CUDA events on the launching stream, max over ranks ----
    allreduce_us = None
    if world > 1:
        ar_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        for k in range(args.steps):
            ar_ev[k][0].record(stream)
            dp.allreduce_sum_(s.gbuf)
            ar_ev[k][1].record(stream)
        barrier()
        t = torch.tensor([sum(a.elapsed_time(b) for a, b in ar_ev) / args.steps], device="cuda", dtype=torch.float64)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        allreduce_us = t.item() * 1e3

    # ---- e2e: same step through the public API with host buffers (H2D of the step's
    # points from pinned memory, D2H of the loss) ----
    e2e = None
    if not args.no_e2e:
        # double-buffered inputs: step k+1's host->device copy runs on a copy stream while step k
        # computes; every step's copy and its loss read-back stay inside the timed region
        hp = torch.empty(N, 3, pin_memory=True)
        hb = torch.empty(Nb, 3, pin_memory=True)
        s.sample(nbm.POINTS_INTERIOR, 1, 0, rank * N, N, pts)
        s.sample(nbm.POINTS_BOUNDARY, 1, 0, rank * Nb, Nb, bpts)
        hp.copy_(pts)
        hb.copy_(bpts)
        hl = torch.empty(args.steps, pin_memory=True)
        dpts = [pts, torch.empty_like(pts)]
        dbps = [bpts, torch.empty_like(bpts)]
        cstream = torch.cuda.Stream()
        copied = [torch.cuda.Event() for _ in range(2)]
        used = [torch.cuda.Event() for _ in range(2)]
        ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]

        def issue_copy(k):   # inside the timed interval of step k - 1 (of step 0 for k = 0)
            b = k & 1
            cstream.wait_stream(stream)
            with torch.cuda.stream(cstream):
                if k >= 2:
                    cstream.wait_event(used[b])      # step k - 2 has consumed this buffer
                dpts[b].copy_(hp, non_blocking=True)
                dbps[b].copy_(hb, non_blocking=True)
                copied[b].record(cstream)

        barrier()
        for k in range(args.steps):
            flush.zero_()
            ee[k][0].record(stream)
            if k == 0:
                issue_copy(0)
            b = k & 1
            stream.wait_event(copied[b])
            if k + 1 < args.steps:
                issue_copy(k + 1)
            s.loss_grad(dpts[b], dbps[b], n_global=Ng, nb_global=Nbg, levels=args.levels)
            used[b].record(stream)
            dp.allreduce_sum_(s.gbuf)
            s.adam_step_at(lr=cfg["lr"])       # the device step counter, as in the timed graph
            hl[k:k + 1].copy_(s.loss, non_blocking=True)
            if k + 1 < args.steps:
                stream.wait_event(copied[(k + 1) & 1])   # step k+1's upload is counted in step k
            ee[k][1].record(stream)
        torch.cuda.synchronize()
        barrier()
        e_ms = sum(x.elapsed_time(y) for x, y in ee)
        if world > 1:
            t = torch.tensor([e_ms], device="cuda", dtype=torch.float64)
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            e_ms = t.item()
        e2e = {"value": Ng * args.steps / (e_ms / 1e3), "unit": "pts/s",
               "h2d_bytes_per_step": 12 * (N + Nb), "d2h_bytes_per_step": 4}
    # ---- inference at scale: nbm_eval of the surrogate pair at the
    # step's interior points (side by phi, one evaluation per point), device-resident inputs ----
    infer = None
    if args.eval:
        u = torch.empty(N, device="cuda")
        for _ in range(args.warmup):
            s.eval(pts, out=u)
        ie = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        barrier()
        for k in range(args.steps):
            flush.zero_()
            ie[k][0].record(stream)
            s.eval(pts, out=u)
            ie[k][1].record(stream)
        barrier()
        i_ms = sum(a.elapsed_time(b) for a, b in ie) / args.steps
        fwd_flop = 2.0 * mlp_macs(cfg["sizes"])[0] * N
        infer = {"pts_per_sec": N / (i_ms / 1e3), "ms_per_call": i_ms, "points": N,
                 "tflops": fwd_flop / (i_ms / 1e3) / 1e12}
    st = s.status()
    if st != 0:
        raise RuntimeError(f"device status {st} after the timed region")

    if rank != 0:
        if world > 1:
            tdist.destroy_process_group()
        return

    peaks, src = load_peaks()
    fwd, fb = mlp_macs(cfg["sizes"])
    # algorithmic FLOP of the fused-MLP launches of one step (levels x 7N stencil evaluations +
    # the N_b boundary evaluations of level 0), averaged per launch
    flop_launch = 2.0 * fb * (args.levels * 7 * N + Nb) / args.levels
    mlp_avg_s = mlp_ms / max(calls, 1) / 1e3
    if cfg["prec"] == inputs.PREC_FP32:
        peak = FP32_FFMA_TFLOPS
        bound, peak_note = "alu", "fp32 FFMA: 148 SM x 128 lanes x 2 FLOP x 1965 MHz (derived, DESIGN.md)"
    elif cfg["prec"] == inputs.PREC_FP32X:
        peak = peaks["bf16_tflops"] / 6.0
        bound, peak_note = "tensor", (f"bf16 dense ({src}, MEASURED_PEAKS.json) / 6: each fp32-accurate product is six "
                                      "bf16 plane products (G26)")
    else:
        peak = peaks["bf16_tflops"]
        bound, peak_note = "tensor", f"bf16 dense, {src} (MEASURED_PEAKS.json)"
    achieved = flop_launch / mlp_avg_s / 1e12
    # secondary bound: the MUFU ceiling, one transcendental per hidden activation of
    # the forward, 16 per clock per SM (B200 MUFU; accurate fp32 tanhf costs more than one)
    acts_launch = sum(cfg["sizes"][1:-1]) * (args.levels * 7 * N + Nb) / args.levels
    mufu_ms = acts_launch / (148 * 16 * 1.965e9) * 1e3
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{cfg['label']}.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("bytes_per_launch")
    val = Ng * args.steps / (tot_ms / 1e3)
    line = {
        "metric": METRIC,
        "value": val, "unit": "pts/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_ms / args.steps, "steps_per_sec": 1e3 * args.steps / tot_ms,
        "loss_grad_pts_per_sec": Ng * calls / args.levels / (lg_ms_max / 1e3) if calls else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": {inputs.PREC_FP32: "f32", inputs.PREC_BF16: "bf16",
                  inputs.PREC_FP32X: "f32 (3-plane bf16 split on tcgen05, f32 accumulate)"}[cfg["prec"]],
        "data": "synthetic (seeded Philox lattice points; manufactured two-phase Poisson)",
        "config": {"workload": cfg["label"], "points_per_gpu": N, "boundary_per_gpu": Nb,
                   "global_points": Ng, "mlp": "x".join(map(str, cfg["sizes"])), "n_nets": cfg["n_nets"],
                   "h": cfg["h"], "levels": args.levels, "stencil": args.stencil, "parallelism": f"dp{world}", "l2": "flushed between steps (256 MiB write)"},
        "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     **({"peak_sustained": peaks["bf16_tflops_sustained"],
                         "frac_sustained": achieved / peaks["bf16_tflops_sustained"]}
                        if cfg["prec"] == inputs.PREC_BF16 else {}),
                     **({"measured_ffma_3reg_peak": FP32_FFMA_3REG_MEASURED_TFLOPS,
                         "frac_of_measured_ffma": achieved / FP32_FFMA_3REG_MEASURED_TFLOPS}
                        if cfg["prec"] in (inputs.PREC_FP32, inputs.PREC_FP32X) else {}),
                     "frac": achieved / peak, "traffic": traffic, "kernel": kernel_name(cfg) + " fused fwd/residual/bwd",
                     "flop_per_launch": flop_launch, "avg_launch_ms": mlp_avg_s * 1e3,
                     "share_of_step": mlp_ms / eager_ms, "peak_src": peak_note,
                     "secondary": {"bound": "mufu", "activations_per_launch": acts_launch,
                                   "t_ms": mufu_ms, "frac": mufu_ms / (mlp_avg_s * 1e3),
                                   "peak_src": "148 SM x 16 MUFU/clk x 1965 MHz (derived)"}},
        "gpu_launches": launches_per_step * args.steps,
        "launch_mode": mode, "ms_per_step_eager": eager_ms / args.steps,
        "clocks": clocks,
        "e2e": e2e,
        "allreduce_us_per_step": allreduce_us,
        **({"nccl": {"ranks": world, "backend": tdist.get_backend()}} if world > 1 else {}),
    }
    if infer is not None:
        line["inference"] = infer
    if not args.no_cpu_baseline and world == 1:   # the oracle baseline: rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline(cfg, levels=args.levels)
    if cfg["name"] == "c4" and not args.no_secondary and world == 1 and args.points is None:
        s.close()
        del flush
        torch.cuda.empty_cache()
        line["secondary"] = run_secondary(args)
    print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
