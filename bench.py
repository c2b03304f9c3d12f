#!/usr/bin/env python
"""bench.py -- NUFFT points/s of the B200 hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2b] [--impl ours|reference]

One STEP = one pass of the whole hot path over one batch of synthetic input
(SURVEY.md §8a): setpts (fold + bin-sort), type-1 NUFFT (spread, FFT,
truncate+deconvolve) and type-2 NUFFT (pre-correct+pad, FFT, interpolate).
value = points of all ranks / device time per step (points/s), inputs resident
in HBM; L2 is flushed (a 512 MB write) before every timed step, outside the
timed events.  `e2e` is the same metric through the C ABI with pinned HOST
buffers (H2D of x, y, z, c, fk and D2H of fk, c inside the timed region).

Default workload = the metric's configuration, BASELINE.json configs[3] (C4):
fp64, 512^3 modes, 2^30 = 1.07e9 Landau-perturbed points on [0, 4 pi)^3, eps =
1e-4 -- the NUFFT step over the PIF particles; the line also carries the PIF
seconds per step of the same configuration (`pif`).  `--config c2b | c3 | ...`
selects the other BASELINE configs.  N > 1 (torchrun): the SAME workload on a z-slab
plan over NCCL ("scaling": "strong"): each rank starts with Np/N points drawn
over the whole domain (setpts redistributes them to their slab owners), halos
are exchanged with the z-neighbours and the slab FFT transposes with
ncclAlltoAll; value = all points / max-over-ranks device time per step.

--impl reference: the CPU oracle (oracle/, plain C++ fp64) on the same config,
rank 0 only, each step a bounded sample of the workload (the same point density
and eps on a 1/64 box: 128^3 modes, 2^24 points for C4; see ref_sample()).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

CONFIGS = {
    # the metric's configuration (BASELINE.json configs[3]): the
    # 512^3-mode Landau workload as a NUFFT step -- fp64, 2^30 = 1.07e9 Landau-perturbed
    # points on [0, 4 pi)^3 (8 per mode), eps = 1e-4.  The default bench line.
    "c4n": dict(name="C4", prec="f64", N=(512, 512, 512), Np=8 * 512 ** 3, eps=1e-4,
                kind="landau", L=4 * math.pi, pif="c4"),
    "c1": dict(name="C1", prec="f64", N=(32, 32, 32), Np=100_000, eps=1e-6, kind="uniform"),
    "c2a": dict(name="C2a", prec="f32", N=(128, 128, 128), Np=1 << 21, eps=1e-4, kind="uniform"),
    "c2b": dict(name="C2b", prec="f32", N=(128, 128, 128), Np=1 << 21, eps=1e-6, kind="uniform"),
    "c3": dict(name="C3", prec="f64", N=(256, 256, 256), Np=8 * 256 ** 3, eps=1e-6,
               kind="uniform"),
    "c3e4": dict(name="C3", prec="f64", N=(256, 256, 256), Np=8 * 256 ** 3, eps=1e-4,
                 kind="uniform"),
    # Landau-damping PIF step: 512^3 modes, 8 particles per mode,
    # fp64, eps = 1e-4, dt = 0.01; metric = seconds per PIF step
    "c4": dict(name="C4", prec="f64", N=(512, 512, 512), Np=8 * 512 ** 3, eps=1e-4,
               kind="pif", dt=0.01),
    # the paper's high-accuracy PIF run: eps = 1e-8, dt = 0.003125
    "c4e8": dict(name="C4-1e-8", prec="f64", N=(512, 512, 512), Np=8 * 512 ** 3, eps=1e-8,
                 kind="pif", dt=0.003125),
    # small PIF for quick checks
    "pif128": dict(name="PIF-128", prec="f64", N=(128, 128, 128), Np=8 * 128 ** 3, eps=1e-4,
                   kind="pif", dt=0.01),
}
OUR_KERNELS_PER_STEP = 9  # bin_count, 3 scan, scatter | spread, truncate_deconv | pad, interp


def kernels_per_step(info, ws):
    """Our kernel launches per setpts + type 1 + type 2 (cuFFT's own not counted):
    bin_count, 3 scan phases, scatter, [weights] | spread, truncate_deconv | pad,
    interp; a slab plan adds 2 halo adds and the x/y pack + unpad instead of the
    single-GPU truncate / pad (z_deconv, z_pad take their places)."""
    n = OUR_KERNELS_PER_STEP + (1 if info.get("weights_precomputed") else 0)
    n += 1 if info.get("sub_bins", 1) > 1 else 0  # sub-bin plans: the per-bin offset gather
    return n + (4 if ws > 1 else 0)
REF_SAMPLE = 1 << 19


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_inputs(cfg, rank, ws, device, mode_block=None):
    """This rank's share of the workload.  The global problem is the same at every N
    (strong scaling): Np points (uniform or Landau, seed 1), strengths (seed 2) and
    modes (seed 3).  With N > 1 ranks every rank keeps the points whose fine z-cell
    lies in its slab -- particles partitioned like the grid -- and
    its block of the modes; the plan is told so (opts.points_owned)."""
    import synthetic
    rdt = torch.float64 if cfg["prec"] == "f64" else torch.float32
    cdt = torch.complex128 if cfg["prec"] == "f64" else torch.complex64
    Np = cfg["Np"]
    pts = gen_points(cfg, Np, device, rdt)
    c = synthetic.strengths(Np, seed=2, device=device, dtype=cdt)
    if ws > 1:
        L = cfg.get("L", 2 * math.pi)
        nf3 = 2 * cfg["N"][2]
        # the library's owner rule: floor(z nf3 / L) (fp64, z in [0, L)) // (nf3 / ws)
        cell = torch.floor(pts[2].double() * (nf3 / L)).clamp_(max=nf3 - 1)
        mine = torch.div(cell, nf3 // ws, rounding_mode="floor") == rank
        pts = tuple(p[mine].contiguous() for p in pts)
        c = c[mine].contiguous()
    fk = synthetic.modes(*cfg["N"], seed=3, device=device, dtype=cdt)
    if mode_block is not None:
        lo, hi = mode_block
        fk = fk[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]].contiguous()
    return pts, c, fk


def algorithmic_bytes(cfg, stage):
    """spread / interp move perm (4 B) + 3 coordinates + one strength
    per point and the fine grid once: Np (4 + 5 r) + nf^3 2 r bytes per launch."""
    r = 8 if cfg["prec"] == "f64" else 4
    nf3 = 8 * cfg["N"][0] * cfg["N"][1] * cfg["N"][2]
    if stage in ("spread", "interp"):
        return cfg["Np"] * (4 + 5 * r) + nf3 * 2 * r
    raise ValueError(stage)


def algorithmic_flops(cfg, w, real=False):
    """Per launch of spread or interp: per point one value x weight
    multiply-add per stencil cell -- 4 w^3 flops complex, 2 w^3 real -- plus the 3 w^2
    products of the separable weights (the 3 w ES evaluations are not counted)."""
    per = (2 if real else 4) * w ** 3 + 3 * w ** 2
    return cfg["Np"] * per


_PEAK_CACHE = {}


def alu_peak_tflops(prec):
    """FMA-pipe peak of THIS GPU, measured by nufft_fma_peak (8 independent FMA chains
    per thread, 8 x 256 threads per SM; the best of three runs).  The datasheet figure
    for comparison: 148 SMs x 128 (fp32) / 64 (fp64) FMA lanes x 2 x 1965 MHz."""
    if prec not in _PEAK_CACHE:
        import paper_2605_10678_b200 as nb
        _PEAK_CACHE[prec] = max(nb.fma_peak(prec) for _ in range(3))
    return _PEAK_CACHE[prec]


def roofline_obj(cfg, dom, dom_ms, ws, w, real, traffic):
    """The dominant kernel against its binding roofline: the spread / interp are bound
    by the FMA pipes and shared memory (profiles/README.md: FP64 pipe 59 % busy at C3,
    fp32 issue 63 % at C2b, DRAM 4-5 %) -> bound "alu"; the north_star's HBM fraction
    of the same launch is reported alongside."""
    hbm, peak_src = peaks()
    bytes_alg = algorithmic_bytes(cfg, dom) / ws
    gbs = bytes_alg / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
    flops = algorithmic_flops(cfg, w, real) / ws
    tfs = flops / (dom_ms / 1e3) / 1e12 if dom_ms > 0 else 0.0
    peak = alu_peak_tflops(cfg["prec"])
    return {"kernel": dom, "bound": "alu", "achieved": tfs, "peak": peak, "unit": "TFLOP/s",
            "frac": tfs / peak,
            "peak_source": f"measured live: nufft_fma_peak ({cfg['prec']} FMA chains, this GPU); "
                           f"datasheet {148 * (64 if cfg['prec'] == 'f64' else 128) * 2 * 1.965e-3:.1f}",
            "traffic": traffic, "algorithmic_flops_per_launch": flops,
            "flops_per_point": (2 if real else 4) * w ** 3 + 3 * w ** 2,
            "ms_per_launch": dom_ms,
            "hbm": {"achieved": gbs, "peak": hbm, "peak_source": peak_src, "unit": "GB/s",
                    "frac": gbs / hbm, "algorithmic_bytes_per_launch": bytes_alg}}


def source_sha():
    """sha256 (16 hex) of the CUDA / C++ sources of libnufft: a committed ncu traffic
    figure is reported only while the kernels it measured are unchanged."""
    import hashlib
    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_2605_10678_b200", "csrc")
    for f in sorted(os.listdir(d)):
        if f.endswith((".cu", ".cuh", ".h", ".cpp")):
            with open(os.path.join(d, f), "rb") as fh:
                h.update(f.encode() + fh.read())
    return h.hexdigest()[:16]


def load_traffic(cfg_key, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu
    capture (profiles/traffic.json), or None if the sources changed since."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            t = json.load(f)
        e = t[cfg_key][kernel]
        if isinstance(e, dict):
            return e["bytes"] if e.get("src_sha") == source_sha() else None
        return None
    except Exception:
        return None


def run_ours(args, cfg):
    import paper_2605_10678_b200 as nb
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    stream = torch.cuda.current_stream(device)

    N, Np_total = cfg["N"], cfg["Np"]
    comm = nb.Comm() if ws > 1 else None   # z-slab plan over NCCL
    plan = nb.Plan(N, cfg["eps"], precision=cfg["prec"], timing=True, device=device,
                   tile=args.tile, spread_warps=args.spread_warps, comm=comm,
                   points_owned=ws > 1, interp_method=args.interp_method,
                   precompute=args.precompute, L=cfg.get("L", 2 * math.pi),
                   fft_method=args.fft_method if ws == 1 else 0)
    pts, c, fk = make_inputs(cfg, rank, ws, device, plan.local_modes() if ws > 1 else None)
    Np = pts[0].numel()
    if args.real:  # real strengths / outputs: the R2C / C2R path
        if ws > 1:
            raise SystemExit("--real is single-GPU only")
        c = c.real.contiguous()
    c2 = torch.empty(Np, dtype=c.dtype, device=device)
    fk_out = torch.empty_like(fk)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=device)
    t1 = plan.type1_real if args.real else plan.type1
    t2 = plan.type2_real if args.real else plan.type2

    def step():
        plan.setpts(*pts)
        t1(c, out=fk_out)
        t2(fk, out=c2)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    stage = {k: [] for k in ("ms_setpts", "ms_spread", "ms_fft", "ms_deconv", "ms_pad",
                             "ms_interp", "ms_comm")}
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(k & 0xff)                      # evict L2 (outside the timed events)
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
        info = plan.info()                         # syncs; per-stage events of this step
        for key in stage:
            stage[key].append(info[key])
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    t_max = t_ms
    if ws > 1:
        t = torch.tensor([t_ms], device=device, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_max = float(t.item())
    ms_per_step = t_max / args.steps
    value = Np_total / (ms_per_step / 1e3)   # all ranks' points per second

    # -- N > 1: setpts WITH redistribution, timed on its own (points handed out round
    # robin, so (P-1)/P of them move: owner counts, count all-to-all, one host sync,
    # grouped send / recv of x, y, z, then the local sort) -- PAPER.md:229-235
    redist = None
    if ws > 1 and not args.no_redist:
        del pts
        torch.cuda.empty_cache()
        plan_r = nb.Plan(N, cfg["eps"], precision=cfg["prec"], timing=True, device=device,
                         tile=args.tile, spread_warps=args.spread_warps, comm=comm,
                         points_owned=False, L=cfg.get("L", 2 * math.pi))
        import synthetic
        rdt = torch.float64 if cfg["prec"] == "f64" else torch.float32
        allp = gen_points(cfg, Np_total, device, rdt)
        rr = tuple(a[rank::ws].contiguous() for a in allp)
        del allp
        torch.cuda.empty_cache()
        plan_r.setpts(*rr)  # warm-up (allocations)
        torch.cuda.synchronize()
        torch.distributed.barrier()
        nrep = max(2, min(args.steps, 5))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(nrep):
            plan_r.setpts(*rr)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / nrep], device=device, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        redist = {"ms": float(t.item()), "moved_fraction": (ws - 1) / ws,
                  "what": "setpts of points handed out round robin (owner counts, NCCL count "
                          "all-to-all, host sync, grouped send/recv of x, y, z, local sort); "
                          "max over ranks"}
        plan_r.close()
        del rr
        torch.cuda.empty_cache()
        pts, _, _ = make_inputs(cfg, rank, ws, device, plan.local_modes())

    # -- end to end through the C ABI with pinned host buffers (the device copies of
    # the inputs are released first: the plan stages host arrays in its own buffers)
    def pinned(t):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h
    hp = [pinned(p) for p in pts]
    hc = pinned(c)
    hfk = pinned(fk)
    hfk_out = torch.empty(fk.shape, dtype=fk.dtype, pin_memory=True)
    hc2 = torch.empty(Np, dtype=c.dtype, pin_memory=True)
    fk_shape, c_dtype, nmodes = fk.shape, c.dtype, fk.numel()
    del pts, c, fk, c2, fk_out, flush
    torch.cuda.empty_cache()

    def e2e_step():
        plan.setpts(*hp)
        t1(hc, out=hfk_out)
        t2(hfk, out=hc2)

    e2e_steps = max(3, min(args.steps, 20 if Np_total <= (1 << 24) else 5))
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    te = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([te], device=device, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        te = float(t.item())
    r = 8 if cfg["prec"] == "f64" else 4
    cr = 1 if args.real else 2  # reals per strength / output value
    h2d = 3 * Np * r + Np * cr * r + nmodes * 2 * r
    d2h = nmodes * 2 * r + Np * cr * r
    if ws > 1:  # whole-job bytes
        tot = torch.tensor([h2d, d2h], device=device, dtype=torch.float64)
        torch.distributed.all_reduce(tot)
        h2d, d2h = int(tot[0].item()), int(tot[1].item())

    # -- roofline of the dominant kernel of ours (spread or interp)
    med = {k: statistics.median(v) for k, v in stage.items() if v and min(v) >= 0}
    dom = "spread" if med.get("ms_spread", 0) >= med.get("ms_interp", 0) else "interp"
    dom_ms = med["ms_" + dom]
    info = plan.info()
    roof = roofline_obj(cfg, dom, dom_ms, ws, info["w"], args.real, load_traffic(args.config, dom))
    plan.close()
    del hp, hc, hfk, hfk_out, hc2
    torch.cuda.empty_cache()
    # the PIF seconds per step of the same configuration (BASELINE metric, 2nd part)
    pif = None
    if cfg.get("pif") and not args.no_pif:
        pargs = argparse.Namespace(**vars(args))
        pargs.steps, pargs.warmup, pargs.no_cpu_baseline = min(args.steps, 10), 3, True
        pif = run_pif(pargs, CONFIGS[cfg["pif"]], comm=comm, inner=True)
    out = None
    if rank == 0:
        cpu = cpu_baseline(cfg) if (ws == 1 and not args.no_cpu_baseline) else None
        out = {
            "metric": "NUFFT points/s (setpts + type-1 spread + type-2 interp per point)",
            "value": value, "unit": "points/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if cfg["prec"] == "f64" else "f32", "data": "synthetic",
            "config": {"workload": f"{cfg['name']}: {cfg['prec']} {N[0]}x{N[1]}x{N[2]} modes, "
                                   f"{Np_total} {cfg['kind']} points, eps={cfg['eps']:g}",
                       "N": list(N), "Np_total": Np_total, "eps": cfg["eps"],
                       "L": cfg.get("L", 2 * math.pi),
                       "w": info["w"], "precision": cfg["prec"], "points": cfg["kind"],
                       "tile": info["tile"],
                       "kernels": {"spread_warps": args.spread_warps, "fft_method": args.fft_method,
                                   "interp_method": args.interp_method,
                                   "weights_precomputed": info["weights_precomputed"]},
                       "values": "real (R2C / C2R)" if args.real else "complex",
                       "parallelism": (f"z-slab x{ws} (points owned by slab, NCCL halos + "
                                       f"all-to-all)") if ws > 1 else "1 GPU",
                       "l2": "flushed (512 MB write) before every timed step"},
            "stage_ms_median": med,
            "e2e": {"value": Np_total / (te / e2e_steps / 1e3), "unit": "points/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": te / e2e_steps},
            "gpu_launches": kernels_per_step(info, ws) * args.steps,
            "roofline": roof,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        if pif is not None:
            out["pif"] = pif
        if redist is not None:
            out["setpts_redistribute"] = redist
    if ws > 1:
        comm.close()
        torch.distributed.destroy_process_group()
    return out


def ref_sample(cfg):
    """The bounded sample of a workload that the CPU oracle runs (cpu_baseline and the
    --impl reference arm): workloads of <= 2^22 points keep their modes and take 2^19
    of the points; larger ones (C3, C4) keep the point distribution, the points per mode
    and eps on 128^3 modes (C3: 1/8, C4: 1/64 of the problem) -- the oracle's per-point
    work is that of the full workload (same w, same density), its FFT share smaller."""
    N, Np = cfg["N"], cfg["Np"]
    if Np <= (1 << 22):
        n = min(Np, REF_SAMPLE)
        return dict(N=N, Np=n, desc=f"{n} {cfg['kind']} points of the {cfg['name']} workload "
                                    f"({N[0]}^3 modes, eps={cfg['eps']:g})")
    Ns = tuple(128 for _ in N)
    n = Np * (128 ** 3) // (N[0] * N[1] * N[2])
    return dict(N=Ns, Np=n, desc=f"the {cfg['name']} workload on a 1/{Np // n} box: {Ns[0]}^3 "
                                 f"modes, {n} {cfg['kind']} points ({Np // (N[0] * N[1] * N[2])} "
                                 f"per mode), eps={cfg['eps']:g}")


def gen_points(cfg, Np, device, rdt):
    """The config's point distribution (seeded, synthetic/): Landau-perturbed,
    uniform, or -- with --points clustered -- Gaussian blobs (a setpts contention and
    load-imbalance stress case, not a paper workload)."""
    import synthetic
    if cfg["kind"] == "landau":
        return synthetic.landau_points(Np, seed=1, device=device, dtype=rdt)
    if cfg["kind"] == "clustered":
        return synthetic.clustered_points(Np, L=cfg.get("L", 2 * math.pi), device=device,
                                          dtype=rdt)
    return synthetic.uniform_points(Np, seed=1, device=device, dtype=rdt)


def sample_inputs(cfg, smp):
    import synthetic
    x, y, z = (v.numpy() for v in gen_points(cfg, smp["Np"], "cpu", torch.float64))
    c = synthetic.strengths(smp["Np"]).numpy()
    fk = synthetic.modes(*smp["N"]).numpy()
    return x, y, z, c, fk


def cpu_baseline(cfg):
    """The oracle as it stands, on a bounded sample of the workload, all host cores."""
    import oracle
    smp = ref_sample(cfg)
    L = cfg.get("L", 2 * math.pi)
    t0 = time.perf_counter()
    x, y, z, c, fk = sample_inputs(cfg, smp)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.type1(x, y, z, c, smp["N"], cfg["eps"], L=L)
    oracle.type2(x, y, z, fk, cfg["eps"], L=L)
    t = time.perf_counter() - t0
    return {"value": smp["Np"] / t, "unit": "points/s", "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": smp["desc"] + "; one type-1 + one type-2 in fp64 (no setpts: the oracle "
                                    "has no sort)",
            "seconds": t, "input_gen_seconds": t_gen}


def run_pif(args, cfg, comm=None, inner=False):
    """Seconds per Landau-damping PIF step: sort, type-1 charge
    scatter, Poisson, three type-2 field gathers + kicks, drift -- all on device.
    inner=True: called from run_ours (process group and comm exist); returns the
    compact `pif` object of the NUFFT line."""
    import paper_2605_10678_b200 as nb
    from paper_2605_10678_b200.pif import LandauPIF
    ws, rank, local = dist_env()
    if ws > 1 and not inner:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    stream = torch.cuda.current_stream(device)
    if not inner:
        comm = nb.Comm() if ws > 1 else None
    sim = LandauPIF(cfg["N"], cfg["Np"], eps=cfg["eps"], dt=cfg["dt"], precision=cfg["prec"],
                    comm=comm, device=device, timing=True, tile=args.tile,
                    spread_warps=args.spread_warps, fused=getattr(args, 'pif_fused', False))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=device)
    for _ in range(args.warmup):
        sim.step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    stage = {k: [] for k in ("ms_setpts", "ms_spread", "ms_fft", "ms_deconv", "ms_pad",
                             "ms_interp", "ms_comm")}
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(k & 0xff)
        evs[k][0].record(stream)
        sim.step()
        evs[k][1].record(stream)
        info = sim.plan.info()   # last call of each stage (interp: the z-component gather)
        for key in stage:
            stage[key].append(info[key])
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    if ws > 1:
        t = torch.tensor([t_ms], device=device, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_ms = float(t.item())
    ms_per_step = t_ms / args.steps
    # e2e: the same step through the public API plus the D2H read of its result
    # (the field-energy diagnostic); the particle state stays resident, so no H2D
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        torch.distributed.barrier()
    e2e_steps = max(2, min(args.steps, 5))
    e0.record(stream)
    for _ in range(e2e_steps):
        sim.step()
        sim.field_energy()
    e1.record(stream)
    torch.cuda.synchronize()
    te = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([te], device=device, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        te = float(t.item())
    med = {k: statistics.median(v) for k, v in stage.items() if v and min(v) >= 0}
    if inner:
        info = sim.plan.info()
        sim.plan.close()
        del sim
        torch.cuda.empty_cache()
        return {"metric": "seconds per Landau-damping PIF step", "value": ms_per_step / 1e3,
                "unit": "s/step", "steps": args.steps, "warmup": args.warmup,
                "higher_is_better": False,
                "workload": f"{cfg['name']}: PIF Landau damping, {cfg['N'][0]}^3 modes, "
                            f"{cfg['Np']} particles, eps={cfg['eps']:g}, dt={cfg['dt']}, "
                            "real-valued transforms", "w": info["w"],
                "stage_ms_median": med, "clocks": clocks,
                "e2e": {"value": te / e2e_steps / 1e3, "unit": "s/step",
                        "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 8}}
    # dominant kernel per step: spread once, interp three times
    sp, ip = med.get("ms_spread", 0.0), 3 * med.get("ms_interp", 0.0)
    dom, dom_ms = ("spread", sp) if sp >= ip else ("interp", med.get("ms_interp", 0.0))
    out = None
    if rank == 0:
        N = cfg["N"]
        cpu = pif_cpu_baseline() if (ws == 1 and not args.no_cpu_baseline) else None
        out = {
            "metric": "seconds per Landau-damping PIF step", "value": ms_per_step / 1e3,
            "unit": "s/step", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if cfg["prec"] == "f64" else "f32",
            "data": "synthetic",
            "config": {"workload": f"{cfg['name']}: PIF Landau damping, {N[0]}^3 modes, "
                                   f"{cfg['Np']} particles (8 per mode), eps={cfg['eps']:g}, "
                                   f"dt={cfg['dt']}", "N": list(N), "Np_total": cfg["Np"],
                       "w": sim.plan.info()["w"], "tile": sim.plan.info()["tile"],
                       "parallelism": f"z-slab x{ws} (NCCL)" if ws > 1 else "1 GPU",
                       "l2": "flushed (512 MB write) before every timed step"},
            "stage_ms_median": med,
            "e2e": {"value": te / e2e_steps / 1e3, "unit": "s/step", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 8,
                    "note": "state resident on device; field-energy scalar read back per step"},
            # setpts 5 [+ weights] | spread, truncate | poisson | 3 x (pad, interp, kick) |
            # drift; a slab plan adds 2 halo adds, the x/y pack / unpads and migration (6)
            "gpu_launches": (18 + (1 if sim.plan.info().get("weights_precomputed") else 0)
                             + (12 if ws > 1 else 0)) * args.steps,
            "roofline": roofline_obj(cfg, dom, dom_ms, ws, sim.plan.info()["w"], sim.real,
                                     load_traffic(args.config, dom)),
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
    sim.plan.close()
    if ws > 1:
        comm.close()
        torch.distributed.destroy_process_group()
    return out


def pif_cpu_baseline():
    """The oracle PIF step (oracle type 1 + 3 type 2, numpy Poisson / push) on a
    bounded sample: 32^3 modes, 8 particles per mode."""
    import numpy as np
    import oracle
    import synthetic
    N, Np, eps, dt, L = (32, 32, 32), 8 * 32 ** 3, 1e-4, 0.01, 4 * math.pi
    x, y, z = (t.numpy() for t in synthetic.landau_points(Np))
    v = [t.numpy().copy() for t in synthetic.maxwellian_velocities(Np)]
    c = np.full(Np, -L ** 3 / Np, dtype=np.complex128)
    t0 = time.perf_counter()
    rho = oracle.type1(x, y, z, c, N, eps, L=L)
    n = [np.arange(N[d]) - N[d] // 2 for d in range(3)]
    ks = [(2 * math.pi / L) * n[0][None, None, :], (2 * math.pi / L) * n[1][None, :, None],
          (2 * math.pi / L) * n[2][:, None, None]]
    kk = ks[0] ** 2 + ks[1] ** 2 + ks[2] ** 2
    inv = np.where(kk > 0, 1.0 / np.where(kk > 0, kk, 1.0), 0.0)
    inv[0, :, :] = inv[:, 0, :] = inv[:, :, 0] = 0.0   # no field on the Nyquist planes (R15)
    for d in range(3):
        e = oracle.type2(x, y, z, -1j * ks[d] * rho * inv, eps, L=L)
        v[d] += -dt * e.real / L ** 3
    x, y, z = (np.mod(a + vd * dt, L) for a, vd in zip((x, y, z), v))
    t = time.perf_counter() - t0
    return {"value": t, "unit": "s/step", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"one oracle PIF step at 32^3 modes, {Np} particles (8 per mode), "
                      "eps=1e-4 (the 512^3 workload does not fit the oracle's budget)"}


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    import oracle
    import synthetic
    if cfg["kind"] == "pif":   # oracle PIF steps on the bounded sample of pif_cpu_baseline
        for _ in range(args.warmup):
            pif_cpu_baseline()
        ts = [pif_cpu_baseline() for _ in range(args.steps)]
        v = statistics.median(t["value"] for t in ts)
        return {"impl": "reference", "metric": "seconds per Landau-damping PIF step", "value": v,
                "unit": "s/step", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": v * 1e3, "higher_is_better": False, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": cfg["name"], "sample": ts[0]["sample"]},
                "cpu_baseline": ts[0],
                "e2e": {"value": v, "unit": "s/step", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
    smp = ref_sample(cfg)
    L = cfg.get("L", 2 * math.pi)
    x, y, z, c, fk = sample_inputs(cfg, smp)

    def step():
        oracle.type1(x, y, z, c, smp["N"], cfg["eps"], L=L)
        oracle.type2(x, y, z, fk, cfg["eps"], L=L)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    t = (time.perf_counter() - t0) / args.steps
    v = smp["Np"] / t
    N = cfg["N"]
    return {
        "impl": "reference", "metric": "NUFFT points/s (setpts + type-1 spread + type-2 interp per point)",
        "value": v, "unit": "points/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg['name']}: {cfg['prec']} {N[0]}x{N[1]}x{N[2]} modes, "
                               f"{cfg['Np']} {cfg['kind']} points, eps={cfg['eps']:g}",
                   "sample": smp["desc"]},
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": oracle.num_threads(),
                         "kind": "oracle",
                         "sample": smp["desc"] + " per step (oracle type-1 + type-2, fp64)"},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4n", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pif", action="store_true", help="skip the PIF s/step key of the c4n line")
    ap.add_argument("--no-redist", action="store_true",
                    help="N > 1: skip the setpts-with-redistribution timing")
    ap.add_argument("--pif-fused", action="store_true",
                    help="PIF: one three-field gather with the kick fused (nufft_pif_gather_kick)")
    ap.add_argument("--tile", default=None, help="bin edge T or Tx,Ty,Tz (default: built-in table)")
    ap.add_argument("--spread-warps", type=int, default=0,
                    help="spread kernel: 1 rows, 2 outer products, 4 / 8 smem planes (default: built-in)")
    ap.add_argument("--precompute", type=int, default=0,
                    help="per-point ES weight table: 0 auto (fp64), 1 always, -1 never")
    ap.add_argument("--fft-method", type=int, default=0,
                    help="1: the paper's pruned sigma = 2 FFT (eight N^3 parity sub-grid FFTs)")
    ap.add_argument("--interp-method", type=int, default=0,
                    help="ablation: 1 / 2 = the paper's Direct Interpolation, caller / sorted order")
    ap.add_argument("--points", default=None, choices=["clustered"],
                    help="NUFFT configs: replace the config's point distribution (stress case)")
    ap.add_argument("--real", action="store_true",
                    help="NUFFT configs: real strengths / outputs (R2C / C2R transforms)")
    args = ap.parse_args()
    if args.tile is not None:
        t = [int(v) for v in args.tile.split(",")]
        args.tile = tuple(t * 3 if len(t) == 1 else t)
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.points and cfg["kind"] != "pif":
        cfg = dict(cfg, kind=args.points)
    if args.impl == "reference":
        out = run_reference(args, cfg)
    elif cfg["kind"] == "pif":
        out = run_pif(args, cfg)
    else:
        out = run_ours(args, cfg)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
