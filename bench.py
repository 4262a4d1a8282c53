#!/usr/bin/env python
"""bench.py -- GPts/s of the acoustic FD forward on BASELINE configs[1] (3D 256^3
physical + 40-pt absorbing layer = 336^3 computational grid, space order 8, nt=1000,
two-layer model, 15 Hz Ricker at the surface centre, 256x256 surface receivers).

One "step" = one complete forward propagation (nt-1 = 999 leapfrog updates of every
grid point, each with source injection and receiver interpolation) through the C-ABI
(sf_forward) from a zero initial state.  value = N_points * (nt-1) * steps * n_gpus /
max-over-ranks device time  [GPts/s = 1e9 grid-point updates per second].

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): weak scaling -- the grid is slab-decomposed along x
with 336 planes per rank (global 336N x 336 x 336) and r=4 halo planes exchanged every
step with NCCL send/recv.  With --config 4 (multi-shot FWI gradient) each rank instead
runs its own shot on the full 400^3 model and every step ends with the NCCL all-reduce
of the gradient (sf_allreduce_gradient) -- weak scaling by shots.  --impl reference runs the fp64 CPU oracle (the only
"reference" this paper-only build has) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GPts/s (grid-point updates/s) at 1/2/4/8 B200, % of HBM roofline"
UNIT = "GPts/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


NCU_ROUND = "r02"


def ncu_traffic(cfg):
    """Per-launch DRAM bytes (read + write) of the stencil kernel on this config from the
    committed ncu --set full capture summary (profiles/<round>_stencil_ncu_c<cfg>.json,
    written by scripts/ncu_summary.py), or None when that config was not captured."""
    # gradient configs: per-mode traffic weighted to the average update of the full config
    # (scripts/ncu_step_traffic.py), the same average as the line's algorithmic bytes
    rel = os.path.join("profiles", f"{NCU_ROUND}_step_traffic_c{cfg}.json")
    if not os.path.exists(os.path.join(ROOT, rel)):
        rel = os.path.join("profiles", f"{NCU_ROUND}_stencil_ncu_c{cfg}.json")
    try:
        with open(os.path.join(ROOT, rel)) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), rel
    except Exception:
        return None, rel


class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"clocks_{os.getpid()}.csv")

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
             "clocks.mem,power.limit")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons, pw, mem, plim = [], None, set(), [], [], None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                c = [x.strip() for x in line.split(",")]
                if len(c) < 9:
                    continue
                try:
                    sm.append(float(c[1]))
                    smax = float(c[2])
                except ValueError:
                    continue
                for nm, v in zip(names, c[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
                try:
                    pw.append(float(c[3]))
                    mem.append(float(c[9]))
                    plim = float(c[10])
                except (ValueError, IndexError):
                    pass
        med = lambda a: statistics.median(a) if a else None
        return {"sm_mhz": med(sm), "sm_max_mhz": smax, "mem_mhz": med(mem), "power_w": med(pw),
                "power_limit_w": plim, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- workload
def build_problem(nt_override=None, rank=0, nranks=1, cfg=1, strong=False):
    """(problem, local m, local eta, global shape).  N > 1 splits the grid into x-slabs
    (configs[1] / configs[3]) or runs one shot per rank (configs[4])."""
    import synth
    if cfg == 4:
        # multi-shot FWI gradient (BASELINE configs[4]): one shot per rank on the
        # full 400^3 model, gradients summed by sf_allreduce_gradient -- weak scaling by shots
        p = synth.make_config(cfg, nt=nt_override, shot=rank)
        return p, p.m, p.damp, p.shape
    p = synth.make_config(cfg, nt=nt_override)
    if nranks == 1:
        return p, p.m, p.damp, p.shape
    if cfg not in (1, 3):
        raise SystemExit("multi-GPU bench: configs[1] / configs[3] slab-decomposed (weak, or --strong "
                         "for configs[3]) or configs[4] (one shot per GPU + gradient all-reduce)")
    spec = slab_spec(p, nranks, strong)
    x0, n0_loc = slab_range(spec, rank, nranks)
    r = p.space_order // 2
    m_loc = spec["m_planes"](x0 - r, x0 + n0_loc + r)
    eta_loc = spec["eta_planes"](x0 - r, x0 + n0_loc + r)
    return spec["p"], m_loc, eta_loc, spec["gshape"]


def slab_range(spec, rank, nranks):
    import paper_1707_03776_b200 as sf
    return sf.slab_plan(spec["gshape"][0], spec["p"].space_order, rank, nranks)


def slab_spec(p, nranks, strong):
    """Global slab problem: configs[1] / configs[3] tiled along x (weak: 336 N / 1024 N planes;
    both models are x-invariant, so the tiling is exact) or, --strong, configs[3] as given.
    Returns the global problem (sources / receivers moved to the global geometry) and
    functions giving the model / damping of a plane range [lo, hi) as host fp32 arrays
    (planes outside the grid replicate the edge: halo planes of m / eta are unused)."""
    import synth as S
    n0 = p.shape[0]
    gn0 = n0 if strong else n0 * nranks
    gshape = (gn0,) + tuple(p.shape[1:])
    m_col = p.m[0]                        # every x-plane of these models is identical
    sig = None
    if p.damp is not None:
        # damping of the global grid from its per-axis profiles (reading C7), evaluated on
        # the requested planes only (no global 3D array per rank)
        vmax = 2500.0                     # configs[1] (the only damped slab config)
        p.sigma = S.damping_profiles_1d(gshape, p.nbl, p.h, vmax)
        sig = [a.astype(np.float64) for a in p.sigma]

    def m_planes(lo, hi):
        return np.ascontiguousarray(np.broadcast_to(m_col, (hi - lo,) + gshape[1:]), dtype=np.float32)

    def eta_planes(lo, hi):
        if sig is None:
            return None
        idx = np.clip(np.arange(lo, hi), 0, gn0 - 1)
        s3 = sig[0][idx][:, None, None] + sig[1][None, :, None] + sig[2][None, None, :]
        return (m_planes(lo, hi).astype(np.float64) * s3).astype(np.float32)

    if not strong:
        src = p.src_coords.copy()
        src[:, 0] = gn0 * p.h / 2.0 if p.damp is not None else (gn0 - 1) * p.h / 2.0
        if p.damp is not None:
            # configs[1]: the 256 x 256 surface grid, centred in the global x extent
            rec = p.rec_coords.copy()
            rec[:, 0] = rec[:, 0] + (nranks - 1) * n0 * p.h / 2.0
        else:
            # configs[3]: one receiver per plane along x at (y = centre, z = 0)
            rec = np.stack([np.arange(gn0) * p.h, np.full(gn0, p.rec_coords[0, 1]), np.zeros(gn0)],
                           axis=1).astype(np.float32)
        p.src_coords, p.rec_coords = src.astype(np.float32), rec
    return {"p": p, "gshape": gshape, "m_planes": m_planes, "eta_planes": eta_planes}


def slab_bitwise_check(args, cfg, comm, rank, world, nt_check=12):
    """The slab run of a short record (nt_check samples) vs the single-domain run of the SAME
    global problem on this rank's GPU: the owned planes of both final levels and the summed
    records must be bitwise equal (reading C18).  Returns the flag agreed over all ranks."""
    import torch
    import torch.distributed as dist

    import paper_1707_03776_b200 as sf
    import synth
    p = synth.make_config(cfg, nt=nt_check)
    spec = slab_spec(p, world, args.strong)
    p, gshape = spec["p"], spec["gshape"]
    r = p.space_order // 2
    x0, nl = slab_range(spec, rank, world)
    dev = lambda x: None if x is None else torch.from_numpy(x).cuda()
    kw = dict(shape=gshape, h=p.h, space_order=p.space_order, nt=p.nt, dt=p.dt,
              src_coords=p.src_coords, rec_coords=p.rec_coords,
              sigma=p.sigma if (args.sep and p.damp is not None) else None)
    sep = kw["sigma"] is not None
    wav = dev(np.ascontiguousarray(p.wavelet))
    ps = sf.Propagator(dev(spec["m_planes"](x0 - r, x0 + nl + r)),
                       None if sep else dev(spec["eta_planes"](x0 - r, x0 + nl + r)),
                       comm=comm, rank=rank, nranks=world, **kw)
    if args.p2p:
        ps.set_option(8, 1)
    rec_s, u_s, _ = ps.forward(wav)
    torch.cuda.synchronize()
    ps.close()
    dist.all_reduce(rec_s)                  # one owner per receiver row: the sum is exact
    p1 = sf.Propagator(dev(spec["m_planes"](0, gshape[0])),
                       None if sep else dev(spec["eta_planes"](0, gshape[0])), **kw)
    rec_1, u_1, _ = p1.forward(wav)
    torch.cuda.synchronize()
    p1.close()
    ok = bool(torch.equal(rec_s, rec_1)) and bool(torch.equal(u_s[:, r:r + nl], u_1[:, x0:x0 + nl]))
    del u_1, rec_1, u_s, rec_s
    torch.cuda.empty_cache()
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return {"bitwise_equal": bool(t.item()), "nt": nt_check,
            "what": "slab run vs single-domain run of the same global problem on each rank's GPU: "
                    "owned planes of both final levels + summed records"}


WORKLOADS = {
    0: "configs[0]: 2D acoustic forward 101^2 phys + nbl 20 -> 141x141, so4, nt=500, 101 receivers",
    1: "configs[1]: 3D acoustic forward 256^3 phys + nbl 40 -> 336^3 comp, so8, nt=1000, "
       "65536 receivers, 1 source",
    2: "configs[2]: 3D FWI gradient 256^3 phys + nbl 40 -> 336^3, so8, nt=1000, save every 4 "
       "(fwd+save, residual, adjoint+correlation; d_obs from the true model outside the timed region)",
    3: "configs[3]: 3D acoustic forward 1024x512x512, so16, nt=500, no damping layer",
    4: "configs[4]: one shot of the multi-shot FWI gradient, 400^3, so12, nt=1500, save every 3",
}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1707_03776_b200 as sf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [sf.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = sf.nccl_comm_init(uid[0], world, rank)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    cfg = args.config
    comm_info = None
    if comm is not None:
        n_c, r_c = sf.nccl_comm_info(comm)
        comm_info = {"nranks": n_c, "rank": r_c, "ok": n_c == world}
        log(f"[bench] NCCL communicator: nranks {n_c} (world {world}), rank {r_c}")
        if n_c != world:
            raise SystemExit(f"NCCL communicator spans {n_c} ranks, world is {world}")
    p, m_loc, eta_loc, gshape = build_problem(args.nt, rank, world, cfg, args.strong)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    m_d = dev(m_loc)
    # damping: the eta array (hoisted beta streamed, 20 B/pt) unless --sep regenerates beta
    # from the separable profiles (sf_desc.sigma, 16 B/pt; measured slower on B200: the
    # kernel is latency-bound there)
    sep = eta_loc is not None and p.sigma is not None and args.sep
    eta_d = None if (eta_loc is None or sep) else dev(eta_loc)
    slab = world > 1 and cfg != 4           # configs[4] shards shots, not the grid
    prop = sf.Propagator(m_d, eta_d, shape=gshape, h=p.h, space_order=p.space_order, nt=p.nt,
                         dt=p.dt, src_coords=p.src_coords, rec_coords=p.rec_coords,
                         comm=comm if slab else None, rank=rank if slab else 0,
                         nranks=world if slab else 1, sigma=p.sigma if sep else None)
    if args.split:
        prop.set_option(2, 1)
        if args.one_launch and world == 1:
            prop.set_option(11, 2)  # SF_OPT_ONE_LAUNCH: the one-launch slab schedule, emulated on one GPU
    if args.graph:
        prop.set_option(5, 1)
    if args.p2p and slab:
        prop.set_option(8, 1)   # peer-store halo exchange instead of NCCL send/recv
    if args.snap_half:
        prop.set_option(7, 1)
    if args.no_pdl:
        prop.set_option(12, 0)  # SF_OPT_PDL off: plain launches
    # time every 16th kernel launch of each kind inside the timed steps (an event pair around
    # every launch costs 1-3 % of a step and defeats PDL; the average over ~60 timed stencil
    # launches per step is the kernel's average launch time)
    prop.set_option(13, args.prof_every)
    tuned = None
    if not args.no_autotune:
        # setup-time tuning (sf_autotune; the paper's runtime block-size tuning):
        # outside the timed region, same bits for every choice
        tuned = prop.autotune(steps=10)
    if args.tblock:
        prop.set_option(15, 1)  # SF_OPT_TBLOCK: two steps per launch (forward without snapshots)
    wav = dev(p.wavelet)
    u = prop.zeros_state()
    rec = torch.empty((p.nt, p.rec_coords.shape[0]), device="cuda")
    npts_local = int(np.prod(prop.local_shape)) if not slab else prop.n0_loc * int(np.prod(gshape[1:]))
    tuning = prop.tuning()
    log(f"[bench] rank {rank}/{world} grid {gshape} local {prop.local_shape} nt {p.nt} tuning {tuning}")

    grad_mode = cfg in (2, 4)
    passes = 2 if grad_mode else 1          # propagations per step (fwd + adj for gradients)
    if grad_mode:
        k = p.save_every
        # observed data from the true model (input preparation, outside the timed region)
        prop_true = sf.Propagator(dev(p.m_true), None if eta_loc is None else dev(eta_loc), shape=gshape,
                                  h=p.h, space_order=p.space_order, nt=p.nt, dt=p.dt,
                                  src_coords=p.src_coords, rec_coords=p.rec_coords)
        d_obs, _, _ = prop_true.forward(wav)
        torch.cuda.synchronize()
        prop_true.close()
        del prop_true
        ws = torch.empty(prop.gradient_workspace_bytes(k), dtype=torch.uint8, device="cuda")
        grad = torch.empty(prop.local_shape, device="cuda")

    def step():
        if grad_mode:
            prop.gradient(wav, d_obs, save_every=k, grad=grad, ws=ws)
            if world > 1:
                # multi-shot: sum the per-shot gradients over the GPUs (NCCL, in-stream)
                prop.allreduce_gradient(comm, grad, rank=rank)
        else:
            u.zero_()
            prop.forward(wav, u=u, rec=rec)

    for _ in range(args.warmup):
        step()
    barrier()
    clk = ClockSampler(local)
    clk.start()
    # per-launch kernel times come from in-stream events recorded by the library; with
    # --graph the timed steps replay CUDA graphs (no events) and one extra profiled eager
    # step after the timed region provides the kernel times
    prop.set_profiling(not (args.graph or args.no_prof))
    prop.profile(reset=True)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    # NVTX range of the timed steps: `ncu --nvtx --nvtx-include sf_timed/` profiles these
    # launches only, so setup-time tuning runs unprofiled and picks what it picks without ncu
    torch.cuda.nvtx.range_push("sf_timed")
    e0.record(stream)
    marks[0].record(stream)
    for i in range(args.steps):
        step()
        marks[i + 1].record(stream)
    e1.record(stream)
    torch.cuda.nvtx.range_pop()
    barrier()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    if args.graph or args.no_prof:
        prop.set_profiling(True)
        prop.profile(reset=True)
        step()
        torch.cuda.synchronize()
        prof = prop.profile(reset=True)
        prof = {k: (v * args.steps if isinstance(v, (int, float)) else v) for k, v in prof.items()}
    else:
        prof = prop.profile(reset=True)
    prop.set_profiling(False)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sf.nccl_check(comm)
    ms_max = float(t.item())
    # points updated per step over all ranks: the global grid (slab: the ranks' owned planes
    # partition it; shots: one full grid per rank)
    updates = (int(np.prod(gshape)) if slab else npts_local * world) * (p.nt - 1) * args.steps * passes
    value = updates / (ms_max * 1e-3) / 1e9

    # roofline of the dominant kernel (stencil step): algorithmic bytes per launch
    bpp = 20 if eta_d is not None else 16      # u^n, u^{n-1}, out, c3 (+beta array) fp32
    # the stencil's average launch duration, two CUDA-event measurements over the timed
    # region, both upper bounds: (a) the event-timed launches (every --prof-every-th; each
    # such interval also holds the launch gap the event forces before the kernel) and (b) the
    # wall time per update (every main-stream kernel of the step, gaps included); the tighter
    # one is reported
    sampled_ms = prof["stencil_ms"] / max(prof["stencil_launches"], 1)
    upl = 2 if args.tblock else 1            # updates per stencil launch
    wall_ms = ms_max / (args.steps * (p.nt - 1) * passes) * upl
    launch_ms = min(sampled_ms, wall_ms)
    split = args.split or slab
    if split:
        # boundary and interior launches overlap: time the stencil by the wall time per update
        launch_ms = wall_ms
    alg_bytes = bpp * npts_local
    if args.tblock:
        alg_bytes = (bpp + 4) * npts_local   # two updates: u^{n-1}, u^n, c3 (, beta) read, two levels written
    if grad_mode:
        # forward: nt-1 launches, (nt-1)//k of them also store a snapshot (+4 B/pt); adjoint:
        # nt-1 launches, (nt-1)//k of them also read the snapshot and update the gradient
        # (+12 B/pt) -- averaged over the 2 (nt-1) stencil launches of a gradient
        nk = (p.nt - 1) // k
        se = 2 if args.snap_half else 4   # snapshot bytes: written on save steps, read on correlation steps
        alg_bytes = int(round(npts_local * (bpp + (se * nk + (se + 8) * nk) / (2 * (p.nt - 1)))))
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    traffic, traffic_rel = ncu_traffic(cfg)

    check = None
    if slab and not args.no_check:
        del u, rec
        prop.close()
        torch.cuda.empty_cache()
        check = slab_bitwise_check(args, cfg, comm, rank, world)
        log(f"[bench] slab check: {check}")
    result = None
    if rank == 0:
        # end to end through the public C-ABI with HOST buffers (pinned), N=1 form
        e2e = None
        if world == 1 and not args.no_e2e and cfg in (0, 1, 3):
            e2e = run_e2e(p, args, sep)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(p, args.cpu_seconds)
        result = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
            "step_ms": {"median": round(statistics.median(step_ms), 3), "best": round(min(step_ms), 3),
                        "rank0_all": [round(x, 3) for x in step_ms]},
            "higher_is_better": True, "scaling": "strong" if (slab and args.strong) else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": f"synthetic (seeded {p.name} model of BASELINE configs[{cfg}], readings of "
                    "SURVEY 8.0; no dataset in the paper)",
            "config": {"workload": WORKLOADS[cfg] + (f" ({'strong' if args.strong else 'weak'}-scaled: "
                                                     f"{'x'.join(map(str, gshape))} global, x-slab per GPU)" if slab else
                                                     f" (weak-scaled: {world} shots, one per GPU, gradient "
                                                     f"all-reduce in every step)" if world > 1 else ""),
                       "grid": list(gshape), "space_order": p.space_order, "nt": p.nt,
                       "points_per_rank": npts_local, "parallelism": f"slab{world}" if slab else f"shots{world}" if world > 1 else "1gpu",
                       "l2": "inputs larger than L2 (each fp32 field >= 152 MB > 126 MB L2; "
                             "4-5 fields streamed per update)" if npts_local * 4 > 126e6 else
                             "grid smaller than L2 (configs[0]: launch-bound toy)",
                       "propagations_per_step": passes,
                       "snapshots": ("fp16" if args.snap_half else "fp32") if grad_mode else None,
                       "damping": ("separable profiles (sf_desc.sigma): beta regenerated in-kernel" if sep else
                                   "eta array (hoisted beta streamed)" if eta_d is not None else "none"),
                       "halo_exchange": (("peer stores from the boundary kernel + stream counters"
                                          if args.p2p else "NCCL send/recv") if slab else None),
                       "schedule": (("one launch per step storing its boundary planes into the neighbours' "
                                     "halos (peer stores), stream-ordered counters" if (slab and args.p2p) else
                                     "one launch per step, boundary ranges signalled to the comm stream"
                                     if (args.one_launch or slab) else
                                     "split (boundary planes, then interior)") if split else
                                    "two steps per launch (temporal blocking)" if args.tblock else
                                    "single launch per step") + (", CUDA graph replay" if args.graph else ""),
                       "kernel_tuning": tuning, "autotune": tuned},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "frac_of_nominal_8TBps": round(achieved / 8000.0, 4),
                         "traffic": None if traffic is None else int(traffic),
                         "traffic_source": ((f"{traffic_rel} (ncu dram read+write of every stencil launch "
                                             "of a gradient step, per-mode means weighted to the average "
                                             "update of this config)") if "step_traffic" in traffic_rel else
                                            (f"{traffic_rel} (ncu --set full, dram read+write per "
                                             "launch, random-init wavefield)")) if traffic is not None
                                           else f"no ncu capture for this config ({traffic_rel})",
                         "peak_source": peak_src,
                         "kernel": ("k_tma3d (boundary + interior launches; wall time per update)" if split else
                                    "k_tma3d (stencil step)") if tuning["variant"] == 2 else
                                   ("k_generic3d" if len(gshape) == 3 else "k_generic2d"),
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "bytes_per_point": round(alg_bytes / npts_local, 3), "avg_launch_ms": round(launch_ms, 5),
                         "launch_time_source": {"event_timed_launches_ms": round(sampled_ms, 5),
                                                "wall_per_update_ms": round(wall_ms, 5),
                                                "timed_every": args.prof_every,
                                                "used": "wall per update" if launch_ms == wall_ms else "event-timed launches"},
                         "stencil_share_of_step": round(prof["stencil_ms"] / max(ms, 1e-9), 4),
                         "per_update_us": {k: round(prof[f"{k}_ms"] * 1e3 / (args.steps * (p.nt - 1)), 2)
                                           for k in ("stencil", "inject", "interp", "other")},
                         "per_update_note": "event time per kind on its own stream: 'interp' is the record "
                                            "kernel on the side stream, overlapped with the next stencil step, "
                                            "and includes its queueing behind the persistent stencil CTAs (its "
                                            "own cost, serialised and cold, is in the ncu launch list: "
                                            "profiles/r02_bench_launches.json)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(prof["launches"]),
            "clocks": clocks,
            "comm": comm_info,
            "slab_check": check,
        }
    if world > 1:
        dist.barrier()
        sf.nccl_comm_destroy(comm) if comm else None
        dist.destroy_process_group()
    return result


def run_e2e(p, args, sep=False):
    import torch

    import paper_1707_03776_b200 as sf
    pin = lambda x: torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).pin_memory()
    m_h, w_h = pin(p.m), pin(p.wavelet)
    d_h = None if (sep or p.damp is None) else pin(p.damp)
    rec_h = torch.empty((p.nt, p.rec_coords.shape[0]), dtype=torch.float32).pin_memory()
    call = lambda: sf.forward_host(m_h.numpy(), None if d_h is None else d_h.numpy(), h=p.h,
                                   space_order=p.space_order, nt=p.nt, dt=p.dt, src_coords=p.src_coords,
                                   wavelet=w_h.numpy(), rec_coords=p.rec_coords,
                                   rec_out=rec_h.numpy(), sigma=p.sigma if sep else None)
    call()  # warm-up (allocates the library's device cache)
    torch.cuda.synchronize()
    n = max(1, min(args.steps, 3))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        call()
    e1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms = max(e0.elapsed_time(e1), wall * 1e3)
    N = int(np.prod(p.shape))
    return {"value": round(N * (p.nt - 1) * n / (ms * 1e-3) / 1e9, 3), "unit": UNIT,
            "h2d_bytes_per_step": int(m_h.numel() * 4 + (0 if d_h is None else d_h.numel() * 4) + w_h.numel() * 4
                                      + (sum(len(a) for a in p.sigma) * 4 if sep else 0)),
            "d2h_bytes_per_step": int(rec_h.numel() * 4), "steps": n,
            "includes": "H2D m/" + ("sigma profiles" if sep else "eta") + "/wavelet, handle setup "
                        "(coefficient hoist, tables, CFL), forward, D2H record"}


def host_cpu():
    """CPU model of this host (/proc/cpuinfo) and the OpenMP thread setting the oracle ran
    with (record nproc, the CPU model and OMP_NUM_THREADS)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.lower().startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(),
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS", "unset (OpenMP default: all cores)")}


def cpu_baseline(p, seconds):
    """The oracle as it stands (fp64, OpenMP over all host cores) on a bounded sample:
    the same grid and model, first `k` time steps, k sized to ~`seconds` of CPU work."""
    import oracle
    oracle.build()
    N = int(np.prod(p.shape))
    # per-update time from two short runs (their difference cancels the fixed setup cost:
    # tables, first touch of the fp64 arrays)
    tps = []
    for probe in (2, 4):
        t0 = time.perf_counter()
        oracle.forward(p, nt=probe, wavelet=p.wavelet[:probe])
        tps.append(time.perf_counter() - t0)
    per_update = max((tps[1] - tps[0]) / 2.0, 1e-4)
    k = int(max(4, min(p.nt, seconds / per_update + 1)))
    t0 = time.perf_counter()
    oracle.forward(p, nt=k, wavelet=p.wavelet[:k])
    t = time.perf_counter() - t0
    return {"value": round(N * (k - 1) / t / 1e9, 5), "unit": UNIT, "cores": oracle.num_threads(),
            "kind": "oracle", "seconds": round(t, 2), **host_cpu(),
            "sample": f"{p.name}: full {'x'.join(map(str, p.shape))} grid, first {k} of {p.nt} time "
                      f"samples ({k - 1} forward updates), fp64 C oracle"}


def run_reference(args):
    """--impl reference: the paper ships no code (PAPER.md only), so the reference arm is
    the fp64 C oracle, timed as it stands on the host cores, on a bounded sample of the
    same workload (the first `--ref-steps-nt` time samples of the config per step)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and rank != 0:
        return None
    import oracle
    import synth
    oracle.build()
    p = synth.make_config(args.config, nt=args.nt)
    N = int(np.prod(p.shape))
    k = min(args.ref_steps_nt, p.nt)
    for _ in range(min(args.warmup, 1)):
        oracle.forward(p, nt=2, wavelet=p.wavelet[:2])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.forward(p, nt=k, wavelet=p.wavelet[:k])
    t = time.perf_counter() - t0
    v = N * (k - 1) * args.steps / t / 1e9
    sample = f"{p.name}: full {'x'.join(map(str, p.shape))} grid, {k} of {p.nt} time samples per step"
    cpu = {"value": round(v, 5), "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
           "sample": sample, **host_cpu()}
    return {"impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t / args.steps * 1e3, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config] + f" -- bounded sample: {sample}"},
            "cpu_baseline": cpu,
            "e2e": {"value": round(v, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nt", type=int, default=None, help="override nt (default: the config's)")
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4],
                    help="BASELINE configs[i] workload (default 1: the metric's headline config)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--split", action="store_true",
                    help="1 GPU: run the slab schedule (boundary planes first, interior second) "
                         "to measure its cost without communication")
    ap.add_argument("--one-launch", action="store_true",
                    help="with --split on 1 GPU: the one-launch slab schedule (SF_OPT_ONE_LAUNCH 2: one "
                         "launch per step, boundary ranges signalled on device counters the comm stream "
                         "waits on) instead of the two-launch split")
    ap.add_argument("--p2p", action="store_true",
                    help="N > 1 slab runs: peer-store halo exchange (SF_OPT_P2P) instead of NCCL send/recv")
    ap.add_argument("--graph", action="store_true",
                    help="replay each step as a CUDA graph (SF_OPT_GRAPH; for launch-bound grids)")
    ap.add_argument("--snap-half", action="store_true",
                    help="gradient configs: fp16 snapshots (SF_OPT_SNAP_HALF, reading C23)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-autotune", action="store_true",
                    help="skip the setup-time tuning (sf_autotune) and keep the library's defaults")
    ap.add_argument("--no-pdl", action="store_true",
                    help="plain launches instead of programmatic dependent launches (SF_OPT_PDL 0)")
    ap.add_argument("--prof-every", type=int, default=16,
                    help="time every n-th kernel launch of each kind inside the timed region (default 16)")
    ap.add_argument("--no-prof", action="store_true",
                    help="A/B runs only: no per-kernel events inside the timed steps (kernel times from "
                         "one extra profiled step after them)")
    ap.add_argument("--strong", action="store_true",
                    help="N > 1, --config 3: split the literal 1024x512x512 grid over the GPUs "
                         "(strong scaling) instead of 1024 planes per GPU (weak)")
    ap.add_argument("--no-check", action="store_true",
                    help="N > 1 slab runs: skip the bitwise slab-vs-single-domain check after the timed region")
    ap.add_argument("--sep", action="store_true",
                    help="damped configs: regenerate beta in-kernel from the separable damping "
                         "profiles (16 B/pt) instead of streaming the hoisted beta array (20 B/pt)")
    ap.add_argument("--tblock", action="store_true",
                    help="forward configs: two time steps per launch (SF_OPT_TBLOCK, temporal "
                         "blocking; r <= 4, one GPU) -- measured slower, A/B only")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-steps-nt", type=int, default=6,
                    help="--impl reference: time samples per timed step of the oracle")
    args = ap.parse_args()
    if args.p2p:
        # the counter waits of the peer-store exchange are blocking stream operations: give
        # every stream its own hardware queue so no wait can stall an unrelated stream
        # (must be set before the CUDA context exists)
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    if args.impl == "reference":
        res = run_reference(args)
    else:
        res = run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
