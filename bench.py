#!/usr/bin/env python3
"""Benchmark of the B200 PCG hot path (driver contract: one JSON line).

A "step" is one linear solve of the configuration to its PCG tolerance
(newton_solve, linear branch: RHS, preconditioner setup, PCG loop, Newton
check, homogenized stress) with all inputs resident in HBM.

  value      DOF * PCG iterations / device time of the PCG iterations
             (CUDA events on the library stream, summed over the K steps)
  e2e        the same metric through the public C ABI with HOST buffers:
             material upload (phase map H2D) + homfe_gpu_solve (u D2H) per
             step, host clock
  roofline   the dominant kernel of one PCG iteration (the largest live
             CUDA-event time among K apply and the three fused FFT passes),
             its algorithmic bytes per launch against
             MEASURED_PEAKS.json hbm_gbs
  cpu_baseline  the CPU oracle (faithful restatement of the reference,
             single thread like the reference) on a bounded sample

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3]
       [--impl reference]
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c1": "c1: 256^2 scalar conductivity, two triangles, 20 circles r=12 px, contrast 10, C_ref=I, eta_cg 1e-8",
    "c2": "c2: 128^3 scalar conductivity, trilinear hex, spheres r=8 f=0.25, contrast 100, volume-mean ref, eta_cg 1e-8",
    "c3": "c3: 256^3 linear elasticity, trilinear hex 2x2x2 Gauss, spheres r=10 f=0.30 (E 1000/1, nu 0.2/0.3), "
          "eps_xy=0.01, C_ref=matrix phase, eta_cg 1e-6",
    "c4": "c4: 512^3 linear elasticity, thresholded GRF l=16 f=0.5, contrast 1e4, C_ref=matrix phase, eta_cg 1e-6",
    "c5": "c5: N^2 scalar conductivity sweep, two triangles, circles f=0.30, volume-mean ref, eta_cg 1e-8",
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def workload_config(args, cfg):
    """The `config` object both arms print (the driver compares them)."""
    return {"workload": WORKLOADS[args.config], "dims": list(cfg.dims), "dof": int(cfg.dof),
            "stencil": cfg.stencil, "eta_cg": cfg.eta_cg}


def setup_problem(cfg):
    import paper_2203_02962_b200 as hb
    t0 = time.time()
    phases = cfg.phases()
    tangents = cfg.tangents()
    g = hb.Grid(cfg.dims, [1.0] * cfg.dim, cfg.stencil)
    mats = [hb.Material(t, cfg.thermal, cfg.dim) for t in tangents]
    return g, mats, phases, tangents, time.time() - t0


def run_gpu(args, rank, world, local_rank):
    import ctypes as C
    import torch
    import paper_2203_02962_b200 as hb
    from paper_2203_02962_b200 import _native, inputs

    torch.cuda.set_device(local_rank)
    cfg = inputs.config(args.config, n=args.n, contrast=args.contrast)
    g, mats, phases, tangents, t_inputs = setup_problem(cfg)
    slab = world > 1 or args.slab
    solver = hb.Solver(g, mats, phases, eta_newton=cfg.eta_newton, eta_cg=cfg.eta_cg,
                       reference=cfg.reference, reference_matrix=cfg.reference_matrix()) if not slab else None
    lib = _native.lib
    dof = cfg.dof
    m = tangents.shape[1]
    e = np.ascontiguousarray(cfg.load, dtype=np.float64)
    if not slab:
        ctx_h = solver.ctx.h
        scfg = solver.cfg
        n_local = g.num_nodes
        ph_local = phases
    else:
        # slab decomposition: one NCCL communicator inside the library
        from paper_2203_02962_b200 import dist as hdist
        obj = [hdist.nccl_unique_id() if rank == 0 else None]
        if world > 1:
            torch.distributed.broadcast_object_list(obj, src=0)
        sc = hdist.SlabContext(g, cfg.components, rank, world, obj[0], device=local_rank)
        transport = {"peer_pull": "peer pull over NVLink + barrier all-reduces",
                     "all_to_all": "NCCL halo + all-to-all", "single": "one rank"}[sc.transport]
        z0, nz = hdist.slab_range(g.dims[0], rank, world)
        plane = int(np.prod(g.dims[1:]))
        ph_local = np.ascontiguousarray(phases[z0 * plane:(z0 + nz) * plane])
        sc.set_material(tangents, ph_local)
        scfg = _native.SolveCfg()
        scfg.eta_newton, scfg.eta_cg, scfg.max_newton, scfg.max_cg = cfg.eta_newton, cfg.eta_cg, 25, 20000
        scfg.reassembly_threshold, scfg.criterion = 0.1, 0
        scfg.reference_policy = {"identity-scaled": 0, "volume-mean": 1, "explicit": 2}[cfg.reference]
        scfg.reference_scale = 1.0
        refm = cfg.reference_matrix()
        _keep = None
        if refm is not None:
            _keep = np.ascontiguousarray(np.asarray(refm).T, dtype=np.float64)
            scfg.reference_matrix = _keep.ctypes.data_as(C.POINTER(C.c_double))
        ctx_h = sc.h
        n_local = sc.n_local
    d_u = torch.empty(cfg.components * n_local, dtype=torch.float64, device="cuda")
    avg = np.zeros(m)

    def solve_device():
        rep = _native.Report()
        code = lib.homfe_gpu_solve_device(ctx_h, e.ctypes.data_as(C.POINTER(C.c_double)), C.byref(scfg),
                                          None, C.c_void_p(d_u.data_ptr()),
                                          avg.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep))
        hb._check(code)
        return rep

    for _ in range(args.warmup):
        solve_device()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    iters, cg_ms, launches = 0, 0.0, 0
    with ClockSampler(local_rank) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            rep = solve_device()
            iters += rep.total_cg
            cg_ms += rep.cg_device_ms
            launches += rep.kernel_launches
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if world > 1:
        torch.distributed.barrier()
    clocks = clk.summary()
    # max over ranks of the timed quantities
    stats = torch.tensor([cg_ms, wall], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(stats, op=torch.distributed.ReduceOp.MAX)
    cg_ms_max, wall_max = float(stats[0]), float(stats[1])
    value = dof * iters / (cg_ms_max / 1e3)  # global DOF (strong scaling over slabs)

    # per-kernel breakdown of one PCG iteration (CUDA events, live)
    ms = np.zeros(8)
    hb._check(lib.homfe_gpu_kernel_times(ctx_h, 20, ms.ctypes.data_as(C.POINTER(C.c_double))))
    fused_planes = bool(ms[2] < 0)  # the fused passes report no separate FFT kernels

    # e2e: host buffers through the C ABI, copies inside the timed region
    # pinned host buffers (the contract's H2D/D2H from page-locked memory)
    ph_host = torch.empty(ph_local.size, dtype=torch.uint8, pin_memory=True).numpy()
    ph_host[:] = np.ascontiguousarray(ph_local, dtype=np.uint8).ravel()
    cm = np.ascontiguousarray(np.stack(tangents).transpose(0, 2, 1), dtype=np.float64)
    u_host = torch.zeros(cfg.components * n_local, dtype=torch.float64, pin_memory=True).numpy()
    e2e_iters = 0
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(e2e_steps):
        hb._check(lib.homfe_gpu_set_material(ctx_h, cm.shape[0], cm.ctypes.data_as(C.POINTER(C.c_double)),
                                             ph_host.ctypes.data_as(C.POINTER(C.c_uint8))))
        rep = _native.Report()
        hb._check(lib.homfe_gpu_solve(ctx_h, e.ctypes.data_as(C.POINTER(C.c_double)), C.byref(scfg), None,
                                      u_host.ctypes.data_as(C.POINTER(C.c_double)),
                                      avg.ctypes.data_as(C.POINTER(C.c_double)), C.byref(rep)))
        e2e_iters += rep.total_cg
    e2e_wall = time.perf_counter() - t0
    if world > 1:
        wt = torch.tensor([e2e_wall], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(wt, op=torch.distributed.ReduceOp.MAX)
        e2e_wall = float(wt[0])
    if solver is not None:
        solver.ctx._material_key = None
    e2e_value = dof * e2e_iters / e2e_wall

    slab_check = None
    if slab:
        # self-check of the decomposed solve (outside every timed region): the
        # slabs of u from the last e2e solve are gathered and compared on rank
        # 0 with a single-device solve of the same input
        u_loc = torch.from_numpy(np.array(u_host, copy=True)).cuda()
        if world > 1:
            parts = torch.empty(world * u_loc.numel(), dtype=torch.float64, device="cuda")
            torch.distributed.all_gather_into_tensor(parts, u_loc)
        else:
            parts = u_loc
        k_slab = int(rep.total_cg)
        if rank == 0:
            c = cfg.components
            u_slab = parts.view(world, c, -1).transpose(0, 1).reshape(c, -1).cpu().numpy()
            del parts, u_loc
            one = hb.Solver(g, mats, phases, eta_newton=cfg.eta_newton, eta_cg=cfg.eta_cg,
                            reference=cfg.reference, reference_matrix=cfg.reference_matrix())
            ref1 = one.solve(e)
            k1 = int(ref1["report"]["cg_total"])
            u1 = ref1["u"]
            slab_check = {"against": "single-device solve of the same input on rank 0",
                          "pcg_iterations": {"slab": k_slab, "single": k1},
                          "rel_u": float(np.linalg.norm(u_slab - u1) / np.linalg.norm(u1)),
                          "rel_sigma": float(np.linalg.norm(avg - ref1["average_stress"]) /
                                             np.linalg.norm(ref1["average_stress"])),
                          "u_checksum": {"slab": float(np.abs(u_slab).sum()), "single": float(np.abs(u1).sum())}}
            slab_check["ok"] = bool(abs(k_slab - k1) <= 1 and slab_check["rel_sigma"] <= 1e-8)
            del one
        if world > 1:
            torch.distributed.barrier()

    hbm, peak_kind = peaks()
    c = cfg.components
    npx = n_local if slab else g.num_pixels
    # dominant kernel of the iteration (largest live CUDA-event time) and its
    # algorithmic bytes per launch
    if fused_planes:
        cands = [("k_hex_z" if cfg.stencil == "trilinear-hex" else "k_apply_elem", "stencil K apply",
                  ms[0], (16 * c + 1) * npx),
                 ("k_plane_fwd", "pass 1: r -= alpha Ap + plane r2c FFTs", ms[1], 32 * c * npx),
                 ("k_pencil", "pass 2: axis-0 FFTs + spectral solve + r.z", ms[3], 16 * c * npx),
                 ("k_plane_inv", "pass 3: plane c2r FFTs + x/p updates", ms[5], 40 * c * npx)]
    else:
        kname = {"trilinear-hex": "k_hex_z", "two-triangles": "k_elem2d"}.get(cfg.stencil, "k_apply_elem")
        cands = [(kname, "stencil K apply", ms[0], (16 * c + 1) * npx)]
    kname, kdesc, kms, bytes_k = max(cands, key=lambda t: t[2])
    achieved = bytes_k / (kms / 1e3) / 1e9
    traffic = None
    iter_traffic = None
    tp = os.path.join(ROOT, "profiles", "r02_c3_ncu_traffic.json")
    if os.path.exists(tp) and world == 1:
        with open(tp) as f:
            tj = json.load(f)
        if list(tj.get("dims", [])) == list(cfg.dims):
            traffic = tj["bytes_per_launch"].get(kname)
            if fused_planes:  # one launch of each of the four iteration kernels
                iter_traffic = sum(tj["bytes_per_launch"].values())
    # ideal fused iteration bytes per GPU: N_p (112 c + 1) / world
    b_iter = (112 * c + 1) * g.num_pixels / world
    iter_ms = cg_ms_max / max(iters, 1)
    nvlink = None
    if slab:
        # algorithmic interconnect bytes per iteration and GPU:
        # two halo planes of p for K, and the forward and inverse spectrum
        # transposes ((G-1)/G of the rank's c N_f / G complex values each)
        nh = g.dims[-1] // 2 + 1
        nf = int(np.prod(g.dims[:-1])) * nh
        halo = 2 * c * int(np.prod(g.dims[1:])) * 8 if world > 1 else 0
        a2a = 2 * c * 16 * (nf / world) * (world - 1) / world
        nbytes = halo + a2a
        nv_peak = 900.0  # GB/s per direction, NVLink 5 (B200 datasheet)
        floor_ms = max(b_iter / hbm / 1e6, nbytes / nv_peak / 1e6)
        nvlink = {"bytes_per_iteration_per_gpu": nbytes, "halo_bytes": halo, "transpose_bytes": a2a,
                  "peak_gbs": nv_peak, "peak_source": "NVLink 5 nominal, per direction",
                  "hbm_nvlink_roofline_ms": floor_ms, "frac": floor_ms / iter_ms}
    out = {
        "metric": "DOF·PCG-iterations/s",
        "value": value,
        "unit": "DOF*it/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": wall_max / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: seeded RSA inclusions / GRF per SURVEY 8(d) (no dataset in the reference)",
        "config": workload_config(args, cfg),
        "solve": {"pcg_iterations_per_step": iters // args.steps, "newton_steps": rep.n_steps,
                  "parallelism": (f"slab decomposition over {world} GPUs ({transport}, "
                                  f"{'fused FFT passes' if fused_planes else 'slab spectra: cuFFT + transposes'})")
                  if slab else "1 GPU",
                  "l2": f"inputs exceed L2: {cfg.components * g.num_pixels * 8 / 1e6:.0f} MB per vector vs 126 MB"
                  if cfg.components * g.num_pixels * 8 > 126e6 else "L2-resident working set (no flush)",
                  "step": "one linear solve to eta_cg (Newton linear branch + PCG), inputs resident in HBM"},
        "time_to_solution_s": wall_max / args.steps,
        "iteration_ms": iter_ms,
        "iteration_roofline_frac": (b_iter / (iter_ms / 1e3) / 1e9) / hbm,
        "iteration_bytes": {"algorithmic": b_iter, "dram_ncu": iter_traffic},
        "roofline": {"kernel": f"{kdesc} ({kname})", "bound": "hbm", "achieved": achieved,
                     "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                     "traffic_source": "profiles/r02_c3_ncu_traffic.json (ncu --set full, per launch)"
                     if traffic else None,
                     "peak_source": peak_kind, "bytes_per_launch": bytes_k, "kernel_ms": kms},
        "kernel_ms": ({"apply_K": ms[0], "update_r": ms[1], "fft_fwd": ms[2], "spectral": ms[3],
                       "fft_inv": ms[4], "update_xp": ms[5], "scalars": ms[6], "sum": ms[7]} if ms[2] >= 0 else
                      {"apply_K": ms[0], "pass1_r_update_plane_fft": ms[1], "pass2_pencil_fft_solve": ms[3],
                       "pass3_plane_ifft_update": ms[5], "scalars": ms[6], "sum": ms[7]}),
        "e2e": {"value": e2e_value, "unit": "DOF*it/s",
                "h2d_bytes_per_step": int(world * (ph_host.nbytes + cm.nbytes + e.nbytes)),
                "d2h_bytes_per_step": int(world * (u_host.nbytes + avg.nbytes)), "steps": e2e_steps},
        "clocks": clocks,
        **({"interconnect": nvlink} if nvlink else {}),
        **({"slab_check": slab_check} if slab_check else {}),
        "gpu_launches": int(launches),
        "input_generation_s": t_inputs,
    }
    return out


def cpu_workload(args):
    """The configuration's inputs for the CPU arms WITHOUT the product library:
    inputs.py is loaded by path (no package import, so libhomfe_gpu.so is
    never mapped) with the oracle's or_uniform as its RNG (the same
    std::mt19937_64 stream, so the phase map is byte-identical to the GPU
    arm's)."""
    import importlib.util
    from oracle import oracle
    name = "homfe_inputs_cpu"
    if name not in sys.modules:
        spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "paper_2203_02962_b200", "inputs.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules[name] = mod
        spec.loader.exec_module(mod)
        mod.set_uniform_source(oracle.uniform_source())
    mod = sys.modules[name]
    cfg = mod.config(args.config, n=args.n, contrast=args.contrast)
    return cfg, cfg.phases(), cfg.tangents()


def oracle_pcg_sample(cfg, ph, tans, warm, timed, threads, pre_cache={}):
    """The reference algorithm (oracle: impulse-probed blocks, PCG of
    solver.cpp:50-97, phase-indexed tangent) on the configuration itself from
    its Newton right-hand side; returns the steady_clock seconds of each of
    the `timed` iterations after `warm` untimed ones. Assembly excluded (it is
    setup, once per solve, in the reference too)."""
    from oracle import oracle
    from oracle.cfgutil import newton_rhs
    oracle.set_threads(threads)
    c = cfg.components
    key = (tuple(cfg.dims), cfg.stencil, c)
    if key not in pre_cache:
        pre_cache.clear()
        og = oracle.Grid(cfg.dims, [1.0] * cfg.dim, cfg.stencil)
        if cfg.reference == "explicit":
            cref = tans[cfg.reference_phase]
        else:
            f = np.bincount(ph, minlength=len(tans)).astype(float) / ph.size
            cref = np.einsum("p,pij->ij", f, tans)
        t0 = time.perf_counter()
        pre = oracle.Preconditioner(og, cref, c)
        b = newton_rhs(cfg.dims, [1.0] * cfg.dim, c, tans, ph, cfg.load)
        pre_cache[key] = (og, pre, b, time.perf_counter() - t0)
    og, pre, b, t_setup = pre_cache[key]
    _, t = oracle.pcg_timed(og, c, tans, ph, pre, b, warm + timed)
    oracle.set_threads(1)
    return t[warm:], t_setup


def host_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def cpu_baseline(args, cpu_inputs=None):
    """cpu_baseline of the GPU arm's line: the reference algorithm (oracle)
    on the box's host cores, on a bounded sample of the same workload: the
    configuration itself, 2 PCG iterations after 1 warm-up."""
    cfg, ph, tans = cpu_inputs or cpu_workload(args)
    threads = host_threads()
    t, t_setup = oracle_pcg_sample(cfg, ph, tans, 1, 2, threads)
    return {"value": cfg.dof * len(t) / float(t.sum()), "unit": "DOF*it/s", "cores": threads, "kind": "port",
            "sample": f"{args.config} at {'x'.join(map(str, cfg.dims))} ({cfg.dof} DOF), the configuration itself: "
                      f"{len(t)} PCG iterations (after 1 warm-up) of the oracle restatement of the reference "
                      f"(probed blocks, per-quad loop order, own FFT) from the Newton RHS on {threads} host threads; "
                      f"assembly ({t_setup:.1f} s) excluded",
            "seconds": float(t.sum())}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path on the box's host cores.
    The reference itself cannot be built here (Eigen3, FFTW3 and vendor/
    are absent), so the oracle restatement of its algorithm runs: threaded
    timing variant on every core this process may use, on the configuration
    itself (same config object as the GPU arm); one step = one PCG iteration
    of that configuration (a full solve is 155 iterations of ~4 s). The
    single-core figure (the reference is single-threaded by design,
    homog.cpp:41-43) is measured beside it on one pinned core."""
    if rank != 0:
        return None
    cfg, ph, tans = cpu_workload(args)
    threads = host_threads()
    t, t_setup = oracle_pcg_sample(cfg, ph, tans, args.warmup, args.steps, threads)
    value = cfg.dof * len(t) / float(t.sum())
    # single core, pinned (taskset -c <first allowed core> equivalent)
    single = None
    if not args.no_single_core:
        aff = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
        try:
            if aff:
                os.sched_setaffinity(0, {aff[0]})
            t1, _ = oracle_pcg_sample(cfg, ph, tans, 0, 1, 1)
        finally:
            if aff:
                os.sched_setaffinity(0, set(aff))
        single = {"value": cfg.dof / float(t1[0]), "unit": "DOF*it/s", "cores": 1,
                  "sample": "1 PCG iteration of the same configuration, serial oracle (reference loop order), "
                            "pinned to one core", "seconds": float(t1[0])}
    sample = (f"{args.config} at {'x'.join(map(str, cfg.dims))} ({cfg.dof} DOF), the configuration itself: "
              f"{args.steps} timed PCG iterations after {args.warmup} warm-up, oracle restatement of the reference "
              f"(probed blocks, phase-indexed tangent, own FFT) from the Newton RHS, {threads} host threads "
              f"(two-colour plane sweep of the fused operator, FFT lines, frequencies and vector entries split "
              f"over the cores); assembly {t_setup:.1f} s excluded")
    return {"metric": "DOF·PCG-iterations/s", "value": value, "unit": "DOF*it/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(t.sum()) / len(t) * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic: seeded RSA inclusions / GRF per SURVEY 8(d)",
            "config": workload_config(args, cfg),
            "cpu_baseline": {"value": value, "unit": "DOF*it/s", "cores": threads, "kind": "port", "sample": sample},
            "single_core": single,
            "e2e": {"value": value, "unit": "DOF*it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "step": "one PCG iteration of the configuration (K apply, update, M^-1 with two FFT sweeps, dots)",
            "note": "reference not buildable in this image (Eigen3, FFTW3, vendor/ absent); its algorithm is "
                    "timed through the oracle restatement, with no product library loaded in this process"}


def _emit(out):
    """The one JSON line, on the real stdout (see main: fd 1 is stderr while
    libraries run, so banners such as NCCL's cannot interleave with it)."""
    os.write(_JSON_FD, (json.dumps(out) + "\n").encode())


_JSON_FD = 1


def main():
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=None, help="override grid size (c3/c4/c5)")
    ap.add_argument("--contrast", type=float, default=None)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-single-core", action="store_true", help="--impl reference: skip the 1-core figure")
    ap.add_argument("--slab", action="store_true", help="use the slab (multi-GPU) context even at N=1")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        r = subprocess.run(cmd, stdout=_JSON_FD)
        sys.exit(r.returncode)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "native":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl")
        else:
            dist.init_process_group("gloo")

    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            _emit(out)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    out = run_gpu(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_baseline(args)
            out["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        _emit(out)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
