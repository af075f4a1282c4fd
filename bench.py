"""bench.py -- V-cycle throughput of the B200 cell-centered multigrid solver.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference]
                    [--workload cfg3|cfg4] [--size n]

A "step" is one V(2,2)-cycle of the whole hot path on the resident hierarchy
(smoothing, residual+restriction, coarse CG, prolongation, residual norm and
its readback), launched through the C-ABI (mg_vcycle).  Workloads:
  N = 1: BASELINE config 3 -- 512^3, h = 1/512, homogeneous Dirichlet,
         f ~ U[-1,1] (seeded), V(2,2) to 8^3.
  N > 1: config 4 weak scaling -- (512 N) x 512 x 512, channel BCs, charged
         spheres R = 6 at 5 % volume, slabs of 512 planes per GPU.
value = global cells x K / max-over-ranks device time (Mcells/s).
e2e   = the same metric for whole config-3 solves (20 cycles each) through
        the public API with host buffers: per solve the H2D of f from pinned
        memory, 20 cycles and the D2H of Phi, all inside the timed region;
        mg_solve_async overlaps each solve's copies with the neighbouring
        solves' cycles.
--impl reference times the CPU oracle (oracle/, plain C fp64) on a bounded
sample of the same workload on the host cores (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MG V-cycle throughput (Mcells/s, fp64) and achieved HBM GB/s vs peak, 1/2/4/8 GPU"
UNIT = "Mcells/s"
HALF_SWEEP_BYTES_PER_CELL = 12  # other-colour Phi 4 + own f 4 + own Phi 4


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# --------------------------------------------------------------------------
# clocks sampled during the timed region
# --------------------------------------------------------------------------
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting",
               0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x10: "sync_boost",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            try:
                a, b, c = [x.strip() for x in ln.split(",")]
                sm.append(float(a))
                mx.append(float(b))
                bits = int(c, 16)
                for k, v in REASON_BITS.items():
                    if bits & k and v != "gpu_idle":
                        reasons.add(v)
            except Exception:
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


CPU_SAMPLE = 256  # oracle sample edge for cpu_baseline and --impl reference


def oracle_rate(n_sample, warm, cycles):
    """Mcells/s of the oracle (as it stands) on the config-3 recipe at
    n_sample^3: `warm` untimed then `cycles` timed V(2,2)-cycles (each with
    its residual norm), and the seconds they took."""
    import oracle
    from paper_1410_6609_b200 import workloads as W
    oracle.build()
    w = W.cfg3(n_sample, seed=0)
    o = oracle.Oracle(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=8)
    o.set_rhs(w.rhs)
    for _ in range(warm):
        o.vcycle()
    t0 = time.perf_counter()
    for _ in range(cycles):
        o.vcycle()
    dt = time.perf_counter() - t0
    return w.cells * cycles / dt / 1e6, dt, o.nlevels


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(n_sample=CPU_SAMPLE, cycles=2):
    """The oracle as it stands on a bounded sample of the config-3 recipe:
    n_sample^3 cells, V(2,2) to 8^3, one warm-up cycle then `cycles` timed --
    the OpenMP build on all host cores (the headline baseline) and, in a
    child process with OMP_NUM_THREADS=1, single-threaded."""
    cores = int(os.environ.get("OMP_NUM_THREADS", host_cores()))
    val, _, _ = oracle_rate(n_sample, 1, cycles)
    single = None
    try:
        env = dict(os.environ, OMP_NUM_THREADS="1")
        out = subprocess.run(
            [sys.executable, "-c",
             "import sys; sys.path.insert(0, %r); import bench; "
             "print(bench.oracle_rate(%d, 1, 1)[0])" % (ROOT, n_sample)],
            env=env, capture_output=True, text=True, timeout=600)
        single = round(float(out.stdout.strip().splitlines()[-1]), 3)
    except Exception:
        single = None
    return {"value": round(val, 3), "unit": UNIT,
            "cores": cores, "kind": "oracle",
            "single_thread_value": single,
            "host_cores": host_cores(),
            "sample": "config-3 recipe at %d^3 (h=1/%d, U[-1,1], V(2,2) to 8^3), "
                      "1 warm-up + %d timed V-cycles incl. residual norm, "
                      "OpenMP threads=%d; single_thread_value: the same sample, "
                      "1 warm-up + 1 timed cycle, OMP_NUM_THREADS=1"
                      % (n_sample, n_sample, cycles, cores)}


def timestep_regime(mg, W, stream, local, steps=10, warm=2):
    """The paper's own use of the solver (Alg.1): per time step
    the spheres move, f is re-set from them (subsampling 2), one
    warm-started V(3,3)-cycle updates Phi (5 at the first step)
    and the Coulomb forces are computed (Eq.14-15) -- one mg_timestep call.
    Metric: the paper's MLUPS, cells whose Poisson problem is solved per
    second.  Positions are generated before the timed region
    (they stand in for the LBM / pe motion, which is out of scope)."""
    import torch
    w = W.timestep_workload(n=512, seed=0)
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, device=local,
                     stream=stream, min_coarse=8, nu1=3, nu2=3)
    L = np.array(w.shape) * w.h
    pos = [w.centers]
    for k in range(1, steps + warm + 1):
        pos.append(W.move_spheres(pos[-1], w.radii, L, k, seed=0, amplitude=0.005))
    s.timestep(pos[0], w.radii, w.charges, cycles=5, subsample=2)  # first step
    for k in range(1, warm + 1):
        s.timestep(pos[k], w.radii, w.charges, cycles=1, subsample=2)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    res = []
    for k in range(warm + 1, warm + 1 + steps):
        _, _, r = s.timestep(pos[k], w.radii, w.charges, cycles=1, subsample=2)
        res.append(r)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    # breakdown of one step: RHS, V(3,3)-cycle (incl. norm), forces
    parts = {"rhs_ms": [], "vcycle_ms": [], "forces_ms": []}
    for k in range(warm + 1, warm + 4):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        s.set_rhs_from_spheres(pos[k], w.radii, w.charges, subsample=2)
        ev[1].record(stream)
        s.vcycle()
        ev[2].record(stream)
        s.coulomb_forces(pos[k], w.radii, w.charges, subsample=2)
        ev[3].record(stream)
        torch.cuda.synchronize()
        for i, key in enumerate(parts):
            parts[key].append(ev[i].elapsed_time(ev[i + 1]))
    # the step's residual reduction: ||r|| after the cycle over ||r|| of the
    # warm start against the moved spheres' f
    rel = []
    for k in range(warm + 4, warm + 7):
        s.set_rhs_from_spheres(pos[k], w.radii, w.charges, subsample=2)
        r0 = s.residual_norm()
        rel.append(s.vcycle() / r0)
    s.close()
    cells = w.cells
    return {"metric": "MLUPS per time step (paper's MG metric, P:1303-1306)",
            "value": round(cells / (ms * 1e-3) / 1e6, 1), "unit": "MLUPS",
            "ms_per_step": round(ms, 3), "steps": steps,
            "step": "mg_timestep: f from %d moved spheres R=6 (s_f=2) + 1 V(3,3)-"
                    "cycle (warm start) + residual norm + Coulomb forces (s_f=2)"
                    % len(w.radii),
            "workload": "cfg4 box 512^3, channel BCs, 5% spheres, 7 levels",
            "residual_mean": float(np.mean(res)), "residual_max": float(np.max(res)),
            "residual_over_r0_mean": float(np.mean(rel)),
            "residual_note": "absolute ||f - A Phi|| after the step's cycle (the paper "
                             "monitors 1.5e-8 absolute, P:1323-1324); over_r0: the same "
                             "over the warm start's residual for the moved spheres",
            "breakdown_ms": {k: round(float(np.mean(v)), 3) for k, v in parts.items()},
            "paper_context": "91.8 MLUPS per SuperMUC node, 16 Sandy Bridge cores "
                             "(P:1346); context only"}


def fused_norm_variant(mg, W, stream, local, steps=20, warm=3):
    """Reading c11 (mg_opts.fused_norm): the same config-3 cycles with the
    termination norm taken from the level-0 residual+restriction kernel
    (no separate norm pass).  Reported beside the headline, which keeps the
    post-cycle norm (the residual histories of SURVEY 8(c))."""
    import torch
    w = W.cfg3(512, seed=0, with_rhs=False)
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, device=local,
                     stream=stream, min_coarse=8, fused_norm=True)
    s.set_rhs(W.uniform_rhs(w.shape, 0))
    for _ in range(warm):
        s.vcycle()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        s.vcycle()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    cells = int(np.prod(w.shape))
    L = s.nlevels
    s.close()
    model = sum((24 * 4 + 34) * 8.0 ** -l for l in range(L - 1))  # no norm pass
    return {"reading": "c11: cycle norm = level-0 residual after pre-smoothing, "
                       "summed by the residual+restriction kernel",
            "ms_per_cycle": round(ms, 4),
            "value": round(cells / (ms * 1e-3) / 1e6, 2), "unit": UNIT,
            "cycle_model_bytes_per_cell": round(model, 2), "steps": steps}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    n = args.ref_size
    val, dt, nlev = oracle_rate(n, args.warmup, args.steps)
    cores = int(os.environ.get("OMP_NUM_THREADS", host_cores()))
    full = args.size ** 3 * max(args.gpus, 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 3),
        "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg3 recipe, CPU oracle sample %d^3 of the %d-cell workload"
                               % (n, full),
                   "schedule": "V(2,2)", "levels": nlev},
        "cpu_baseline": {"value": round(val, 3), "unit": UNIT, "cores": cores,
                         "kind": "oracle",
                         "sample": "%d^3 cells per step (one V(2,2)-cycle incl. norm)" % n},
        "e2e": {"value": round(val, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_cuda(args):
    import torch
    ws, rank, local = dist_env()
    N = args.gpus
    if ws != N:
        raise SystemExit("--gpus %d but WORLD_SIZE=%d" % (N, ws))
    torch.cuda.set_device(local)
    dist = None
    if N > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1410_6609_b200 import _build
    if rank == 0 or N == 1:
        _build.build()
    if dist is not None:
        dist.barrier()
    from paper_1410_6609_b200 import mg
    from paper_1410_6609_b200 import workloads as W

    n = args.size
    workload = args.workload or ("cfg3" if N == 1 else "cfg4")
    kw = dict(min_coarse=8, nu1=2, nu2=2)
    if N > 1:
        from paper_1410_6609_b200 import dist as D
        uid = D.share_nccl_id(rank, mg.nccl_unique_id)
        kw.update(nranks=N, rank=rank, halo="nccl", nccl_id=uid)
    stream = torch.cuda.Stream(device=local)
    if workload == "cfg3":
        assert N == 1, "cfg3 is the single-GPU configuration"
        w = W.cfg3(n, seed=0, with_rhs=False)
        shape = w.shape
        s = mg.Multigrid(shape, w.h, w.bc_type, w.bc_value, device=local,
                         stream=stream, **kw)
        rhs_host = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        rhs_host.numpy()[...] = W.uniform_rhs(shape, 0)
        s.set_rhs(rhs_host)
        wl = "cfg3: %d^3, h=1/%d, homogeneous Dirichlet, f~U[-1,1] seed 0" % (n, n)
    elif workload == "cfg5":
        # strong scaling: 2048 x 512 x 512 total (scaled by --size/512)
        sc = 512 // n
        w = W.cfg5(scale=sc)
        shape = w.shape
        kw.update(nu1=3, nu2=3)
        s = mg.Multigrid(shape, w.h, w.bc_type, w.bc_value, device=local,
                         stream=stream, **kw)
        s.set_mask(w.solid)
        s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
        rhs_host = None
        wl = ("cfg5: %dx%dx%d bifurcating channel (beam mask), electrodes 0/1, "
              "%d spheres R=4, V(3,3)" % (shape + (len(w.radii),)))
    else:
        w = W.cfg4(P=N, n=n, seed=0)
        shape = w.shape
        s = mg.Multigrid(shape, w.h, w.bc_type, w.bc_value, device=local,
                         stream=stream, **kw)
        s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
        rhs_host = None
        wl = ("cfg4: (%d*%d)x%dx%d weak scaling, channel BCs, %d spheres R=6 (5%%)"
              % (n, N, n, n, len(w.radii)))
    cells = int(np.prod(shape))
    L = s.nlevels

    # ---- warm-up (includes graph capture) ----
    for _ in range(args.warmup):
        s.vcycle()
    # ---- roofline of the dominant kernel (level-0 RBGS half-sweep), live:
    # CUDA events between the phases of recorded cycles (a graph of its own,
    # with event nodes), run right after the warm-up from the same idle state
    # as the timed region (a pause between the two lets the board's power
    # management recover from these cycles) ----
    s.set_profiling(True)
    prof = []
    for _ in range(max(3, min(args.steps, 10))):
        s.vcycle()
        prof.append(s.last_cycle_times())
    s.set_profiling(False)
    for _ in range(2):  # re-record the cycle graphs (one per red buffer)
        s.vcycle()
    torch.cuda.synchronize()
    time.sleep(1.0)
    # ---- timed region: K V-cycles, barrier + sync on both sides ----
    clocks = ClockSampler(local)
    clocks.start()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    norms = []
    for _ in range(args.steps):
        norms.append(s.vcycle())
    e1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    ck = clocks.stop()
    if dist is not None:
        from paper_1410_6609_b200 import dist as D
        ms = D.max_over_ranks(ms, device="cuda")
    launches = s.cycle_launches

    # ---- sustained: the same cycles back to back for ~0.5 s (the board's
    # power management lowers the clocks after ~80 ms of full load; the
    # timed region above is the first K cycles after warm-up) ----
    sustained = None
    if not args.no_sustained:
        nsus = max(1, int(round(500.0 / max(ms / args.steps, 1e-3))))
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(nsus):
            s.vcycle()
        b.record(stream)
        torch.cuda.synchronize()
        # the last fifth of them: the steady state
        tail = max(1, nsus // 5)
        c0 = torch.cuda.Event(enable_timing=True)
        c1 = torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(tail):
            s.vcycle()
        c1.record(stream)
        torch.cuda.synchronize()
        sms = c0.elapsed_time(c1) / tail
        sustained = {"cycles": nsus + tail, "ms_per_cycle_steady": round(sms, 4),
                     "value": round(cells / (sms * 1e-3) / 1e6, 2), "unit": UNIT,
                     "ms_per_cycle_mean": round(a.elapsed_time(b) / nsus, 4),
                     "note": "cycles back to back for ~0.5 s after the timed region; "
                             "steady = the last %d (power-capped clocks)" % tail}

    sm0 = np.mean([p["smooth0_ms"] for p in prof])
    nsm = prof[0]["smooth0_launches"]
    cyc_prof = np.mean([p["cycle_ms"] for p in prof])
    per_launch_ms = sm0 / nsm
    local_cells = cells // N
    # SURVEY 8(d) per-unit figure (12 B per cell and half-sweep) x the cells
    # one launch updates (the rank's level-0 slab)
    alg_bytes = int(HALF_SWEEP_BYTES_PER_CELL * local_cells)
    achieved = alg_bytes / (per_launch_ms * 1e-3) / 1e9
    peak, peak_src = peaks()
    traffic = None
    tf = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            if tj.get("cells") == local_cells and tj.get("kernel") == "k_smooth_march":
                traffic = tj.get("bytes_per_launch")
        except Exception:
            traffic = None
    # whole-cycle model roofline (SURVEY 8(d) byte model)
    model_bytes = 0.0
    nsw = 6 if workload == "cfg5" else 4
    for l in range(L - 1):
        frac = 8.0 ** -l
        model_bytes += (24 * nsw + 34) * frac
    # the norm: 16 B/cell; the split cycle-end norm reads 12 --
    # the black residuals ride on the last black half-sweep; with the
    # look-ahead red sweep the red residuals cost its read of the current
    # red values, 4.  The library reports which path the recorded cycle took
    # (mg_cycle_paths).
    split = bool(s.cycle_paths & mg.MG_PATH_SPLIT_NORM)
    lookahead = bool(s.cycle_paths & mg.MG_PATH_LOOKAHEAD)
    model_bytes += 4 if lookahead else (12 if split else 16)
    cycle_ms = ms / args.steps
    cycle_frac = model_bytes * local_cells / (cycle_ms * 1e-3) / 1e9 / peak

    # ---- e2e: config-3 solves through the public API, host buffers ----
    # Each step = one independent solve: H2D of f from pinned host memory,
    # Phi := 0, 20 V(2,2)-cycles (each with its residual norm), D2H of Phi.
    # mg_solve_async pipelines them: the next problem's upload and the
    # previous one's download run on copy streams while the cycles run; the
    # timed region spans all steps, from an event before the first H2D to the
    # end of the last D2H (mg_wait).
    e2e = None
    if workload == "cfg3" and not args.no_e2e:
        ncyc = 20
        nsteps = max(4, min(2 * args.steps, 40))  # pipeline fill/drain amortised
        outs = [torch.empty(shape, dtype=torch.float64, pin_memory=True)
                for _ in range(2)]
        s.solve_async(rhs_host, outs[0], 1)  # warm-up: staging, copy streams
        s.wait()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(nsteps):
            s.solve_async(rhs_host, outs[k % 2], ncyc)
        res_e2e = s.wait()            # compute and copy streams drained
        e1.record(stream)
        torch.cuda.synchronize()
        dt = e0.elapsed_time(e1) * 1e-3
        e2e = {"value": round(cells * ncyc * nsteps / dt / 1e6, 2), "unit": UNIT,
               "h2d_bytes_per_step": cells * 8, "d2h_bytes_per_step": cells * 8,
               "step": "one config-3 solve: H2D f (pinned) + Phi=0 + %d V(2,2)-cycles "
                       "+ D2H Phi (mg_solve_async)" % ncyc,
               "steps": nsteps, "ms_per_step": round(dt * 1e3 / nsteps, 2),
               "pipeline": "uploads / downloads on library copy streams overlap "
                           "the previous / next solve's cycles",
               "final_residual": res_e2e}

    if workload == "cfg4" and not args.no_e2e:
        # end to end per step: H2D of the step's input (the sphere list) and
        # the RHS built from it, Phi := 0, the 11 V(2,2)-cycles config 4
        # needs to reach 1e-8, D2H of the rank's Phi slab
        ncyc, nsteps = 11, max(2, min(args.steps, 10))
        outs = [torch.empty(s.local_shape(0), dtype=torch.float64, pin_memory=True)
                for _ in range(2)]
        s.get_solution_async(outs[0])  # warm-up: staging slots, copy stream
        s.wait()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        a_ = torch.cuda.Event(enable_timing=True)
        b_ = torch.cuda.Event(enable_timing=True)
        a_.record(stream)
        for k in range(nsteps):
            s.zero_solution()
            s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
            for _ in range(ncyc):
                s.vcycle()
            # D2H of this step's Phi on the library's copy stream, overlapping
            # the next step's RHS and cycles (mg_get_solution_async)
            s.get_solution_async(outs[k % 2])
        s.wait()
        b_.record(stream)
        torch.cuda.synchronize()
        dt = a_.elapsed_time(b_) * 1e-3
        if dist is not None:
            from paper_1410_6609_b200 import dist as D
            dt = D.max_over_ranks(dt, device="cuda")
        e2e = {"value": round(cells * ncyc * nsteps / dt / 1e6, 2), "unit": UNIT,
               "h2d_bytes_per_step": int(5 * 8 * len(w.radii)),
               "d2h_bytes_per_step": int(8 * cells // N),
               "step": "set_rhs_from_spheres (H2D of the %d-sphere list) + Phi=0 + "
                       "%d V(2,2)-cycles + D2H of the rank's Phi slab "
                       "(mg_get_solution_async: overlaps the next step)"
                       % (len(w.radii), ncyc),
               "steps": nsteps, "ms_per_step": round(dt * 1e3 / nsteps, 2)}

    line = {
        "metric": METRIC,
        "value": round(cells * args.steps / (ms * 1e-3) / 1e6, 2),
        "unit": UNIT, "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(cycle_ms, 4), "higher_is_better": True,
        "scaling": "strong" if workload == "cfg5" else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": wl, "global_cells": cells, "levels": L,
                   "schedule": ("V(3,3)" if workload == "cfg5" else "V(2,2)")
                               + ", RBGS red-black, alpha=2, CG coarsest",
                   "parallelism": "x-slab x%d (NCCL halo)" % N if N > 1 else "single GPU",
                   "l2": "inputs larger than L2 (hierarchy %.2f GB vs 126 MB L2); no flush"
                         % (mg.workspace_bytes(shape, min_coarse=8) / 1e9 / N)},
        "roofline": {"bound": "hbm",
                     "kernel": "k_smooth_march (level-0 RBGS half-sweep)",
                     "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "alg_bytes_per_launch": alg_bytes,
                     "avg_launch_ms": round(per_launch_ms, 5),
                     "share_of_cycle": round(sm0 / cyc_prof, 4),
                     "peak_source": peak_src,
                     "peak_note": "measured copy bandwidth (1:1 read/write); the "
                                  "half-sweep reads 2 B per B written and the "
                                  "cycle model can exceed it slightly",
                     "cycle_model_frac": round(cycle_frac, 4),
                     "breakdown_ms": {k: round(float(np.mean([p[k] for p in prof])), 4)
                                      for k in prof[0]},
                     "cycle_model_bytes_per_cell": round(model_bytes, 2),
                     "norm_path": ("look-ahead red sweep" if lookahead else
                                   "split" if split else "full pass")},
        "gpu_launches": int(launches * args.steps),
        "clocks": ck,
        "e2e": e2e,
        "sustained": sustained,
        "final_residual": norms[-1] if norms else None,
        "paper_context": "the paper's MG: 91.8 MLUPS per 16-core SuperMUC node "
                         "(V(3,3) time steps, P:1346), 121,083 MLUPS on 2048 nodes "
                         "(P:1434); other hardware and workload, context only",
    }
    s.close()
    if N == 1 and workload == "cfg3" and not args.no_ts:
        try:
            line["timestep_regime"] = timestep_regime(mg, W, stream, local)
        except Exception as ex:  # reported, never fatal
            line["timestep_regime"] = {"error": repr(ex)}
    if N == 1 and workload == "cfg3" and not args.no_fused:
        try:
            line["fused_norm"] = fused_norm_variant(mg, W, stream, local)
        except Exception as ex:  # reported, never fatal
            line["fused_norm"] = {"error": repr(ex)}
    if rank == 0 and N == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(args.cpu_size)
        except Exception as ex:  # reported, never fatal
            line["cpu_baseline"] = {"error": repr(ex)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--workload", default=None, choices=[None, "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--cpu-size", type=int, default=CPU_SAMPLE)
    ap.add_argument("--ref-size", type=int, default=CPU_SAMPLE)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ts", action="store_true",
                    help="skip the time-stepping regime measurement")
    ap.add_argument("--no-sustained", action="store_true",
                    help="skip the sustained (0.5 s back-to-back) cycle measurement")
    ap.add_argument("--no-fused", action="store_true",
                    help="skip the fused-termination-norm variant (reading c11)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_cuda(args)


if __name__ == "__main__":
    sys.exit(main())
