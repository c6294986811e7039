#!/usr/bin/env python
"""Benchmark of the hot path: the time-stepped 3-D acoustic FD operator on B200.

Workload (BASELINE.json configs[1], the paper's roofline config): 3-D acoustic isotropic,
256^3 grid per GPU, space order 8 (headline; SO 4/12/16 reported in "sweep"), h = 10 m,
c = 1500 m/s, dt = cfl_dt, Ricker 10 Hz source at the centre, no damping.  A bench "step"
is one time step of the operator over the whole grid.  With N GPUs the grid is
256N x 256 x 256 in N z-slabs (reference dim 0) with the SO/2-plane halo exchange over
NVLink peer memory (weak scaling).

  value     GPts/s of the whole job, inputs resident in HBM, CUDA events on the operator's
            stream, max over ranks
  e2e       same metric through the public API with host buffers: handle creation (H2D of
            m, damp, wavelet), H2D of the 3 initial levels from pinned memory, K steps, D2H of
            the 3 final levels and the per-step max|u| (the exec::run contract)
  roofline  algorithmic 20 B/point (read u[t], u[t-1], m, damp; write u[t+1]) / mean stencil
            launch time vs the measured HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline  the reference's own exec::run (basic IET, all host threads) on a bounded
            sample of the same workload (rank 0, N=1)

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2|c4]

--gpus N without torchrun re-launches itself under torch.distributed.run with N ranks (one per
GPU); under torchrun WORLD_SIZE must equal N.  --workload c4 is BASELINE config 4: 512^3 global,
SO 8, absorbing layer (damp_width 10, damp_max 2e-5), strong scaling over the N GPUs.
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

METRIC = "GPts/s & % HBM roofline (3D acoustic, 256³, SO 4–16) at 1/2/4/8 B200 vs CPU"
BYTES_PER_POINT = 20  # u[t], u[t-1], m, damp read + u[t+1] written, FP32 (SURVEY §8(d) convention)
# bytes the kernel must move per point: u[t], u[t-1], B = 1/(m+g) read + u[t+1] written; the A tile
# (the damping coefficient) only where damp != 0, so 16 B/pt on an undamped grid
BYTES_REQUIRED_UNDAMPED = 16
DAMP_C4 = 3 * 1500.0 / (10 * 10.0) / 1500.0 ** 2  # config 4 layer: 3c/(width h) x m-scale ~ 2e-5
FLOPS_AGGRESSIVE = {2: 24, 4: 34, 8: 57, 12: 75, 16: 93}  # reference's count_scalar_ops
FLOPS_BASIC = {2: 69, 4: 105, 8: 165, 12: 225, 16: 285}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """SM clock and throttle-reason sampling DURING the timed region (B200_PROFILING.md clocks
    line).  NVML (pynvml) is polled every ~2 ms from a thread between start() and stop(), which
    bracket exactly the timed steps (the step loop blocks in the driver with the GIL released);
    without pynvml it falls back to nvidia-smi at 100 ms."""

    _REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
                ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
                ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
                ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap")]

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None
        self.thread = None
        self.samples = []
        self.n_before = 0
        self.nv = None

    def start(self):
        try:
            import threading

            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nv = (nv, h)
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.running = True

            def poll():
                while self.running:
                    try:
                        self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                             int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            # the poller must be running before the timed region opens (a bench line once carried
            # a single sample of a 50 ms region)
            t_end = time.time() + 0.5
            while len(self.samples) < 3 and time.time() < t_end:
                time.sleep(0.001)
            self.n_before = len(self.samples)
            return
        except Exception:
            self.nv = None
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)

    def stop(self):
        if self.nv is not None:
            self.running = False
            self.thread.join(timeout=2)
            nv = self.nv[0]
            if not self.samples:
                return None
            reasons = set()
            for _, r in self.samples:
                for name, attr in self._REASONS:
                    if r & int(getattr(nv, attr, 0)):
                        reasons.add(name)
            sm = [c for c, _ in self.samples[self.n_before:]] or [c for c, _ in self.samples]
            return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": self.smax, "reasons": sorted(reasons),
                    "samples": len(sm), "source": "nvml, 2 ms polling inside the timed region"}
        if self.proc is None:
            return None
        time.sleep(0.2)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi, 100 ms"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allsum(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def traffic_from_profiles(so, n=256):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the stencil kernel, from the
    committed ncu capture: the steady-state one (a range of consecutive launches with
    --cache-control none, so u[t+1] written back from L2 is counted) when present, else the
    cold-cache per-launch capture.  Returns (bytes, kind)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        st = d.get("k_tma_steady", {}).get(f"n{n}_so{so}")
        if st:
            return st["dram_bytes_per_launch"], "steady-state (ncu range, --cache-control none)"
        if n == 256:
            return d["k_tma"][f"so{so}"]["dram_bytes_per_launch"], "cold-cache single launch (ncu)"
    except Exception:
        pass
    return None, None


def host_threads():
    """Host cores this process may use. Passed to the CPU arms explicitly: torchrun exports
    OMP_NUM_THREADS=1 to every rank, which would otherwise pin the reference to one thread."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def pinned(shape):
    import torch
    return torch.empty(shape, dtype=torch.float32, pin_memory=True).numpy()


def link_report(op, rank, device):
    """One line per rank on stderr: the slab, the neighbours' devices and how each halo exchange
    is ordered (fused = inside the stencil kernel over peer memory)."""
    st = op.stats()
    lo, hi = op.slab
    print(f"[rank {rank}] device {device} slab [{lo},{hi}) grid {st.grid} CTAs | "
          f"lower: device {st.peer_lo} fused {st.fused_lo} | upper: device {st.peer_hi} fused {st.fused_hi}",
          file=sys.stderr, flush=True)


def hold_stream(op, device, us=400):
    """Keep the operator's stream busy for ~`us` (a device sleep) while the host enqueues the timed
    launches, so the first timed launch does not wait on host-side launch latency: the events
    around the time loop then bracket back-to-back device work only (what one CUDA-graph launch of
    the loop would give).  Without it a 20-step region carries ~30 us of enqueue gap (3.5 % at SO 8).
    Host costs are measured separately, in `e2e`."""
    import torch
    s = torch.cuda.ExternalStream(op.stream_ptr(), device=device)
    with torch.cuda.stream(s):
        torch.cuda._sleep(int(us * 1e-6 * 2.0e9))


def measure_operator(P, D, prob, args, rank, world, device, slab, m, damp, steps, warm):
    """Device-resident GPts/s of `prob` over this rank's slab (max over ranks)."""
    o2 = P.Operator(prob, form="factorised", device=device, slab=slab, m=m, damp=damp)
    if world > 1:
        D.exchange_and_link(o2, rank, world)
    o2.apply(warm, 0)
    barrier(world)
    hold_stream(o2, device)
    o2.apply_async(steps, warm)
    o2.collect(steps)
    barrier(world)
    t = allmax(o2.stats().device_ms * 1e-3, world)
    lo, hi = o2.slab
    so = prob.space_order
    hh = so // 2
    n0, n1, n2 = prob.shape
    pl = (min(hi, n0 - hh) - max(lo, hh)) * (n1 - so) * (n2 - so)
    o2.close()
    return allsum(pl, world) * steps / t / 1e9, pl


def run_ours(args, rank, world, local):
    import torch

    import paper_1912_00695_b200 as P
    from paper_1912_00695_b200 import dist as D

    ndev = torch.cuda.device_count()
    if ndev == 0:
        raise SystemExit("no CUDA device")
    if ndev < world and not args.allow_shared_gpu:
        raise SystemExit(f"{world} ranks but only {ndev} visible GPU(s): one rank per GPU "
                         f"(--allow-shared-gpu runs ranks on shared devices, for plumbing tests only)")
    device = local % ndev
    n, so, K, W = args.n, args.so, args.steps, args.warmup
    c4 = args.workload == "c4"
    scaling = args.scaling or ("strong" if c4 else "weak")
    shape = (n, n, n) if scaling == "strong" else (n * world, n, n)
    damp_max = DAMP_C4 if c4 else 0.0
    nt_total = max(K, 1000) + W + 8
    prob = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0), space_order=so,
                                                   steps=nt_total, damp_max=damp_max, damp_width=10))
    slab = D.slab_bounds(shape[0], world, rank) if world > 1 else None
    m, damp = pinned(shape), pinned(shape)  # user-side host buffers in pinned memory
    m[...] = prob.m_data()
    damp[...] = prob.damp_data()
    op = P.Operator(prob, form="factorised", device=device, slab=slab, m=m, damp=damp)
    if world > 1:
        D.exchange_and_link(op, rank, world)
        link_report(op, rank, device)
    lo, hi = op.slab
    h = so // 2
    pts_local = (min(hi, shape[0] - h) - max(lo, h)) * (n - so) * (n - so)
    pts_total = allsum(pts_local, world)
    # warm-up
    op.apply(W, 0)
    barrier(world)
    torch.cuda.synchronize(device)
    clk = Clocks(device) if rank == 0 else None
    if clk:
        clk.start()
    barrier(world)
    torch.cuda.synchronize(device)
    hold_stream(op, device)
    op.apply_async(K, W)
    op.collect(K)
    torch.cuda.synchronize(device)
    barrier(world)
    st = op.stats()
    clocks = clk.stop() if clk else None
    dev_s = allmax(st.device_ms * 1e-3, world)
    value = pts_total * K / dev_s / 1e9
    launches = int(st.kernel_launches)
    stencil_launches = K  # one fused stencil launch per time step
    mean_launch_s = st.device_ms * 1e-3 / stencil_launches
    hbm, peak_kind = peaks()
    achieved = BYTES_PER_POINT * pts_local * (K / stencil_launches) / mean_launch_s / 1e9
    req = BYTES_PER_POINT if damp_max > 0 else BYTES_REQUIRED_UNDAMPED
    traffic, traffic_kind = traffic_from_profiles(so, n) if not c4 and world == 1 else (None, None)
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(achieved / hbm, 4), "traffic": traffic,
            "peak_kind": peak_kind, "kernel": "k_tma (factorised 2.5D TMA stencil)",
            "bytes_per_point": BYTES_PER_POINT,
            # the same launch time against the bytes this problem requires (16 B/pt undamped: no
            # damping-coefficient tile is loaded) and against the DRAM bytes ncu measured
            "bytes_per_point_required": req,
            "frac_required": round(req * pts_local / mean_launch_s / 1e9 / hbm, 4),
            "dram_frac": (round(traffic / mean_launch_s / 1e9 / hbm, 4) if traffic else None),
            "traffic_kind": traffic_kind}
    # ---- sweep over the other space orders (device-resident, same protocol) ----
    sweep = {}
    if not args.no_sweep and not c4:
        for s2 in (4, 8, 12, 16):
            if s2 == so:
                g2 = value
            else:
                p2 = P.make_wave_problem(P.WaveProblemConfig(shape=shape, spacing=(10.0, 10.0, 10.0),
                                                             space_order=s2, steps=args.sweep_steps + 16))
                g2, _ = measure_operator(P, D, p2, args, rank, world, device, slab, m, damp, args.sweep_steps, 5)
            sweep[f"so{s2}"] = {"gpts": round(g2, 2),
                                "frac": round(BYTES_PER_POINT * g2 / world / hbm, 4),
                                "frac_required": round(BYTES_REQUIRED_UNDAMPED * g2 / world / hbm, 4),
                                "gflops": round(g2 * FLOPS_AGGRESSIVE[s2], 1),
                                "oi_flop_per_byte": round(FLOPS_AGGRESSIVE[s2] / BYTES_PER_POINT, 3)}
    # ---- BASELINE config 4 geometry on this node (512^3 global, SO 8, absorbing layer): the
    # damped case, where the damping-coefficient tiles near the faces are loaded ----
    damped = None
    if not args.no_sweep and not c4:
        p4 = P.make_wave_problem(P.WaveProblemConfig(shape=(512, 512, 512), spacing=(10.0, 10.0, 10.0),
                                                     space_order=8, steps=args.sweep_steps + 16,
                                                     damp_max=DAMP_C4, damp_width=10))
        slab4 = D.slab_bounds(512, world, rank) if world > 1 else None
        g4, _ = measure_operator(P, D, p4, args, rank, world, device, slab4, None, None, args.sweep_steps // 2, 5)
        damped = {"workload": "BASELINE config 4: 512^3 global, SO 8, damp_width 10, damp_max %.3g, "
                              "z-slabs over the N GPUs (strong scaling)" % DAMP_C4,
                  "gpts": round(g4, 2), "frac": round(BYTES_PER_POINT * g4 / world / hbm, 4),
                  "steps": args.sweep_steps // 2}
    op.close()
    # ---- end to end through the public API with host buffers ----
    e2e = None
    if not args.no_e2e:
        init = [pinned(shape) for _ in range(3)]
        for a in init:
            a[...] = 0.0
        out = [pinned(shape) for _ in range(3)]

        def e2e_at(steps, reps):
            runs = []
            for _ in range(max(1, reps)):  # median of a few runs: host/PCIe timing varies run to run
                barrier(world)
                torch.cuda.synchronize(device)
                t0 = time.perf_counter()
                o3 = P.Operator(prob, form="factorised", device=device, slab=slab, m=m, damp=damp)
                if world > 1:
                    D.exchange_and_link(o3, rank, world)
                for l in range(3):
                    o3.set_level(l, init[l])
                o3.apply(steps, 0)
                for l in range(3):
                    o3.get_level(l, out[l])
                barrier(world)
                t1 = time.perf_counter()
                o3.close()
                runs.append(allmax(t1 - t0, world))
            e2e_s = float(np.median(runs))
            planes = hi - lo
            # m, the 3 levels (and damp only when the problem is damped: zero damp is not copied)
            h2d = (1 + (1 if float(prob.damp_max) != 0.0 else 0) + 3) * planes * n * n * 4 + \
                4 * prob.source.wavelet.size
            d2h = 3 * planes * n * n * 4 + 4 * steps
            return {"value": round(pts_total * steps / e2e_s / 1e9, 2), "unit": "GPts/s",
                    "h2d_bytes_per_step": int(allsum(h2d, world) / steps),
                    "d2h_bytes_per_step": int(allsum(d2h, world) / steps),
                    "steps": steps, "seconds": round(e2e_s, 4), "runs_seconds": [round(x, 4) for x in runs]}

        e2e = e2e_at(K, args.e2e_reps)
        e2e["includes"] = ("handle create (H2D m, damp if damped, wavelet) + H2D 3 levels (pinned) + K steps + "
                           "D2H 3 levels + per-step max|u|")
        if K != 1000:
            # the copies are a fixed cost per call: the same contract at the paper's 1000 steps
            e2e["at_1000_steps"] = e2e_at(1000, 3)
        if world == 1 and not c4:
            e2e["dropin_exec_run"] = dropin_e2e(n, so, 1000)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not c4:
        cpu = cpu_baseline(n, so, args.cpu_steps)
    if rank == 0:
        res = {
            "metric": METRIC, "value": round(value, 2), "unit": "GPts/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": round(dev_s * 1e3 / K, 5), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
            "config": {"workload": (f"3D acoustic isotropic FD, {n}^3 per GPU (global {shape[0]}x{n}x{n}), "
                                    f"SO {so}, factorised form, c=1500 m/s, h=10 m, dt=cfl_dt, Ricker 10 Hz")
                       if not c4 else
                       (f"BASELINE config 4: 3D acoustic isotropic FD, {n}^3 global over {world} GPU(s), SO {so}, "
                        f"absorbing layer damp_width 10, damp_max {DAMP_C4:.3g}, factorised form"),
                       "grid": list(shape), "space_order": so, "time_steps_timed": K,
                       "points_per_step": int(pts_total),
                       "timed_region": "CUDA events around the K launches on the operator's stream; the stream is "
                                       "held by a ~400 us device sleep while the host enqueues them (no host "
                                       "launch gap inside the region)",
                       "l2": "inputs larger than L2 (%d B/pt x %.1fM pts = %d MB/step > 126 MB)"
                             % (BYTES_PER_POINT, pts_total / 1e6, BYTES_PER_POINT * pts_total / 1e6),
                       "parallelism": f"z-slab x{world} (reference dim 0), peer-memory halo exchange"},
            "gflops": round(value * FLOPS_AGGRESSIVE[so], 1),
            "roofline": roof, "sweep": sweep, "damped": damped,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(res), flush=True)


def dropin_e2e(n, so, steps):
    """exec::run through the reference's own API with the drop-in executor
    (integration/_build/dropin_run: the reference's host code + integration/executor_b200.cpp +
    libswb.so): make_wave_problem -> ... -> build_iet(aggressive) -> exec::run, which returns all
    three levels in the reference's padded Field (pageable std::vector storage).  Median of 3 calls
    after one warm-up call in the same process."""
    exe = os.path.join(ROOT, "integration", "_build", "dropin_run")
    if not os.path.exists(exe):
        return {"unavailable": "integration/_build/dropin_run not built (needs /root/reference at build time)"}
    env = dict(os.environ, DROPIN_REPS="3")
    try:
        p = subprocess.run([exe, "aggressive", str(n), str(n), str(n), str(so), str(steps), "0", "-"],
                           capture_output=True, text=True, timeout=600, env=env)
        kv = dict(x.split("=", 1) for x in p.stdout.split() if "=" in x)
        run_s, wall_s = float(kv["run"]), float(kv["wall"])
    except Exception as e:  # pragma: no cover
        return {"error": f"{e}"}
    pts = (n - so) ** 3 * steps
    cells = n ** 3
    return {"value": round(pts / run_s / 1e9, 2), "unit": "GPts/s", "steps": steps, "seconds": round(run_s, 4),
            "time_loop_seconds": round(wall_s, 4),
            "h2d_bytes_per_step": int((1 + 1) * cells * 4 / steps),
            "d2h_bytes_per_step": int((3 * cells * 4 + 4 * steps) / steps),
            "includes": "exec::run(iet, problem, {}) as called by a reference user: IET classification, "
                        "handle create (H2D m, damp, wavelet), the time loop, D2H of 3 levels straight into "
                        "the padded Field, RunResult assembly"}


def cpu_baseline(n, so, steps):
    """The reference's own exec::run (oracle/_ref, basic IET, all host threads) on a bounded
    sample of the workload; falls back to the C restatement (oracle/port) if _ref is absent."""
    from oracle import bindings as O
    cfg = O.OracleConfig(shape=(n, n, n), space_order=so, steps=steps)
    try:
        if O.ref_available():
            cores = host_threads()
            r = O.ref_run(cfg, threads=cores)
            kind = "reference"
        else:
            cores = host_threads()
            r = O.port_run(cfg, threads=cores)
            kind = "port"
    except Exception as e:  # pragma: no cover
        return {"error": str(e)}
    gp = r["point_updates"] / r["wall_seconds"] / 1e9
    return {"value": round(gp, 6), "unit": "GPts/s", "cores": cores, "kind": kind,
            "sample": f"{n}^3 SO {so}, {steps} time steps of exec::run (basic DSE), "
                      f"RunResult.point_updates / wall_seconds ({r['wall_seconds']:.2f} s)"}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU path on this arm's config (rank 0 only)."""
    if rank != 0:
        return
    from oracle import bindings as O
    n, so = args.n, args.so
    c4 = args.workload == "c4"
    scaling = args.scaling or ("strong" if c4 else "weak")
    shape = (n, n, n) if scaling == "strong" else (n * world, n, n)
    steps = max(1, min(args.steps, args.ref_steps if not c4 else 1))
    cfg = O.OracleConfig(shape=shape, space_order=so, steps=steps, damp_max=DAMP_C4 if c4 else 0.0,
                         damp_width=10)
    use_ref = O.ref_available()
    fn = O.ref_run if use_ref else O.port_run
    cores = host_threads()
    r = fn(cfg, threads=cores)
    gp = r["point_updates"] / r["wall_seconds"] / 1e9
    kind = "reference" if use_ref else "port"
    res = {
        "metric": METRIC, "value": round(gp, 6), "unit": "GPts/s", "n_gpus": world, "steps": steps,
        "warmup": 0, "ms_per_step": round(r["wall_seconds"] * 1e3 / steps, 3), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "fp64-compute/fp32-storage", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": f"3D acoustic isotropic FD, global {shape[0]}x{n}x{n}, SO {so}, basic DSE "
                               f"(exec::run, OpenMP)" + (f", damp_width 10, damp_max {DAMP_C4:.3g}" if c4 else ""),
                   "grid": list(shape), "space_order": so},
        "cpu_baseline": {"value": round(gp, 6), "unit": "GPts/s", "cores": cores, "kind": kind,
                         "sample": f"{steps} time steps of the full grid (bounded sample; the K requested "
                                   f"steps would take {args.steps * r['wall_seconds'] / steps:.0f} s)"},
        "e2e": {"value": round(gp, 6), "unit": "GPts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--so", type=int, default=8)
    ap.add_argument("--sweep-steps", type=int, default=300)
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--ref-steps", type=int, default=3)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-reps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="c2", choices=["c2", "c4"],
                    help="c2: 256^3 per GPU, SO 8 (weak scaling); c4: BASELINE config 4, 512^3 global, SO 8, "
                         "damped (strong scaling)")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"])
    ap.add_argument("--allow-shared-gpu", action="store_true",
                    help="allow more ranks than visible GPUs (plumbing tests on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("warmup must be >= 3")
    if args.workload == "c4" and args.n == 256:
        args.n = 512
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run (the driver does this itself)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.run(cmd).returncode)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}: launch one rank per GPU")
    rank, world, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
