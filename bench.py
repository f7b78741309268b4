#!/usr/bin/env python
"""bench.py -- throughput of the ESDG right-hand side + LSRK update on B200.

    python bench.py --gpus N --steps K --warmup W          (our arm)
    python bench.py --impl reference --gpus N --steps K --warmup W

A "step" is one five-stage LSRK step (5 RHS evaluations + 5 updates) of the
rising-thermal-bubble case (BASELINE.json configs[1]: N=4, ~1e8 DOF per GPU,
FP64). metric = RHS DOF-updates/s = elements * (N+1)^3 * RHS evaluations / s,
whole job. For N > 1 the driver launches this file under torchrun, one rank
per GPU; the mesh grows with N (configs[4], weak scaling) and the face-trace
halo moves over NCCL while the volume kernel runs.

Prints ONE JSON line on rank 0. See DESIGN.md "Measurement" for every field.
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

METRIC = "rhs_dof_updates_per_s"
UNIT = "DOF-updates/s"

# configs[4] of BASELINE.json: base lattice per GPU count at refinement 5
WEAK_BASE = {1: (3, 3, 3), 2: (6, 3, 3), 4: (6, 6, 3), 8: (6, 6, 6)}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"])
    ap.add_argument("--path", default="stage", choices=["stage", "fused", "split"])
    ap.add_argument("--refinement", type=int, default=5)
    ap.add_argument("--base", type=int, nargs=3, default=None,
                    help="override the base lattice (default: configs[4] table)")
    ap.add_argument("--case", default=None, choices=["bubble", "baroclinic"],
                    help="default: bubble (weak scaling), baroclinic (strong scaling)")
    ap.add_argument("--scaling", default=os.environ.get("ESDG_BENCH_SCALING", "weak"),
                    choices=["weak", "strong"],
                    help="weak: BASELINE.json configs[4], ~1e8 DOF per GPU (bubble); strong: configs[3], "
                         "the fixed 3,145,728-element (~4e8 DOF) baroclinic channel cut into --gpus parts")
    ap.add_argument("--no-stream-e2e", action="store_true",
                    help="e2e: skip the streamed three-member ensemble (three pinned host states "
                         "per rank), report the coupled step_swap figure as e2e.value")
    ap.add_argument("--overlap", default="auto", choices=["auto", "on", "off"],
                    help="N > 1: interior element groups run while the traces travel (on), or the "
                         "kernel waits for them and runs as one launch (off); auto times two steps "
                         "of each after the warm-up and keeps the faster (the two launches cost "
                         "2.5-5.6 %% of a step, an NVLink exchange tens of microseconds)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "torch"],
                    help="N > 1: ncclSend/ncclRecv issued by the library (default) or the "
                         "torch.distributed callback (halo.py)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    if args.case is None:
        args.case = "baroclinic" if args.scaling == "strong" else "bubble"
    return args


# --------------------------------------------------------------------------
# clocks: sampled with nvidia-smi DURING the timed region
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc, self.first, self.warm = device, [], None, 0, 0

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def wait_first(self, timeout=8.0):
        """Blocks until nvidia-smi has delivered its first row (its start-up can
        take longer than the whole timed region on a fresh box); from then on a
        row arrives every 100 ms."""
        t0 = time.perf_counter()
        while self.proc and not self.rows and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)
        self.warm = len(self.rows)      # the warm-up starts here

    def mark(self):
        """Rows before this call (idle, warm-up) do not count."""
        self.first = len(self.rows)

    def stop(self):
        if not self.proc:
            return
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.proc = None

    def snapshot(self, first=None):
        """Median SM clock and the throttle reasons seen since mark(). A timed
        region shorter than the sampling period may see no row at all: the
        rows since the warm-up began (the same load) are used then, and the
        result says so."""
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": ["nvidia-smi unavailable"]}
        first = self.first if first is None else first
        if first == self.first and len(self.rows) <= self.first and self.first > self.warm:
            out = self.snapshot(self.warm)
            out["window"] = "warm-up + timed region (no sample fell into the timed region)"
            return out
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in list(self.rows[first:]):
            if len(r) < 7:
                continue
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except ValueError:
                continue
            for n, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# --------------------------------------------------------------------------
# algorithmic work per element per RHS (the
# reference's own PerfRecord model, diagnostics.cpp:33-81)
# --------------------------------------------------------------------------
def work_model(nq: int, bytes_per_real: int):
    n2, n3, h = nq * nq, nq ** 3, nq // 2
    return {
        "volume_flops": n3 * (189 * h + 205),
        "volume_bytes": (11 * n3 + n2) * bytes_per_real,
        "surface_flops": 843 * n2,
        "surface_bytes": 66 * n2 * bytes_per_real,
        "update_bytes": 15 * n3 * bytes_per_real,
    }


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "MEASURED_PEAKS.json"
    return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str, order: int, precision: str, case: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    ("stage", "fused", "volume") from the committed ncu captures of this very
    workload (profiles/traffic.json, keyed kernel/N<order>/<precision>/<case>;
    tools/collect_traffic.sh regenerates it), or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        with open(path) as f:
            table = json.load(f)
        return table.get(f"{kernel}/N{order}/{precision}/{case}")
    return None


# --------------------------------------------------------------------------
# CPU arm: the reference's own Solver<Real> (oracle/_ref) or the oracle port
# --------------------------------------------------------------------------
def cpu_has_avx2_fma() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            flags = next((l for l in f if l.startswith("flags")), "")
        return " avx2 " in flags + " " and " fma " in flags + " "
    except OSError:
        return False


def run_cpu_reference(order, precision, target_seconds, steps=None, warmup=1):
    """Times Solver::step on a bounded sample of the bench workload: the same
    bubble case, same order and precision, on a 16^3-element box (the
    reference cannot hold 1e8 DOF: 17 Reals of flux record per face node)."""
    from oracle import pyoracle as po
    threads = os.cpu_count() or 1
    if po.reference_available():
        fast = po.reference_available(fast=True) and cpu_has_avx2_fma()
        ora, kind = po.Oracle("reference", fast=fast), "reference"
        build = "-O3 -march=x86-64-v3" if fast else "-O2"
    else:
        ora, kind, build, threads = po.Oracle("port"), "port", "-O2 (C restatement, serial)", 1
    refinement = 4
    mesh = ora.mesh(po.bubble_mesh_config(refinement))
    ranks = max(1, min(threads, mesh.ne))
    solver = mesh.solver(order, precision, ranks=ranks) if kind == "reference" else mesh.solver(order, precision)
    solver.init_case(po.CASE_BUBBLE_SHARP)
    dt = solver.compute_dt(0.5)
    dof = mesh.ne * solver.n3
    for _ in range(max(1, warmup)):
        t0 = time.perf_counter()
        solver.step(dt)
        one = time.perf_counter() - t0
    if steps is None:
        steps = int(max(2, min(200, target_seconds / max(one, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(steps):
        solver.step(dt)
    wall = time.perf_counter() - t0
    value = dof * 5 * steps / wall
    return {
        "value": value, "unit": UNIT, "cores": ranks if kind == "reference" else 1, "kind": kind,
        "sample": (f"bubble N={order} {precision} on {mesh.ne} elements ({dof} DOF), {steps} LSRK steps, "
                   f"Solver<Real>::step with ranks={ranks} worker threads, built {build}"),
        "ms_per_step": 1e3 * wall / steps, "steps": steps,
    }


def main_reference(args, rank):
    if rank != 0:
        return
    res = run_cpu_reference(args.order, args.precision, args.cpu_seconds,
                            steps=args.steps, warmup=args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": f"rising thermal bubble, N={args.order}, {args.precision}: "
                               "bounded CPU sample of BASELINE.json configs[1]",
                   "sample": res["sample"]},
        "cpu_baseline": {"value": res["value"], "unit": UNIT, "cores": res["cores"],
                         "kind": res["kind"], "sample": res["sample"]},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def main_b200(args, rank, local_rank, world):
    import torch
    from paper_2605_16684_b200 import capi

    dist = None
    if world > 1:
        # the NCCL log lets whoever runs this count ranks and see the transport
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        import torch.distributed as dist
    # ESDG_BENCH_DIST_BACKEND=gloo (tests only): the ranks of a one-GPU box share
    # cuda:0 and torch.distributed runs over gloo on host tensors, so that the
    # multi-rank flow of this file can be exercised where NCCL refuses two ranks
    # on one device (tests/test_gpu_bench_ranks.py)
    backend = os.environ.get("ESDG_BENCH_DIST_BACKEND", "nccl") if world > 1 else None
    device = local_rank % max(torch.cuda.device_count(), 1) if backend == "gloo" else local_rank
    torch.cuda.set_device(device)
    if world > 1:
        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{device}"))
    cdev = "cpu" if backend == "gloo" else f"cuda:{device}"   # where collectives' tensors live

    nq = args.order + 1
    rb = 8 if args.precision == "f64" else 4
    base = tuple(args.base) if args.base else WEAK_BASE.get(world, (3 * world, 3, 3))
    if args.case == "bubble":
        scale = tuple(b / 3.0 for b in base) if not args.base else (1, 1, 1)
        cfg = capi.bubble_mesh_config(args.refinement, False, base, scale)
        settings = capi.Settings(1, 0, 0.0, 0.0, 0.0)
        case_id = capi.CASE_BUBBLE_SHARP
    else:
        # strong: configs[3], the same 384 x 128 x 64 mesh for every N;
        # weak: configs[2] per GPU, widened in y with N
        base = tuple(args.base) if args.base else ((12, 4, 2) if args.scaling == "strong" else (12, 2 * world, 1))
        cfg = capi.channel_mesh_config(args.refinement, base)
        settings = capi.Settings(1, 2, 1e-4, 1.6e-11, 3e6)
        case_id = capi.CASE_BAROCLINIC_JET
    mesh = capi.Mesh(cfg)

    exchange = None
    if world > 1 and args.exchange == "nccl":
        # the exchange lives in the library: rank 0 makes the NCCL unique id,
        # torch.distributed (plumbing) hands it round, no Python runs in a step
        uid = torch.zeros(128, dtype=torch.uint8, device=cdev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(capi.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        solver = None
        try:
            solver = capi.GpuSolver(mesh, args.order, args.precision, settings=settings,
                                    nccl=(world, rank, device, bytes(uid.cpu().numpy().tobytes())))
        except Exception as exc:  # noqa: BLE001 -- every rank must take the same way out
            print(f"[bench] rank {rank}: library-side NCCL exchange unavailable ({exc})", file=sys.stderr)
        ok = torch.tensor([1 if solver is not None else 0], dtype=torch.int32, device=cdev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            # fall back to the torch.distributed callback on all ranks alike
            solver = None
            args.exchange = "torch"
    if world > 1 and args.exchange == "torch":
        from paper_2605_16684_b200 import halo
        solver = capi.GpuSolver(mesh, args.order, args.precision, settings=settings,
                                distributed=(world, rank, device))
        cb, exchange = halo.make_exchange_callback(solver, device)
        solver.exchange_impl = cb
    elif world == 1:
        solver = capi.GpuSolver(mesh, args.order, args.precision, settings=settings, devices=[device])
    assert solver is not None
    if world > 1 and solver.end - solver.begin >= mesh.ne:
        raise RuntimeError(f"rank {rank} of {world} holds the whole mesh: the partitioned solver was not created")
    solver.set_path({"stage": capi.PATH_STAGE, "fused": capi.PATH_FUSED, "split": capi.PATH_SPLIT}[args.path])
    solver.init_case(case_id)
    dt_local = solver.compute_dt(0.5)
    if world > 1:
        t = torch.tensor([dt_local], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        dt_local = float(t.item())
    dt = dt_local
    n_local = solver.end - solver.begin
    dof_total = mesh.ne * solver.n3

    stream = torch.cuda.ExternalStream(solver.stream, device=device)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(device)

    # clocks: nvidia-smi is started before the warm-up and must have delivered
    # a row before the timed region begins; only rows of the timed region count
    sampler = ClockSampler(device)
    if rank == 0:
        sampler.start()
        sampler.wait_first()

    # ---- warm-up ----------------------------------------------------------
    for _ in range(max(args.warmup, 3)):
        solver.step(dt, check_state=True)
    solver.sync()
    overlap_choice = None
    if world > 1:
        probe = {}
        modes = ["on", "off"] if args.overlap == "auto" else [args.overlap]
        for mode in modes:
            solver.set_overlap(mode == "on")
            solver.step(dt, check_state=True)          # settle the mode's launch lists
            barrier()
            t0 = time.perf_counter()
            for _ in range(2):
                solver.step(dt, check_state=True)
            barrier()
            t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=cdev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)      # every rank sees the same number
            probe[mode] = float(t.item()) * 1e3 / 2
        best = min(probe, key=probe.get)
        solver.set_overlap(best == "on")
        solver.step(dt, check_state=True)
        solver.sync()
        overlap_choice = {"mode": best, "selected_by": args.overlap,
                          "probe_ms_per_step": {k: round(v, 3) for k, v in probe.items()}}

    # ---- timed region: exactly K steps, device events, max over ranks -----
    # A pass whose clock samples show a hardware or thermal slowdown, or SM
    # clocks far below their maximum without a reason (a leftover clock lock),
    # is discarded and measured once more; sw_power_cap is kept and noted.
    def timed_pass():
        solver.enable_timing(True)
        solver.timers(reset=True)
        l0 = solver.timers()["launches"]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        if rank == 0:
            sampler.mark()
        e0.record(stream)
        for _ in range(args.steps):
            solver.step(dt, check_state=True)   # the flag read-back step() does by default
        e1.record(stream)
        solver.sync()
        barrier()
        t_ms = e0.elapsed_time(e1)
        c = sampler.snapshot() if rank == 0 else None
        tm = solver.timers(reset=True)
        solver.enable_timing(False)
        return t_ms, c, tm, l0

    def suspicious(c):
        if not c or c.get("sm_mhz") is None:
            return False
        bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(c["reasons"])
        stuck = c["sm_mhz"] < 0.8 * c["sm_max_mhz"] and not c["reasons"]
        return bool(bad) or stuck

    ms, clocks, timers, launches0 = timed_pass()
    redo = 1 if (rank == 0 and suspicious(clocks)) else 0
    if world > 1:
        t = torch.tensor([redo], dtype=torch.int32, device=cdev)
        dist.broadcast(t, 0)
        redo = int(t.item())
    if redo:
        first = clocks
        ms, clocks, timers, launches0 = timed_pass()
        if rank == 0:
            clocks["remeasured_after"] = first
    if rank == 0:
        sampler.stop()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    n_rhs = 5 * args.steps
    value = dof_total * n_rhs / (ms * 1e-3)

    # one more step with the RankEvents timeline on (exchange.hpp:83-89):
    # did the first kernel of the last RHS start before its last trace arrived?
    # (taken with the overlap on, whichever order the timed region ran in)
    if world > 1 and overlap_choice["mode"] != "on":
        solver.set_overlap(True)
        solver.step(dt, check_state=True)
    solver.record_events(True)
    solver.step(dt, check_state=True)
    solver.sync()
    events = solver.rank_events()
    solver.record_events(False)
    if world > 1 and overlap_choice["mode"] != "on":
        solver.set_overlap(False)
        solver.step(dt, check_state=True)
        solver.sync()
    halo_bytes = solver.halo_bytes
    interior_el, local_el = solver.overlap_elements()

    # ---- e2e: host buffers in, host buffers out, copies inside the region --
    e2e = None
    if not args.no_e2e:
        torch_dtype = torch.float64 if rb == 8 else torch.float32
        host_q = torch.empty((n_local, 5, solver.n3), dtype=torch_dtype, pin_memory=True)
        nbytes = host_q.numel() * host_q.element_size()
        L = capi.lib()
        capi.check(L.esdg_b200_solver_get_state(solver.h, capi.REG_Q, host_q.data_ptr()))
        e2e_steps = max(2, min(args.steps, 4))

        def timed(body, n_steps=None):
            n_steps = n_steps or e2e_steps
            barrier()
            t0 = time.perf_counter()
            for _ in range(n_steps):
                body()
            barrier()
            wall = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([wall], dtype=torch.float64, device=cdev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                wall = float(t.item())
            return dof_total * 5 * n_steps / wall

        # (a) the plain calls: upload, step, download, one after the other
        def sequential():
            capi.check(L.esdg_b200_solver_set_state(solver.h, capi.REG_Q, host_q.data_ptr()))
            solver.step(dt, check_state=True)
            capi.check(L.esdg_b200_solver_get_state(solver.h, capi.REG_Q, host_q.data_ptr()))

        # (b) one call per step: the result goes to the host while the next
        # step's input comes in (chunk-pipelined, full duplex), and the runs of
        # the last stage that have finished leave while the rest still computes
        # (esdg_b200_solver_step_swap; every step still moves its input H2D and
        # its result D2H, and reports a non-physical state)
        def duplex():
            capi.check(L.esdg_b200_solver_step_swap(solver.h, dt, host_q.data_ptr(), host_q.data_ptr(), 1),
                       solver.h)

        seq_value = timed(sequential)
        capi.check(L.esdg_b200_solver_set_state(solver.h, capi.REG_Q, host_q.data_ptr()))
        dup_value = timed(duplex)

        # (c) independent states (an ensemble advanced round-robin, each member's
        # state host-resident between its steps): while member i is stepped on
        # the device, member i+1's state is uploaded and member i-1's result is
        # downloaded into its host buffer (esdg_b200_solver_step_stream). Every
        # timed step still moves one state H2D and one result D2H and reports a
        # non-physical state; the pipeline is primed by untimed calls and
        # drained after the region. Three pinned host states per rank; with
        # N ranks every rank streams its own Morton range of each member (the
        # halo exchange of the step keeps its own copy stream) and all ranks
        # decide together whether the host has the memory for it.
        stream_value = None
        stream_note = None
        if not args.no_stream_e2e:
            import psutil
            enough = psutil.virtual_memory().available > world * 3 * nbytes + (16 << 30) * (2 if world > 1 else 1)
            if world > 1:
                t = torch.tensor([1 if enough else 0], dtype=torch.int32, device=cdev)
                dist.all_reduce(t, op=dist.ReduceOp.MIN)
                enough = bool(int(t.item()))
            if enough:
                members = [host_q] + [torch.empty_like(host_q, pin_memory=True) for _ in range(2)]
                for m in members[1:]:
                    m.copy_(host_q)
                capi.check(L.esdg_b200_solver_set_state(solver.h, capi.REG_Q, members[0].data_ptr()))
                call = [0]

                def ensemble():
                    i = call[0]
                    capi.check(L.esdg_b200_solver_step_stream(
                        solver.h, dt, members[(i + 1) % 3].data_ptr(),
                        members[(i + 2) % 3].data_ptr() if i > 0 else None, 1), solver.h)
                    call[0] = i + 1

                for _ in range(3):          # primes the pipeline (untimed)
                    ensemble()
                stream_steps = max(e2e_steps, args.steps)
                stream_value = timed(ensemble, stream_steps)
                capi.check(L.esdg_b200_solver_stream_collect(solver.h, members[(call[0] + 2) % 3].data_ptr()),
                           solver.h)
                if not all(bool(torch.isfinite(m).all()) for m in members):
                    raise RuntimeError("ensemble e2e: a member's state is not finite")
                del members
            else:
                stream_note = "not run: less than three pinned host states of free memory"
        coupled_call = ("esdg_b200_solver_step_swap (one LSRK step; the result goes to the pinned host "
                        "StateField, run by run of the last stage, while the next step's input is "
                        "uploaded from it, chunk-pipelined)")
        e2e = {"value": stream_value if stream_value is not None else dup_value, "unit": UNIT,
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "steps": stream_steps if stream_value is not None else e2e_steps,
               "call": ("esdg_b200_solver_step_stream (one LSRK step per call on a three-member ensemble "
                        "advanced round-robin, every member's state in pinned host memory between its "
                        "steps: each call uploads the next member's state, steps the current one, "
                        "downloads the previous one's result; pipeline primed before and drained "
                        "after the timed region)") if stream_value is not None else coupled_call,
               "coupled_value": dup_value, "coupled_steps": e2e_steps,
               "coupled_call": coupled_call + " -- one state, the next input is this output",
               "sequential_value": seq_value,
               "sequential_call": "esdg_b200_solver_set_state + esdg_b200_solver_step + "
                                  "esdg_b200_solver_get_state on pinned host StateField buffers"}
        if stream_note:
            e2e["stream_note"] = stream_note

    halo_exchanges = None
    if exchange is not None:
        halo_exchanges = exchange.exchanges
        exchange.close()        # before the solver (and its stream) is destroyed
    if rank != 0:
        if world > 1:
            del solver
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel -----------------------------------
    peaks, peak_src = measured_peaks()
    fma_peak = capi.measure_fma_peak(device, rb)
    fma3_peak = capi.measure_fma_peak(device, rb, vector_operands=3)
    # nominal CUDA-core FMA peak: SMs x FP64 (FP32) lanes x 2 x max SM clock
    sm_count = torch.cuda.get_device_properties(device).multi_processor_count
    sm_mhz = (clocks or {}).get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
    peak_nominal = sm_count * (64 if rb == 8 else 128) * 2 * sm_mhz * 1e6 / 1e12
    w = work_model(nq, rb)
    per_launch = {k: timers[k] / n_rhs for k in ("volume", "surface", "update")}
    kernels = {}
    # the three kernels of the split path, timed on their own right after the
    # timed region (two LSRK steps, CUDA events around every launch): the
    # volume kernel against the FMA peak, surface and update against HBM
    if args.path != "split" and world == 1:
        solver.set_path(capi.PATH_SPLIT)
        solver.step(dt, check_state=False)
        solver.sync()
        solver.enable_timing(True)
        solver.timers(reset=True)
        for _ in range(2):
            solver.step(dt, check_state=False)
        solver.sync()
        ts = solver.timers(reset=True)
        solver.enable_timing(False)
        vol_s, surf_s, upd_s = (ts[k] / 10 for k in ("volume", "surface", "update"))
        vol_tf = w["volume_flops"] * n_local / vol_s / 1e12
        kernels["volume"] = {"bound": "fp64" if rb == 8 else "fp32", "achieved": vol_tf,
                             "peak": fma_peak, "unit": "TFLOP/s", "frac": vol_tf / fma_peak,
                             "peak_nominal": peak_nominal, "frac_nominal": vol_tf / peak_nominal,
                             "ms": 1e3 * vol_s, "traffic": ncu_traffic("volume", args.order, args.precision, args.case),
                             "flops_model": f"{w['volume_flops']} flops/element/launch"}
        surf_gbs = w["surface_bytes"] * n_local / surf_s / 1e9
        kernels["surface"] = {"bound": "hbm", "achieved": surf_gbs, "peak": peaks["hbm_gbs"],
                              "unit": "GB/s", "frac": surf_gbs / peaks["hbm_gbs"], "ms": 1e3 * surf_s}
        upd_gbs = w["update_bytes"] * n_local / upd_s / 1e9
        kernels["update"] = {"bound": "hbm", "achieved": upd_gbs, "peak": peaks["hbm_gbs"],
                             "unit": "GB/s", "frac": upd_gbs / peaks["hbm_gbs"], "ms": 1e3 * upd_s}
    upd_flops = 10 * nq ** 3          # q += b k: 2 flops per value
    if args.path == "stage":
        flops = (w["volume_flops"] + w["surface_flops"] + upd_flops) * n_local
        dom = "rhs_kernel<VOL,SURF> + register update (K1+K2+K3, one launch per LSRK stage)"
        dom_s = per_launch["volume"]
        traffic_key = "stage"
    elif args.path == "fused":
        flops = (w["volume_flops"] + w["surface_flops"]) * n_local
        dom = "rhs_kernel<VOL,SURF> (fused K1+K2)"
        dom_s = per_launch["volume"]
        traffic_key = "fused"
    else:
        flops = w["volume_flops"] * n_local
        dom = "rhs_kernel<VOL> (K1 volume)"
        dom_s = per_launch["volume"]
        traffic_key = "volume"
        surf_gbs = w["surface_bytes"] * n_local / per_launch["surface"] / 1e9
        kernels["surface"] = {"bound": "hbm", "achieved": surf_gbs, "peak": peaks["hbm_gbs"],
                              "unit": "GB/s", "frac": surf_gbs / peaks["hbm_gbs"],
                              "ms": 1e3 * per_launch["surface"]}
    achieved = flops / dom_s / 1e12
    # the HBM side of the same kernel: its algorithmic bytes per element
    # over the same launch time
    stage_bytes = {"stage": 21 * nq ** 3 * rb, "fused": 16 * nq ** 3 * rb, "volume": w["volume_bytes"]}[traffic_key]
    hbm_gbs = stage_bytes * n_local / dom_s / 1e9
    if per_launch["update"] > 0 and "update" not in kernels:
        upd_gbs = w["update_bytes"] * n_local / per_launch["update"] / 1e9
        kernels["update"] = {"bound": "hbm", "achieved": upd_gbs, "peak": peaks["hbm_gbs"],
                             "unit": "GB/s", "frac": upd_gbs / peaks["hbm_gbs"],
                             "ms": 1e3 * per_launch["update"]}
    roofline = {
        "kernel": dom, "bound": "fp64" if rb == 8 else "fp32",
        "achieved": achieved, "peak": fma_peak, "unit": "TFLOP/s", "frac": achieved / fma_peak,
        "peak_nominal": peak_nominal, "frac_nominal": achieved / peak_nominal,
        "hbm": {"achieved": hbm_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": hbm_gbs / peaks["hbm_gbs"],
                "bytes_model": f"{stage_bytes} algorithmic bytes/element/launch"},
        "traffic": ncu_traffic(traffic_key, args.order, args.precision, args.case) if world == 1 else None,
        "ms_per_launch": 1e3 * dom_s,
        "flops_model": "reference PerfRecord model (diagnostics.cpp:33-81): "
                       f"{flops // n_local} flops/element/launch",
        "peak_source": ("CUDA-core FMA peak measured in this run by esdg_b200_measure_fma_peak "
                        f"(one vector-register operand per FMA); HBM peak from {peak_src}"),
        "peak_3_vector_operands": fma3_peak,
        "other_kernels": kernels,
    }

    cpu = None
    if not args.no_cpu_baseline and world == 1:     # the CPU leg belongs to the N=1 line only
        try:
            cpu = run_cpu_reference(args.order, args.precision, args.cpu_seconds)
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as exc:  # the baseline must never sink the bench line
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                   "sample": f"unavailable: {exc!r}"}

    if args.case == "bubble":
        config_index = 1 if world == 1 else 4
    else:  # channel: configs[2] fills one GPU, configs[3] is the fixed ~4e8-DOF mesh
        config_index = 3 if (world > 1 or mesh.ne * solver.n3 > 2e8) else 2
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None,
        "dtype": args.precision, "data": "synthetic",
        "config": {
            "workload": (f"{'rising thermal bubble' if args.case == 'bubble' else 'baroclinic channel'}"
                         f", N={args.order}, {mesh.ne} hex elements, {dof_total} DOF, {args.precision}"
                         f" (BASELINE.json configs[{config_index}])"),
            "elements": mesh.ne, "dof": dof_total, "order": args.order,
            "base": list(base), "refinement": args.refinement, "path": args.path,
            "rhs_per_step": 5, "dt": dt, "partition": f"morton x{world}",
            "l2": "inputs_exceed_l2 (state registers are GBs; 126 MB L2)",
        },
        "clocks": clocks, "e2e": e2e, "gpu_launches": timers["launches"] - launches0,
        "roofline": roofline, "cpu_baseline": cpu,
    }
    if world > 1:
        # rank 0's share: trace bytes it sends (= receives) per RHS, the
        # elements whose one-pass kernel runs while the traces travel, and the
        # CUDA-event timeline of one RHS (ns since it was enqueued)
        line["config"]["halo"] = {
            "exchange": ("ncclSend/ncclRecv in one group per RHS, issued by the library (C++)"
                         if args.exchange == "nccl" else "torch.distributed batch_isend_irecv callback"),
            "nccl_version": capi.lib().esdg_b200_solver_nccl_version(solver.h),
            "halo_bytes_per_rhs": halo_bytes,
            "interior_fraction": interior_el / max(local_el, 1),
            "interior_elements": interior_el, "local_elements": local_el,
            "overlap": overlap_choice,
            "events_ns": events,
            "interior_kernel_started_before_last_recv": events["volume_start_ns"] <= events["last_arrival_ns"],
        }
        if halo_exchanges is not None:
            line["config"]["halo"]["exchanges"] = halo_exchanges
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        main_reference(args, rank)
        return
    main_b200(args, rank, local_rank, world)


if __name__ == "__main__":
    main()
