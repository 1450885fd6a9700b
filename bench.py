#!/usr/bin/env python3
"""bench.py — headline benchmark of the B200 QMC sampling path.

Metric (BASELINE.json): Gsamples/s, one sample = one (index, dimension)
component, plus % of the HBM write roofline. The headline workload is
BASELINE.json configs[1]: Sobol' 2^28 points x 32 dimensions, unscrambled,
materialised fp32 row-major ("C2"). One step = one qmc_sobol_fill over the
whole index range (one kernel launch) with the 32 GiB output resident in HBM.
Weak scaling: rank r fills indices [r*2^28, (r+1)*2^28) (no collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--no-extra] [--no-cpu] [--no-e2e]

--gpus N > 1 without torchrun re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one rank per GPU over
NCCL); fewer than N visible GPUs is an error (exit 2), never a silent N=1 run.

--impl reference times the reference's own CPU implementation (the
unmodified qmckit library compiled from its sources into
oracle/_ref/libqmcref.so) on the host cores, rank 0 only.

Every other BASELINE config (C1, C3, C4, C5) and the SPEC acceptance-9
comparison are reported under "configs", each with its own roofline and a
same-run CPU baseline of the reference (1 thread and all cores).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_POINTS = 1 << 28
DIMS = 32
METRIC = "Gsamples/s (index x dim)"
UNIT = "Gsamples/s"
WORKLOAD = "sobol_2^28x32_unscrambled_fp32"
# C5's unit is the pixel-sample; its algorithmic FP64 work in
# the reference formulation (render.cpp:58-79, scene_value :17-26 with the
# sine as Cody-Waite reduction + degree-13/12 polynomials, Neumaier
# quality.hpp:22-30), flops with an FMA counted as 2: sample point 4
# (2 add, 2 mul), 8*pi*x and 8*pi*y 2, two sines 2 x 24 (rint argument 1,
# 3-FMA reduction 6, r^2 1, 7-FMA polynomial 14, final FMA 2), product and
# 0.5*(1+s) 3, disc test and weight 6, Neumaier 4.
C5_FLOPS_PER_PIXEL_SAMPLE = 67
CPU_WINDOWS = 16


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def cpu_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count() or 1, "model": model}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the kernels run."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
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
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sms, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sms)}


# ------------------------------------------------------------ distributed
def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> int:
    """--gpus N > 1 without torchrun: one rank per GPU under
    torch.distributed.run on this node. Fewer than N GPUs is an error."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": "bench.py --gpus %d: only %d CUDA device(s) visible"
                          % (args.gpus, have)}), flush=True)
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node",
           str(args.gpus), "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_init(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (n_gpus, world))
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL communicator init in the log (comm ranks / NVLS / transport)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------ CPU (reference) legs
def windows(total: int, n: int, k: int = CPU_WINDOWS, align: int = 4096):
    """k windows of about n/k indices spread evenly over [0, total) — a
    bounded sample of the whole index range, not its cheap start."""
    per = max(align, (n // k) // align * align)
    step = total // k
    return [(w * step, min(per, total - w * step)) for w in range(k)]


class CpuRef:
    """The CPU implementation timed beside the GPU: the unmodified reference
    build (oracle/_ref, kind "reference") — or, when that build is absent,
    the C restatement (oracle/, kind "port", Sobol' only)."""

    def __init__(self):
        from oracle import load_oracle, load_ref, ref_available

        self.oracle = load_oracle()
        if ref_available():
            self.kind, self.lib = "reference", load_ref()
        else:
            self.kind, self.lib = "port", None

    # --- one timed sample; returns (seconds, units) -----------------------
    def sobol(self, total, n, dims, threads, words=None):
        import numpy as np

        from oracle import ptr

        w = None if words is None else np.ascontiguousarray(words, np.uint32)
        wins = windows(total, n)
        out = np.empty((max(c for _, c in wins), dims), np.float32)
        t0 = time.perf_counter()
        for first, cnt in wins:
            if self.lib is not None:
                rc = self.lib.ref_sobol_fill(first, cnt, dims, None if w is None else ptr(w),
                                             ptr(out), threads)
                if rc != 0:
                    raise RuntimeError(self.lib.ref_last_error().decode())
            else:
                self._port_sobol(first, cnt, dims, w, out, threads)
        return time.perf_counter() - t0, sum(c for _, c in wins) * dims

    def _port_sobol(self, first, cnt, dims, w, out, threads):
        from concurrent.futures import ThreadPoolExecutor

        import numpy as np

        import paper_2307_15584_b200 as q
        from oracle import ptr

        cols = np.ascontiguousarray(q.GeneratorMatrixSet.builtin(dims).columns(), np.uint32)
        cuts = [cnt * t // threads for t in range(threads + 1)]

        def run(t):
            a, b = cuts[t], cuts[t + 1]
            self.oracle.qo_sobol_fill_f32(first + a, b - a, dims, ptr(cols),
                                          None if w is None else ptr(w), out[a:].ctypes.data)

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(run, range(threads)))

    def radical(self, total, n, threads):
        import numpy as np

        from oracle import ptr

        wins = windows(total, n)
        out = np.empty(max(c for _, c in wins), np.float32)
        t0 = time.perf_counter()
        for first, cnt in wins:
            rc = self.lib.ref_radical_fill(first, cnt, 0, ptr(out), threads)
            if rc != 0:
                raise RuntimeError(self.lib.ref_last_error().decode())
        return time.perf_counter() - t0, sum(c for _, c in wins)

    def halton_linear(self, total, n, dims, threads):
        import numpy as np

        from oracle import ptr

        wins = windows(total, n)
        out = np.empty((max(c for _, c in wins), dims), np.float32)
        t0 = time.perf_counter()
        for first, cnt in wins:
            rc = self.lib.ref_halton_linear_fill(first, cnt, dims, ptr(out), threads)
            if rc != 0:
                raise RuntimeError(self.lib.ref_last_error().decode())
        return time.perf_counter() - t0, sum(c for _, c in wins) * dims

    def lattice_cp(self, total, n, g, shifts, threads):
        import numpy as np

        from oracle import ptr

        ga, sa = np.ascontiguousarray(g, np.uint32), np.ascontiguousarray(shifts, np.uint32)
        dims = len(g)
        wins = windows(total, n)
        out = np.empty((max(c for _, c in wins), dims), np.float32)
        t0 = time.perf_counter()
        for first, cnt in wins:
            rc = self.lib.ref_lattice_fill(first, cnt, dims, ptr(ga), ptr(sa), ptr(out), threads)
            if rc != 0:
                raise RuntimeError(self.lib.ref_last_error().decode())
        return time.perf_counter() - t0, sum(c for _, c in wins) * dims

    def owen_port(self, total, n, dims, seeds, threads):
        """Hash-Owen has no reference implementation: the
        oracle's C restatement (qo_sobol_owen_fill_fixed) on `threads`
        Python threads (ctypes releases the GIL)."""
        from concurrent.futures import ThreadPoolExecutor

        import numpy as np

        import paper_2307_15584_b200 as q
        from oracle import ptr

        cols = np.ascontiguousarray(q.GeneratorMatrixSet.builtin(dims).columns(), np.uint32)
        sd = np.ascontiguousarray(seeds, np.uint32)
        wins = windows(total, n)
        out = np.empty((max(c for _, c in wins), dims), np.uint32)
        t0 = time.perf_counter()
        for first, cnt in wins:
            cuts = [cnt * t // threads for t in range(threads + 1)]

            def run(t, first=first, cuts=cuts):
                a, b = cuts[t], cuts[t + 1]
                self.oracle.qo_sobol_owen_fill_fixed(first + a, b - a, dims, ptr(cols), ptr(sd),
                                                     out[a:].ctypes.data)

            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(run, range(threads)))
        return time.perf_counter() - t0, sum(c for _, c in wins) * dims

    def render(self, w, h, spp, kind, accum, workers):
        import numpy as np

        from oracle import ptr

        out = np.empty((h, w), np.float32)
        t0 = time.perf_counter()
        rc = self.lib.ref_render(w, h, spp, kind.encode(), accum.encode(), 0, workers, ptr(out))
        if rc != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return time.perf_counter() - t0, w * h * spp


def calibrated(fn, target_s: float, n0: int = 1 << 14, nmax: int = 1 << 28):
    """Grow n until one sample takes > 0.2 s, then time one sample sized for
    about target_s. fn(n) -> (seconds, units). Returns (seconds, units)."""
    n = n0
    while True:
        dt, _ = fn(n)
        if dt > 0.2 or n >= nmax:
            break
        n <<= 2
    want = int(n * target_s / max(dt, 1e-6))
    return fn(max(n0, min(want, nmax)))


def cpu_leg(fn, target_s, scale_unit=1e9, what="", all_cores=True, one_thread=True,
            nmax=1 << 28, kind="reference"):
    """cpu_baseline dict for fn(n, threads): all host threads and 1 thread."""
    info = cpu_info()
    res = {"unit": UNIT, "kind": kind, "cores": info["nproc"], "cpu_model": info["model"],
           "nproc": info["nproc"]}
    if all_cores:
        sec, units = calibrated(lambda n: fn(n, info["nproc"]), target_s, nmax=nmax)
        res["value"] = units / sec / scale_unit
        res["sample"] = "%s; %d units in %.2f s on %d threads" % (what, units, sec, info["nproc"])
    if one_thread:
        sec, units = calibrated(lambda n: fn(n, 1), target_s, nmax=nmax)
        res["value_1thread"] = units / sec / scale_unit
        res["sample_1thread"] = "%d units in %.2f s on 1 thread" % (units, sec)
    return res


def run_reference(args):
    """The reference arm: qmc::sobol_component (reference build) on all host
    threads, each step one bounded sample of C2 spread over 16 windows of
    the whole [0, 2^28) index range. Rank 0 only."""
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cpu = CpuRef()
    threads = os.cpu_count() or 1
    fn = lambda n: cpu.sobol(N_POINTS, n, DIMS, threads)  # noqa: E731
    # size one step for ~3 s of CPU work
    n = 1 << 14
    while True:
        dt, _ = fn(n)
        if dt > 0.2 or n >= N_POINTS:
            break
        n <<= 2
    n = max(1 << 16, min(int(n * 3.0 / max(dt, 1e-6)), N_POINTS))
    for _ in range(args.warmup):
        fn(n)
    samples = [fn(n) for _ in range(args.steps)]
    sec = statistics.median(s for s, _ in samples)
    units = samples[0][1]
    value = units / sec / 1e9
    sample = ("%d points x %d dims per step in %d windows spread over [0, 2^28) "
              "(qmc::sobol_component, %s build, %d threads)"
              % (units // DIMS, DIMS, CPU_WINDOWS, cpu.kind, threads))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": max(world, args.gpus),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "points": N_POINTS, "dims": DIMS,
                   "sampled": "%d windows spread over the whole index range" % CPU_WINDOWS},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": cpu.kind,
                         "sample": sample, "cpu_model": cpu_info()["model"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm
def time_steps(fn, steps: int, stream, between=None):
    """Per-step CUDA-event durations (ms) on the launching stream; `between`
    (untimed, e.g. an L2 flush) runs before each step."""
    import torch

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for a, b in evs:
        if between is not None:
            between()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def measure_fill(name, fn, samples_per_step, steps, warmup, peak, stream, between=None):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ms = time_steps(fn, steps, stream, between)
    avg = sum(ms) / len(ms)
    gbs = samples_per_step * 4 / (avg * 1e-3) / 1e9
    return {"workload": name, "value": samples_per_step / (avg * 1e-3) / 1e9, "unit": UNIT,
            "ms_per_step": avg, "ms_median": statistics.median(ms),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",
                         "frac": gbs / peak}}


def host_ram() -> str:
    try:
        import psutil

        vm = psutil.virtual_memory()
        return "%.0f GiB total, %.0f GiB available" % (vm.total / 2**30, vm.available / 2**30)
    except Exception:
        return "unknown"


def host_bytes_ok(nbytes: int) -> bool:
    try:
        import psutil

        return psutil.virtual_memory().available > 1.5 * nbytes
    except Exception:
        return False


def run_ours(args):
    import torch

    world, rank, local = dist_init(args.gpus)
    torch.cuda.set_device(local)
    import paper_2307_15584_b200 as q

    q.lib()
    peak, peak_src = peaks()
    stream = torch.cuda.current_stream()
    first = rank * N_POINTS
    out = torch.empty((N_POINTS, DIMS), dtype=torch.float32, device="cuda")
    m = q.GeneratorMatrixSet.builtin(DIMS)

    def step():
        q.sobol_fill(N_POINTS, DIMS, first=first, matrices=m, out=out)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    per = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    t0.record(stream)
    for a, b in per:
        a.record(stream)
        step()
        b.record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    total_ms = max_over_ranks(t0.elapsed_time(t1), world)
    kern_ms = sum(a.elapsed_time(b) for a, b in per) / args.steps
    # keep the GPU busy long enough for the clock sampler
    tend = time.time() + 0.6
    while time.time() < tend:
        step()
        torch.cuda.synchronize()
    clk = clocks.stop()

    # write-only streaming ceiling on the same buffer (diagnostic denominator)
    wp_ms = time_steps(lambda: q.write_probe(out), 5, stream)
    write_probe_gbs = N_POINTS * DIMS * 4 / (sum(wp_ms) / len(wp_ms) * 1e-3) / 1e9

    ms_per_step = total_ms / args.steps
    samples = N_POINTS * DIMS
    value = samples * world / (ms_per_step * 1e-3) / 1e9
    achieved = samples * 4 / (kern_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("c2_sobol_fast", None)
        except Exception:
            traffic = None

    # e2e: the same metric through the C-ABI with a pinned HOST output
    # buffer; every step = device fill + D2H of the step's points (no input).
    del out
    torch.cuda.empty_cache()
    e2e = None
    if not args.no_e2e:
        full = N_POINTS * DIMS * 4
        # every rank of the node pins its own slab
        e2e_pts = N_POINTS if host_bytes_ok(full * world) else (1 << 26)
        host = torch.empty((e2e_pts, DIMS), dtype=torch.float32, pin_memory=True)
        hn = host.numpy()
        q.sobol_fill(e2e_pts, DIMS, first=first, matrices=m, out=hn)
        barrier(world)
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(1, min(args.steps, 3))):
            a = time.perf_counter()
            q.sobol_fill(e2e_pts, DIMS, first=first, matrices=m, out=hn)
            ts.append(time.perf_counter() - a)
        sec = max_over_ranks(sum(ts) / len(ts), world)
        e2e = {"value": e2e_pts * DIMS * world / sec / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": e2e_pts * DIMS * 4,
               "sample": "%d points x %d dims per rank per step into pinned host memory "
                         "(C-ABI qmc_sobol_fill, chunked D2H pipeline)%s"
                         % (e2e_pts, DIMS, "" if e2e_pts == N_POINTS else
                            "; the full 2^28 x 32 (32 GiB pinned) skipped: host RAM %s"
                            % host_ram()),
               "full_config": e2e_pts == N_POINTS}
        del host, hn

    extra = {}
    if not args.no_extra:
        torch.cuda.empty_cache()
        if world > 1:
            extra["c5_render_4k_distributed"] = run_render_distributed(q, world, stream)
        if rank == 0:
            extra.update(run_extra(q, stream, peak, args))

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            ref = CpuRef()
            cpu = cpu_leg(lambda n, t: ref.sobol(N_POINTS, n, DIMS, t), args.cpu_seconds,
                          what="qmc::sobol_component (%s build), C2 sampled in %d windows "
                               "spread over [0, 2^28)" % (ref.kind, CPU_WINDOWS),
                          kind=ref.kind)
        except Exception as e:  # pragma: no cover
            cpu = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "points_per_gpu": N_POINTS, "dims": DIMS,
                       "scramble": "none", "layout": "row-major [n][dims] fp32",
                       "parallelism": "index-range shards, no collective",
                       "l2": "no flush: each step writes 32 GiB >> 126 MB L2"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": "profile-derived: dram__bytes_read.sum + "
                                           "dram__bytes_write.sum per launch from the committed "
                                           "ncu --set full capture (profiles/traffic.json), "
                                           "not measured by this run",
                         "peak_source": peak_src,
                         "write_probe_gbs": write_probe_gbs,
                         "frac_of_write_probe": achieved / write_probe_gbs,
                         "algorithmic_bytes_per_launch": samples * 4},
            "gpu_launches": args.steps,
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "configs": extra,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_render_distributed(q, world, stream):
    """C5 across ranks through the library's own NCCL communicator
    (qmc_render_nccl): row bands + ncclAllGather (bit-identical to the 1-GPU
    image) and the paper's sample partition + int64 ncclAllReduce; device
    time, max over ranks."""
    import torch

    comm = q.Comm.from_torch_group()
    img = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
    res = {"comm": comm.info(), "nccl_version": q.nccl_version()}

    def timed(fn, reps=3):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(b) / reps, world)

    for spp in (16, 64, 256):
        ms = timed(lambda: q.render_nccl(3840, 2160, spp, comm, "rows", out=img))
        res["pixel-shifted-lattice/rows/spp%d" % spp] = {
            "value": 3840 * 2160 * spp / (ms * 1e-3) / 1e9, "unit": "G pixel-samples/s",
            "ms_per_step": ms, "n_gpus": world,
            "collective": "ncclAllGather of fp32 row bands (qmc_render_nccl, in the library)"}
    if world & (world - 1) == 0:
        spp = 256
        ms = timed(lambda: q.render_nccl(3840, 2160, spp, comm, "samples", accum="int", out=img))
        res["pixel-shifted-lattice/int/samples/spp256"] = {
            "value": 3840 * 2160 * spp / (ms * 1e-3) / 1e9, "unit": "G pixel-samples/s",
            "ms_per_step": ms, "n_gpus": world,
            "collective": "ncclAllReduce(sum) of int64 accumulators (qmc_render_nccl)"}
    comm.destroy()
    # §8f rank 1 across ranks: chunk ranges + one all-gather of the Kahan
    # partials, combined by reduce_deterministic (bit-identical to 1 GPU)
    from paper_2307_15584_b200.distributed import integrate_distributed

    ni = 1 << 28
    fn = lambda: integrate_distributed("sobol", "product-sine", ni, 8)  # noqa: E731
    fn()
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    est = fn()
    sec = max_over_ranks(time.perf_counter() - t0, world)
    res["integrate_sobol_product_sine_2^28x8"] = {
        "value": ni * 8 / sec / 1e9, "unit": "Gsamples/s (host-timed, max over ranks)",
        "n_gpus": world, "estimate": est,
        "collective": "all_gather_into_tensor of chunk partials (NCCL) + reduce_deterministic"}
    return res


def run_extra(q, stream, peak, args):
    """Other BASELINE configs and the §8f rows, one entry each (not the
    headline), each with a same-run CPU baseline of the reference. Each
    section is guarded: a failing config records its error instead of
    costing the headline line."""
    import torch

    res = {}
    steps, warm = 5, 3
    cpu_s = args.cpu_config_seconds
    want_cpu = not args.no_cpu
    ref = CpuRef() if want_cpu else None

    def section(fn):
        try:
            fn()
        except Exception as e:  # noqa: BLE001 - reported in the JSON line
            res.setdefault("errors", {})[fn.__name__] = "%s: %s" % (type(e).__name__, e)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    def cpu(name, fn, **kw):
        if not want_cpu or ref is None or ref.lib is None:
            return None
        try:
            return cpu_leg(fn, cpu_s, what=name, **kw)
        except Exception as e:  # noqa: BLE001
            return {"error": "%s: %s" % (type(e).__name__, e)}

    def c1():
        # van der Corput 2^24 x 1 (launch-bound parity config). Timed per
        # launch with an untimed 512 MiB read between launches (L2 flush: the
        # previous output is written back during the flush and the launch
        # finds L2 full of clean lines); the CUDA-graph replay of 12 launches
        # over 4 rotating buffers is reported beside it.
        n1 = 1 << 24
        o1 = [torch.empty(n1, dtype=torch.float32, device="cuda") for _ in range(4)]
        # 1 GiB read: long enough (~170 us) that the host has always queued
        # the timed launch before the flush ends (no host gap in the events)
        flush = torch.ones(1 << 28, dtype=torch.float32, device="cuda")
        r1 = measure_fill("vdc 2^24 x 1, one launch per step, L2 flushed between steps",
                          lambda: q.radical_inverse_fill(n1, 0, out=o1[0]), n1, 20, 5, peak,
                          stream, between=lambda: flush.sum())
        r1["l2"] = "1 GiB read (torch.sum) before every timed launch"
        # the same single-launch conditions for a pure streaming-store kernel
        # on the same 64 MiB: the ceiling of a one-shot 64 MiB write
        wp = measure_fill("write probe 64 MiB, L2 flushed", lambda: q.write_probe(o1[0]), n1, 20,
                          5, peak, stream, between=lambda: flush.sum())
        r1["write_probe_same_conditions"] = {"ms": wp["ms_per_step"],
                                             "frac": wp["roofline"]["frac"]}
        g1 = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        with torch.cuda.graph(g1, stream=cap):
            for k in range(12):
                q.radical_inverse_fill(n1, 0, out=o1[k % 4], stream=cap.cuda_stream)
        rg = measure_fill("vdc graph", g1.replay, n1 * 12, 20, 5, peak, stream)
        r1["graph_of_12_launches"] = {"value": rg["value"], "ms_per_launch": rg["ms_per_step"] / 12,
                                      "frac": rg["roofline"]["frac"],
                                      "l2": "4 rotating 64 MiB outputs, no flush"}
        # the whole C1 range on the CPU (2^24 indices), 1 thread and all cores
        r1["cpu_baseline"] = cpu("qmc::radical_inverse(i, 0), the whole 2^24 range "
                                 "in %d windows" % CPU_WINDOWS,
                                 lambda n, t: ref.radical(n1, n, t), nmax=n1)
        res["c1_vdc_2^24"] = r1

    def halton():
        # the paper's "previous approach": linearly scrambled Halton, 32 dims
        nh = 1 << 24
        oh = torch.empty((nh, 32), dtype=torch.float32, device="cuda")
        rh = measure_fill("halton linear 2^24 x 32",
                          lambda: q.halton_fill(nh, 32, scramble="linear", out=oh), nh * 32, steps,
                          warm, peak, stream)
        rh["roofline"]["bound"] = ("hbm (issue/latency-limited walk: two shared-memory table loads, "
                                   "the carry add and the map per sample; TMA store; k_halton_lv)")
        rh["cpu_baseline"] = cpu("qmc::halton_point(i, 32, default_linear_factors(32)), "
                                 "%d windows over [0, 2^24)" % CPU_WINDOWS,
                                 lambda n, t: ref.halton_linear(nh, n, 32, t), nmax=nh)
        res["halton_linear_2^24x32"] = rh

    def c3():
        # Owen / XOR scrambled Sobol' 2^28 x 64
        n3, d3 = 1 << 28, 64
        seeds = [q.pixel_hash(j, 1, 0x5EED) for j in range(d3)]
        m64 = q.GeneratorMatrixSet.builtin(d3)
        o3 = torch.empty((n3, d3), dtype=torch.float32, device="cuda")
        r_owen = measure_fill(
            "owen sobol 2^28 x 64", lambda: q.sobol_fill(n3, d3, matrices=m64, scramble="owen",
                                                         words=seeds, out=o3), n3 * d3, steps,
            warm, peak, stream)
        r_xor = measure_fill(
            "xor sobol 2^28 x 64", lambda: q.sobol_fill(n3, d3, matrices=m64, scramble="xor",
                                                        words=seeds, out=o3), n3 * d3, steps,
            warm, peak, stream)
        r_xor["cpu_baseline"] = cpu(
            "qmc::sobol_component(i, j, M, pixel_hash(j, 1, 0x5eed)) (XOR scramble, the "
            "reference's digital scramble), %d windows over [0, 2^28)" % CPU_WINDOWS,
            lambda n, t: ref.sobol(n3, n, d3, t, words=seeds), nmax=n3)
        if want_cpu:
            try:
                r_owen["cpu_baseline"] = cpu_leg(
                    lambda n, t: ref.owen_port(n3, n, d3, seeds, t), cpu_s, kind="port",
                    what="hash-Owen has no reference implementation (SPEC.md:271): the oracle's "
                         "C restatement qo_sobol_owen_fill_fixed (integer stage), %d windows"
                         % CPU_WINDOWS, one_thread=False)
            except Exception as e:  # noqa: BLE001
                r_owen["cpu_baseline"] = {"error": str(e)}
        res["c3_owen_2^28x64"] = r_owen
        res["c3_xor_2^28x64"] = r_xor

    def c4():
        # lattice 2^30 x 16 + integer CP rotation
        n4, d4 = 1 << 30, 16
        g = q.lfsr_generator_vector(0xACE1, d4)
        s = [q.pixel_hash(j, 1, 0x5EED) for j in range(d4)]
        o4 = torch.empty((n4, d4), dtype=torch.float32, device="cuda")
        r4 = measure_fill("lattice+cp 2^30 x 16", lambda: q.lattice_fill(n4, g, shifts=s, out=o4),
                          n4 * d4, steps, warm, peak, stream)
        r4["cpu_baseline"] = cpu(
            "map_u32_to_unifloat(lattice_component_fixed(i, g_j) + s_j), %d windows over "
            "[0, 2^30)" % CPU_WINDOWS, lambda n, t: ref.lattice_cp(n4, n, g, s, t), nmax=n4)
        res["c4_lattice_cp_2^30x16"] = r4

    def c5():
        # fused per-pixel render 3840x2160, Kahan; pixel-shifted lattice at
        # every spp, the other kinds at 64 spp
        img = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
        c5r = {}
        xt = q.XorTables.white_noise(2, 1 << 12, 7)
        fp64 = q.fp64_probe(4096) / 1e12
        for spp in (1, 16, 64, 256):
            kinds = ("pixel-shifted-lattice",) if spp != 64 else (
                "pixel-shifted-lattice", "image-plane-halton", "halton-hilbert",
                "pixel-random-lattice", "sobol", "sobol-xor-table")
            for kind in kinds:
                kw = {"tables": xt} if kind == "sobol-xor-table" else {}
                fn = lambda: q.render(3840, 2160, spp, kind=kind, out=img, **kw)  # noqa: E731
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                ms = time_steps(fn, 3, stream)
                avg = sum(ms) / len(ms)
                rate = 3840 * 2160 * spp / (avg * 1e-3)
                ach = rate * C5_FLOPS_PER_PIXEL_SAMPLE / 1e12
                c5r["%s/spp%d" % (kind, spp)] = {
                    "value": rate / 1e9, "unit": "G pixel-samples/s", "ms_per_step": avg,
                    "roofline": {"bound": "fp64", "achieved": ach, "peak": fp64,
                                 "unit": "TFLOP/s", "frac": ach / fp64, "traffic": None,
                                 "algorithmic_flops_per_pixel_sample": C5_FLOPS_PER_PIXEL_SAMPLE,
                                 "peak_source": "measured in this run: qmc_fp64_probe (dense "
                                                "DFMA chains, one wave of CTAs)"}}
        # the paper's comparison at the render level
        c5r["ratio_psl_over_image_plane_halton_spp64"] = {
            "value": c5r["pixel-shifted-lattice/spp64"]["value"] /
            c5r["image-plane-halton/spp64"]["value"], "unit": "x"}
        # e2e: qmc_render into pinned HOST memory (device render + D2H of the
        # 33 MB image inside the timed region)
        host = torch.empty((2160, 3840), dtype=torch.float32, pin_memory=True).numpy()
        for spp in (16, 64):
            q.render(3840, 2160, spp, out=host)
            ts = []
            for _ in range(3):
                a = time.perf_counter()
                q.render(3840, 2160, spp, out=host)
                ts.append(time.perf_counter() - a)
            sec = sum(ts) / len(ts)
            c5r["pixel-shifted-lattice/spp%d" % spp]["e2e"] = {
                "value": 3840 * 2160 * spp / sec / 1e9, "unit": "G pixel-samples/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 3840 * 2160 * 4,
                "sample": "C-ABI qmc_render into a pinned host image, host-timed"}
        if want_cpu and ref is not None and ref.lib is not None:
            info = cpu_info()
            for spp in (16, 64):
                key = "pixel-shifted-lattice/spp%d" % spp
                try:
                    sec, units = ref.render(3840, 2160, spp, "pixel-shifted-lattice", "kahan",
                                            info["nproc"])
                    cb = {"value": units / sec / 1e9, "unit": "G pixel-samples/s",
                          "cores": info["nproc"], "nproc": info["nproc"],
                          "cpu_model": info["model"], "kind": ref.kind,
                          "sample": "qmc::render(job) 3840x2160 at %d spp, workers = %d, "
                                    "%.2f s" % (spp, info["nproc"], sec)}
                    if spp == 16:
                        sec1, _ = ref.render(3840, 2160, spp, "pixel-shifted-lattice", "kahan", 1)
                        cb["value_1thread"] = units / sec1 / 1e9
                        cb["sample_1thread"] = "workers = 1, %.2f s" % sec1
                    c5r[key]["cpu_baseline"] = cb
                except Exception as e:  # noqa: BLE001
                    c5r[key]["cpu_baseline"] = {"error": str(e)}
            try:
                sec, units = ref.render(3840, 2160, 64, "image-plane-halton", "kahan",
                                        info["nproc"])
                c5r["image-plane-halton/spp64"]["cpu_baseline"] = {
                    "value": units / sec / 1e9, "unit": "G pixel-samples/s",
                    "cores": info["nproc"], "kind": ref.kind,
                    "sample": "qmc::render(job) image-plane-halton 4K 64 spp, %.2f s" % sec}
            except Exception as e:  # noqa: BLE001
                c5r["image-plane-halton/spp64"]["cpu_baseline"] = {"error": str(e)}
        res["c5_render_4k"] = c5r

    def acceptance9():
        # SPEC acceptance 9 on its own basis:
        # `qmckit bench` = run_bench_kernel (bench.cpp:79-150), component
        # generation of pixel-shifted-lattice vs halton-tabled (linearly
        # scrambled 32-dim Halton), 32 dims — here the same walk and checksum
        # on the device, and the reference's own CPU run beside it.
        a9 = {}
        # not a multiple of the walk's period (128 x 128 pixels x 16 indices x
        # 32 dims = 2^23 components, whose folds cancel in pairs); the ABI
        # runs a count/8 warm-up walk first, like bench.cpp:53
        count = 1000000000
        for k in ("pixel-shifted-lattice", "halton-tabled", "halton", "sobol", "lattice",
                  "pixel-random-lattice"):
            r = q.run_bench_kernel(k, count, 32)
            a9["gpu/" + k] = {"value": r["components_per_second"] / 1e9,
                              "unit": "G components/s", "evaluations": count,
                              "checksum": "%016x" % r["checksum"]}
        a9["ratio_psl_over_halton_tabled_gpu"] = {
            "value": a9["gpu/pixel-shifted-lattice"]["value"] / a9["gpu/halton-tabled"]["value"],
            "unit": "x", "bar": ">= 2.0 (SPEC.md:626)"}
        # materialised 32-dim fills: one pixel's pixel-shifted-lattice stream
        # (imageplane.hpp:26-31) vs the linear Halton fill, 2^24 x 32 each
        n, d = 1 << 24, 32
        g32 = q.lfsr_generator_vector(0xACE1, d)
        o = torch.empty((n, d), dtype=torch.float32, device="cuda")
        rp = measure_fill("pixel-shifted-lattice stream 2^24 x 32", lambda: q.stream_fill(
            "pixel-shifted-lattice", n, d, generator=g32, pixel=(1234, 567), order=12, out=o),
            n * d, steps, warm, peak, stream)
        rh = measure_fill("halton linear 2^24 x 32", lambda: q.halton_fill(
            n, d, scramble="linear", out=o), n * d, steps, warm, peak, stream)
        a9["fill/pixel-shifted-lattice_2^24x32"] = rp
        a9["fill/halton-linear_2^24x32"] = rh
        res["ratio_psl_over_halton_linear_components"] = {
            "value": rp["value"] / rh["value"], "unit": "x",
            "basis": "materialised 2^24 x 32 fp32 fills on the device (Gsamples/s ratio)"}
        if want_cpu and ref is not None and ref.lib is not None:
            import ctypes as C

            cps = {}
            for k in ("pixel-shifted-lattice", "halton-tabled"):
                v, ck = C.c_double(), C.c_uint64()
                if ref.lib.ref_run_bench_kernel(k.encode(), 8000000, 32, C.byref(v),
                                                C.byref(ck)) == 0:
                    cps[k] = v.value
            if len(cps) == 2:
                a9["reference_cpu"] = {
                    "pixel-shifted-lattice": cps["pixel-shifted-lattice"] / 1e9,
                    "halton-tabled": cps["halton-tabled"] / 1e9, "unit": "G components/s",
                    "ratio": cps["pixel-shifted-lattice"] / cps["halton-tabled"],
                    "sample": "qmc::run_bench_kernel, 8e6 evaluations x 32 dims "
                              "(`qmckit bench` defaults), 1 thread"}
        res["acceptance9_component_generation"] = a9

    def integrate():
        # §8f rank 1: fused QMC integration (quality.cpp:214-282), Sobol' 8 dims
        ni = 1 << 26
        fn = lambda: q.integrate("sobol", "product-sine", ni, 8, "kahan")  # noqa: E731
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        row = fn()
        b.record(stream)
        sec = time.perf_counter() - t0
        torch.cuda.synchronize()
        dev_s = a.elapsed_time(b) * 1e-3
        res["integrate_sobol_product_sine_2^26x8"] = {
            "value": ni * 8 / sec / 1e9, "unit": "Gsamples/s (host-timed call incl. D2H combine)",
            "device_value": ni * 8 / dev_s / 1e9,
            "device_unit": "Gsamples/s (CUDA events around the call: the chunk kernel and the "
                           "partials' D2H; the host's chunk-order combine excluded)",
            "estimate": row["estimate"], "abs_error": row["abs_error"]}

    def l2_star():
        # §8f rank 4: Warnock L2-star discrepancy, O(N^2 s) pair terms
        nl, dl = 1 << 14, 4
        pts = q.sobol_fill(nl, dl)
        q.l2_star_discrepancy(pts)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q.l2_star_discrepancy(pts)
        sec = time.perf_counter() - t0
        res["l2_star_2^14x4"] = {"value": nl * (nl - 1) / 2 / sec / 1e9,
                                 "unit": "G pair terms/s (host-timed call)", "ms": sec * 1e3}

    for fn in (c1, halton, c3, c4, c5, acceptance9, integrate, l2_star):
        section(fn)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=5.0)
    ap.add_argument("--cpu-config-seconds", type=float, default=1.5)
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
