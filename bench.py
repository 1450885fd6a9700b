#!/usr/bin/env python3
"""bench.py — headline benchmark of the B200 QMC sampling path.

Metric (BASELINE.json): Gsamples/s, one sample = one (index, dimension)
component, plus % of the HBM write roofline. The headline workload is
BASELINE.json configs[1]: Sobol' 2^28 points x 32 dimensions, unscrambled,
materialised fp32 row-major ("C2"). One step = one qmc_sobol_fill over the
whole index range (one kernel launch) with the 32 GiB output resident in HBM.
Weak scaling under torchrun: rank r fills indices [r*2^28, (r+1)*2^28).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--no-extra] [--no-cpu]

--impl reference times the reference's own CPU implementation (the
unmodified qmckit library compiled from its sources into
oracle/_ref/libqmcref.so) on the host cores, rank 0 only.
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

N_POINTS = 1 << 28
DIMS = 32
METRIC = "Gsamples/s (index x dim)"
UNIT = "Gsamples/s"
WORKLOAD = "sobol_2^28x32_unscrambled_fp32"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


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
def dist_init(n_gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch

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


# --------------------------------------------------------- reference arm
class CpuSobol:
    """The CPU implementation timed beside the GPU (cpu_baseline and --impl
    reference): the unmodified reference build (oracle/_ref, kind
    "reference") on all host threads, or — if that build is absent — the C
    restatement (oracle/, kind "port") on as many Python threads (ctypes
    releases the GIL)."""

    def __init__(self):
        from oracle import load_oracle, load_ref, ref_available

        if ref_available():
            self.kind, self.lib = "reference", load_ref()
            self.what = "qmc::sobol_component, reference build"
        else:
            import numpy as np

            import paper_2307_15584_b200 as q

            self.kind, self.lib = "port", load_oracle()
            self.cols = np.ascontiguousarray(q.GeneratorMatrixSet.builtin(DIMS).columns(),
                                             dtype=np.uint32)
            self.what = "oracle qo_sobol_fill_f32 (C restatement)"

    def sample(self, n_pts: int, threads: int, first: int = 0) -> float:
        """Seconds for n_pts x 32 dims of float Sobol' points on the CPU."""
        import numpy as np

        from oracle import ptr

        out = np.empty((n_pts, DIMS), np.float32)
        t0 = time.perf_counter()
        if self.kind == "reference":
            rc = self.lib.ref_sobol_fill(first, n_pts, DIMS, None, ptr(out), threads)
            if rc != 0:
                raise RuntimeError(self.lib.ref_last_error().decode())
        else:
            from concurrent.futures import ThreadPoolExecutor

            cuts = [n_pts * t // threads for t in range(threads + 1)]

            def run(t):
                a, b = cuts[t], cuts[t + 1]
                self.lib.qo_sobol_fill_f32(first + a, b - a, DIMS, ptr(self.cols), None,
                                           out[a:].ctypes.data)

            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(run, range(threads)))
        return time.perf_counter() - t0


def calibrate_cpu(cpu: "CpuSobol", threads: int, target_s: float) -> int:
    n = 1 << 16
    while True:
        dt = cpu.sample(n, threads)
        if dt > 0.25 or n >= (1 << 26):
            break
        n <<= 2
    want = int(n * target_s / max(dt, 1e-6))
    return max(1 << 16, min(want, 1 << 26)) & ~4095


def run_reference(args):
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return 0
    cpu = CpuSobol()
    threads = os.cpu_count() or 1
    n_pts = calibrate_cpu(cpu, threads, 3.0)
    for _ in range(args.warmup):
        cpu.sample(n_pts, threads)
    times = [cpu.sample(n_pts, threads) for _ in range(args.steps)]
    sec = statistics.median(times)
    value = n_pts * DIMS / sec / 1e9
    sample = "%d points x %d dims per step (%s, %d threads)" % (n_pts, DIMS, cpu.what, threads)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": WORKLOAD, "points": N_POINTS, "dims": DIMS, "sampled": True},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": cpu.kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- our arm
def time_steps(fn, steps: int, stream):
    """Per-step CUDA-event durations (ms) on the launching stream."""
    import torch

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for a, b in evs:
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def measure_fill(name, fn, samples_per_step, steps, warmup, peak, stream):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ms = time_steps(fn, steps, stream)
    avg = sum(ms) / len(ms)
    gbs = samples_per_step * 4 / (avg * 1e-3) / 1e9
    return {"workload": name, "value": samples_per_step / (avg * 1e-3) / 1e9, "unit": UNIT,
            "ms_per_step": avg, "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak,
                                             "unit": "GB/s", "frac": gbs / peak}}


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

    # e2e: same metric through the C-ABI with a pinned HOST output buffer;
    # every step = device fill + D2H of the step's points.
    e2e = None
    if not args.no_e2e:
        # the job's host image stays ~8.6 GB however many ranks share it
        # (each rank pins only its slab)
        e2e_pts = max(1 << 20, min(N_POINTS, args.e2e_points) // world)
        host = torch.empty((e2e_pts, DIMS), dtype=torch.float32, pin_memory=True)
        hn = host.numpy()
        for _ in range(2):
            q.sobol_fill(e2e_pts, DIMS, first=first, matrices=m, out=hn)
        barrier(world)
        torch.cuda.synchronize()
        ts = []
        for _ in range(max(1, min(args.steps, 5))):
            a = time.perf_counter()
            q.sobol_fill(e2e_pts, DIMS, first=first, matrices=m, out=hn)
            ts.append(time.perf_counter() - a)
        sec = max_over_ranks(sum(ts) / len(ts), world)
        e2e = {"value": e2e_pts * DIMS * world / sec / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": e2e_pts * DIMS * 4,
               "sample": "%d points x %d dims per step into pinned host memory" % (e2e_pts, DIMS)}
        del host, hn

    extra = {}
    if not args.no_extra:
        del out
        torch.cuda.empty_cache()
        if world > 1:
            extra["c5_render_4k_distributed"] = run_render_distributed(q, world, stream)
        if rank == 0:
            extra.update(run_extra(q, stream, peak, args))

    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            impl = CpuSobol()
            threads = os.cpu_count() or 1
            n_pts = calibrate_cpu(impl, threads, args.cpu_seconds)
            sec = impl.sample(n_pts, threads)
            cpu = {"value": n_pts * DIMS / sec / 1e9, "unit": UNIT, "cores": threads,
                   "kind": impl.kind,
                   "sample": "%d points x %d dims (%s, %.1f s)" % (n_pts, DIMS, impl.what, sec)}
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
    """C5 across ranks: row bands + one NCCL all-gather (bit-identical to the
    1-GPU image); device time, max over ranks."""
    import torch

    from paper_2307_15584_b200.distributed import render_distributed

    res = {}
    for spp in (16, 256):
        fn = lambda: render_distributed(3840, 2160, spp)  # noqa: E731
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(3):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(a.elapsed_time(b) / 3, world)
        res["pixel-shifted-lattice/spp%d" % spp] = {
            "value": 3840 * 2160 * spp / (ms * 1e-3) / 1e9, "unit": "G pixel-samples/s",
            "ms_per_step": ms, "n_gpus": world, "collective": "all_gather_into_tensor (NCCL)"}
    if world & (world - 1) == 0:  # the paper's sample partition (int accumulator)
        from paper_2307_15584_b200.distributed import render_distributed_samples

        spp = 256
        fn = lambda: render_distributed_samples(3840, 2160, spp)  # noqa: E731
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        barrier(world)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(3):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        ms = max_over_ranks(a.elapsed_time(b) / 3, world)
        res["pixel-shifted-lattice/int/sample-partition/spp256"] = {
            "value": 3840 * 2160 * spp / (ms * 1e-3) / 1e9, "unit": "G pixel-samples/s",
            "ms_per_step": ms, "n_gpus": world,
            "collective": "all_reduce(sum) of int64 accumulators (NCCL)"}
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
    headline). Each section is guarded: a failing config records its error
    instead of costing the headline line."""
    import torch

    res = {}
    steps, warm = 5, 3

    def section(fn):
        try:
            fn()
        except Exception as e:  # noqa: BLE001 - reported in the JSON line
            res.setdefault("errors", {})[fn.__name__] = "%s: %s" % (type(e).__name__, e)
        torch.cuda.synchronize()
        torch.cuda.empty_cache()

    def c1():
        # van der Corput 2^24 x 1 (launch-bound parity config): captured once
        # in a CUDA graph and replayed, so the device time is not hidden
        # behind per-call host latency; 4 rotating 64 MiB outputs (256 MiB >
        # 126 MB L2), so consecutive launches write different buffers
        n1 = 1 << 24
        o1 = [torch.empty(n1, dtype=torch.float32, device="cuda") for _ in range(4)]
        q.radical_inverse_fill(n1, 0, out=o1[0])
        torch.cuda.synchronize()
        g1 = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        with torch.cuda.graph(g1, stream=cap):
            for k in range(12):
                q.radical_inverse_fill(n1, 0, out=o1[k % 4], stream=cap.cuda_stream)
        r1 = measure_fill("vdc 2^24 x 1 (CUDA graph of 12 launches over 4 rotating buffers)",
                          g1.replay, n1 * 12, 20, 5, peak, stream)
        r1["ms_per_step"] /= 12
        r1["l2"] = "4 rotating 64 MiB outputs (256 MiB > L2)"
        res["c1_vdc_2^24"] = r1

    def halton():
        # the paper's "previous approach": linearly scrambled Halton, 32 dims
        # (incremental hi/lo split: a table load, an integer magic division
        # and the map per sample; issue-bound, not HBM-bound)
        nh = 1 << 24
        oh = torch.empty((nh, 32), dtype=torch.float32, device="cuda")
        rh = measure_fill("halton linear 2^24 x 32",
                          lambda: q.halton_fill(nh, 32, scramble="linear", out=oh), nh * 32, steps,
                          warm, peak, stream)
        rh["roofline"]["bound"] = "issue (quotient-table load + 3 integer ops + map per sample; TMA store)"
        res["halton_linear_2^24x32"] = rh

    def c3():
        # Owen / XOR scrambled Sobol' 2^28 x 64
        n3, d3 = 1 << 28, 64
        seeds = [q.pixel_hash(j, 1, 0x5EED) for j in range(d3)]
        m64 = q.GeneratorMatrixSet.builtin(d3)
        o3 = torch.empty((n3, d3), dtype=torch.float32, device="cuda")
        res["c3_owen_2^28x64"] = measure_fill(
            "owen sobol 2^28 x 64", lambda: q.sobol_fill(n3, d3, matrices=m64, scramble="owen",
                                                         words=seeds, out=o3), n3 * d3, steps,
            warm, peak, stream)
        res["c3_xor_2^28x64"] = measure_fill(
            "xor sobol 2^28 x 64", lambda: q.sobol_fill(n3, d3, matrices=m64, scramble="xor",
                                                        words=seeds, out=o3), n3 * d3, steps,
            warm, peak, stream)

    def c4():
        # lattice 2^30 x 16 + integer CP rotation
        n4, d4 = 1 << 30, 16
        g = q.lfsr_generator_vector(0xACE1, d4)
        s = [q.pixel_hash(j, 1, 0x5EED) for j in range(d4)]
        o4 = torch.empty((n4, d4), dtype=torch.float32, device="cuda")
        res["c4_lattice_cp_2^30x16"] = measure_fill(
            "lattice+cp 2^30 x 16", lambda: q.lattice_fill(n4, g, shifts=s, out=o4), n4 * d4,
            steps, warm, peak, stream)

    def c5():
        # fused per-pixel render 3840x2160, Kahan; pixel-shifted lattice at
        # every spp, the other kinds (incl. the XOR-table sampler, §8f rank 2)
        # at 64 spp
        img = torch.empty((2160, 3840), dtype=torch.float32, device="cuda")
        c5r = {}
        xt = q.XorTables.white_noise(2, 1 << 12, 7)
        for spp in (1, 16, 64, 256):
            kinds = ("pixel-shifted-lattice",) if spp != 64 else (
                "pixel-shifted-lattice", "image-plane-halton", "pixel-random-lattice", "sobol",
                "sobol-xor-table")
            for kind in kinds:
                kw = {"tables": xt} if kind == "sobol-xor-table" else {}
                fn = lambda: q.render(3840, 2160, spp, kind=kind, out=img, **kw)  # noqa: E731
                for _ in range(2):
                    fn()
                torch.cuda.synchronize()
                ms = time_steps(fn, 3, stream)
                avg = sum(ms) / len(ms)
                c5r["%s/spp%d" % (kind, spp)] = {
                    "value": 3840 * 2160 * spp / (avg * 1e-3) / 1e9,
                    "unit": "G pixel-samples/s", "ms_per_step": avg}
        # the paper's comparison: pixel-shifted
        # lattice vs the image-plane Halton enumeration, same render
        c5r["ratio_psl_over_image_plane_halton_spp64"] = {
            "value": c5r["pixel-shifted-lattice/spp64"]["value"] /
            c5r["image-plane-halton/spp64"]["value"], "unit": "x"}
        res["c5_render_4k"] = c5r

    def integrate():
        # §8f rank 1: fused QMC integration (quality.cpp:214-282), Sobol' 8 dims
        ni = 1 << 26
        fn = lambda: q.integrate("sobol", "product-sine", ni, 8, "kahan")  # noqa: E731
        fn()
        t0 = time.perf_counter()
        row = fn()
        sec = time.perf_counter() - t0
        res["integrate_sobol_product_sine_2^26x8"] = {
            "value": ni * 8 / sec / 1e9, "unit": "Gsamples/s (host-timed call incl. D2H combine)",
            "estimate": row["estimate"], "abs_error": row["abs_error"]}

    def l2_star():
        # §8f rank 4: Warnock L2-star discrepancy, O(N^2 s) pair terms
        # (quality.cpp:76-114)
        nl, dl = 1 << 14, 4
        pts = q.sobol_fill(nl, dl)
        q.l2_star_discrepancy(pts)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q.l2_star_discrepancy(pts)
        sec = time.perf_counter() - t0
        res["l2_star_2^14x4"] = {"value": nl * (nl - 1) / 2 / sec / 1e9,
                                 "unit": "G pair terms/s (host-timed call)", "ms": sec * 1e3}

    for fn in (c1, halton, c3, c4, c5, integrate, l2_star):
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
    ap.add_argument("--e2e-points", type=int, default=1 << 26)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
