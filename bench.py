"""Benchmark of the direct-method bispectrum hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

Workload: BASELINE.json's metric config (cfg2: bispectrum, n = 2^20 float32
bilinear series, M = 1024, K = 1024, Hann, L = 4 -> w = 9), seeded synthetic
input (paper_1805_11775_b200.signals).  One step = segment + demean + taper
-> cuFFT -> triple products over the dilated principal domain -> fp64 scans
-> box sums, input resident in HBM.  Metric units: K * |D_h| segment.bin
triple products.

Timing: W untimed warm-up steps, then exactly K steps, each bracketed by CUDA
events on the launching stream with a 256 MiB L2-flush write between steps
(outside the events); barrier + synchronize around the region; max over
ranks.  N > 1 (torchrun): segments sharded across ranks, NCCL reduce-scatter
of the partial raw sums + halo + gather (distributed_estimate), strong
scaling of one series.

--impl reference: the reference's CPU algorithm (the oracle port of the
EFFICIENT plan, bit-exact with hospectra; the Python reference cannot travel
to the GPU box) on all host cores, on a bounded sample of the same workload.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "segment·bin triple-products/sec (bispectrum n=2^20, M=1024) + % roofline"
UNIT = "units/s"
STAGE_REPS = 50
FLOPS_PER_UNIT = 14  # 6 (a*b) + 6 (*conj c) + 2 (accumulate)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-segments", type=int, default=0, help="segments in the CPU sample (0 = auto)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def _one(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10)
            for line in out.stdout.strip().splitlines():
                self.rows.append([v.strip() for v in line.split(",")])
        except Exception:
            pass

    def start(self):
        self._one()
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        self._one()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
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
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm (oracle port) on all host cores


def cpu_baseline(cfg_name: str, steps: int, warmup: int, segments: int = 0, budget_s: float = 0.0):
    from oracle import hos_oracle as O
    from paper_1805_11775_b200 import signals

    c = signals.baseline_config(cfg_name)
    x = signals.baseline_series(c)
    if x.ndim == 2:
        x = x[0]
    cores = os.cpu_count() or 1
    if segments <= 0:
        segments = min(c.k, max(64, 8 * cores))
    spec = O.segment_spectra(x, c.m, segments, c.taper)
    dom = O.principal_domain(c.order, c.m)
    import multiprocessing as mp
    from concurrent.futures import ProcessPoolExecutor

    bounds = O._row_block_bounds(dom, cores)
    parts = [dom[bounds[i]: bounds[i + 1]] for i in range(cores) if bounds[i + 1] > bounds[i]]
    pool = ProcessPoolExecutor(max_workers=len(parts), mp_context=mp.get_context("spawn"))
    try:
        jobs = lambda: list(pool.map(O._worker, [(spec, c.order, c.m3, True, p) for p in parts]))
        for _ in range(max(1, warmup)):
            jobs()
        times = []
        for i in range(max(1, steps)):
            t0 = time.perf_counter()
            jobs()
            times.append(time.perf_counter() - t0)
            if budget_s and sum(times) + times[0] > budget_s:  # keep the whole run within minutes
                break
    finally:
        pool.shutdown()
    units = segments * _dh_cells(c)
    t = statistics.median(times)
    return {"value": units / t, "unit": UNIT, "cores": len(parts), "kind": "port",
            "sample": f"{cfg_name}: first {segments} of {c.k} segments, full principal domain "
                      f"({len(dom)} points), EFFICIENT-plan port (oracle/hos_oracle.py, bit-exact with "
                      f"hospectra), {len(parts)} processes over row blocks, median of {len(times)}",
            "seconds_per_step": t, "units_per_step": units, "steps_timed": len(times)}


def _dh_cells(c) -> int:
    """|D_h| of a config (logical cells of the dilated principal domain),
    the same count hos_plan_cells reports."""
    h = c.m3 // 2
    lo, hi = -h, c.m3 - 1 - h
    m = c.m
    rows = (m - 1) // 2 + 1
    stop = [min(k1, (m - 2 * k1 - 1) // 2) + 1 for k1 in range(rows)]
    if c.order == 3:
        total = 0
        for a in range(lo, rows - 1 + hi + 1):
            ks = range(max(0, a - hi), min(rows - 1, a - lo) + 1)
            total += max(stop[k] - 1 for k in ks) + hi - lo + 1
        return total
    raise NotImplementedError("order-4 cell count comes from the plan")


# ---------------------------------------------------------------------------
# our arm


def peak_fp32(lib, stream):
    import ctypes

    tf, mhz = ctypes.c_double(), ctypes.c_double()
    rc = lib.hos_peak_fp32(ctypes.byref(tf), ctypes.byref(mhz), stream)
    if rc:
        raise RuntimeError(lib.hos_last_error())
    return tf.value, mhz.value


def load_traffic(cfg_name):
    p = os.path.join(ROOT, "profiles", "ncu_triple_latest.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            if d.get("config") == cfg_name:
                return d.get("dram_bytes_per_launch")
        except Exception:
            return None
    return None


def run_ours(args):
    import torch

    import __graft_entry__

    __graft_entry__.build()
    import ctypes

    import paper_1805_11775_b200 as P
    from paper_1805_11775_b200 import _native

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    force_dist = os.environ.get("HOS_BENCH_FORCE_DIST") == "1"  # test hook: the multi-GPU code path on 1 rank
    if world > 1 or force_dist:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    c = P.baseline_config(args.config)
    prec = 32 if args.precision == "fp32" else 64
    x_host = P.baseline_series(c)
    batch = c.batch
    cfg = P.EstimationConfig(c.order, P.SegmentConfig(m=c.m, k=c.k), c.m3, precision=args.precision, taper=c.taper)
    plan = _native.get_plan(c.order, c.m, c.k, c.m3, True, prec, c.taper, batch, local)
    units = plan.units * batch
    stream = torch.cuda.current_stream(dev)
    cstream = ctypes.c_void_p(stream.cuda_stream)
    lib = _native.lib()

    x = torch.from_numpy(x_host).to(dev)
    out = plan.empty_out()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    native = False
    multi = world > 1 or force_dist
    if not multi:
        step = lambda: plan.estimate(x, out)
    else:
        # the library's own NCCL path (collectives issued inside the C-ABI);
        # the torch.distributed restatement if it cannot be set up
        try:
            from paper_1805_11775_b200.parallel import native_distributed_plan

            dplan = native_distributed_plan(cfg)
            dout = dplan.empty_out()
            dplan.estimate_distributed(x, dout)
            torch.cuda.synchronize()
            step = lambda: dplan.estimate_distributed(x, dout)
            native = True
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] native NCCL path unavailable ({exc}); torch.distributed path", file=sys.stderr)
            step = lambda: P.distributed_estimate(x, cfg, gather=True)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev[i][0].record(stream)
        step()  # the whole pipeline replays as one CUDA graph
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    sampler.stop()
    # per-stage device times on the launching stream: each stage's R launches
    # replayed as one CUDA graph between two CUDA events (mean per launch; the inputs
    # of every stage are the ones the last estimate left in HBM / L2, as in
    # the pipeline, where each stage reads what the previous one just wrote)
    tri, stages = [], {}
    if world == 1:
        for _ in range(3):
            st = plan.time_stages(x, reps=STAGE_REPS, out=out)
            tri.append(st["triple"])
            for k_, v_ in st.items():
                stages.setdefault(k_, []).append(v_)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = units / (ms_per_step * 1e-3)

    # ---- e2e: host buffers through the C-ABI (hos_estimate_host), wall clock
    e2e_ms = []
    if not multi:
        xp = torch.from_numpy(x_host).pin_memory()
        cd = torch.complex64 if prec == 32 else torch.complex128
        op = torch.empty(out.shape, dtype=cd).pin_memory()
        xn, on = xp.numpy(), op.numpy()
        for _ in range(3):
            plan.estimate_host(xn, on)
        # host buffers: every step copies the series in and the values out, so the
        # device-side L2 state does not matter; no flush (it would only cold-start
        # the GPU TLBs the copy engine uses)
        for i in range(max(5, min(args.steps, 50))):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            plan.estimate_host(xn, on)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d = xn.nbytes
        d2h = on.nbytes
    else:
        shard = (c.k + world - 1) // world * c.m
        xp = torch.from_numpy(x_host).pin_memory()
        for i in range(max(5, min(args.steps, 50))):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            xd = xp.to(dev, non_blocking=True)
            vals = dplan.estimate_distributed(xd, dout) if native else P.distributed_estimate(xd, cfg, gather=True)
            if rank == 0:
                vals.cpu()
            torch.cuda.synchronize()
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        h2d = x_host.nbytes
        d2h = plan.npoints * (8 if prec == 32 else 16) if rank == 0 else 0
        t = torch.tensor([statistics.median(e2e_ms)], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = [float(t.item())]
    e2e_value = units / (statistics.median(e2e_ms) * 1e-3)

    result = None
    if rank == 0:
        clocks = sampler.summary()
        peak_tf, probe_mhz = peak_fp32(lib, cstream)
        roof = None
        if tri:
            t_tri = statistics.median(tri)
            achieved = FLOPS_PER_UNIT * units / (t_tri * 1e-3) / 1e12
            roof = {"bound": "fp32", "achieved": round(achieved, 3), "peak": round(peak_tf, 3), "unit": "TFLOP/s",
                    "frac": round(achieved / peak_tf, 4), "traffic": load_traffic(args.config),
                    "kernel": ("k_triple_cta" if lib.hos_plan_k2_kind(plan.handle) == 1 else "k_triple_w")
                              + (" (fp32 FFMA2 triple product)" if prec == 32 else " (fp64 DFMA triple product; peak below is the FP32 one)"), "kernel_ms": round(t_tri, 5),
                    "kernel_share_of_step": round(t_tri / ms_per_step, 3),
                    "stage_us": {k_: round(statistics.median(v_) * 1e3, 2) for k_, v_ in stages.items()},
                    "stage_timing": f"mean of {STAGE_REPS} launches per stage replayed as one CUDA graph, median of 3",
                    "peak_source": f"live FFMA2 outer-product microbenchmark (hos_peak_fp32) at {probe_mhz:.0f} MHz; "
                                   "MEASURED_PEAKS.json has no FP32 figure",
                    "tiling_efficiency": round(plan.units / plan.issued, 4)}
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32" if prec == 32 else "f64",
            "data": "synthetic (seeded BASELINE cfg2 bilinear process, paper_1805_11775_b200/signals.py)",
            "config": {"workload": c.name, "order": c.order, "n": c.n, "M": c.m, "K": c.k, "w": c.m3,
                       "L": c.m3 // 2, "taper": c.taper, "batch": batch, "precision": args.precision,
                       "units_per_step": units, "points_per_step": plan.npoints * batch,
                       "l2": "flushed: 256 MiB device write between timed steps (outside the events)",
                       "parallelism": f"segments sharded over {world} GPUs (NCCL reduce-scatter + halo"
                                      + (" inside the C-ABI)" if native else ", torch.distributed)")
                       if world > 1 else "1 GPU"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": statistics.median(e2e_ms),
                    "path": "hos_estimate_host (C-ABI, pinned host buffers, copies inside the timed call)"
                    if world == 1 else "pinned H2D + distributed_estimate + rank-0 D2H"},
            "roofline": roof,
            "clocks": clocks,
            "gpu_launches": lib.hos_plan_launches(plan.handle) * args.steps if world == 1 else None,
            "gpu_launches_note": "per step: front end (k_front: fused demean+Hann+FFT+extension; or k_prep + "
                                 "cuFFT + k_extend_half for non-power-of-two M, cuFFT not counted), k_triple_cta (k_triple_w for large M), "
                                 "smoothing (k_line_scan + k_box3/k_box4, or k_smooth_series3 for grids that fit in "
                                 "shared memory)",
        }
        if not args.no_cpu_baseline and world == 1:
            cb = cpu_baseline(args.config, steps=1, warmup=1, segments=args.cpu_segments)
            result["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if result is not None:
        print(json.dumps(result))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from paper_1805_11775_b200 import signals

    c = signals.baseline_config(args.config)
    # every step is one bounded sample of the workload (~60 ms on 16 cores); K and
    # W as requested, K cut short only if the run would exceed ~150 s
    cb = cpu_baseline(args.config, steps=max(1, args.steps), warmup=max(1, args.warmup), segments=args.cpu_segments,
                      budget_s=150.0)
    steps = cb["steps_timed"]
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": max(1, args.warmup), "ms_per_step": cb["seconds_per_step"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE cfg2 bilinear process)",
        "config": {"workload": c.name, "order": c.order, "n": c.n, "M": c.m, "K": c.k, "w": c.m3,
                   "taper": c.taper, "units_per_step": cb["units_per_step"]},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
