#!/usr/bin/env python3
"""Headline benchmark: BASELINE.json config 1 — batched objective evaluation, fp64, D=1000,
pop=1024 (seed 7), on 1 B200 (N>1: independent replicas, weak scaling).

One step = the three config-1 objectives (elliptic, Rastrigin, Ackley; shared o and M)
evaluated over the 1024-point population through ``evaluate_batch_problems`` — one launch of the
multi-problem fused TMA + DMMA kernel (three contractions, X staged once per K-slice), 3072
objective evaluations; ``per_problem`` times the same step as 3 ``evaluate_batch`` launches.  The reference arm (``--impl reference``) does the
identical work through the reference's own ``problems::evaluate_batch`` (compiled from
/root/reference by oracle/Makefile into oracle/_ref) on all host cores.

Timing: W warm-up steps, then K steps each bracketed by CUDA events on the launching stream; L2
is flushed (256 MiB write) between steps outside the events; barrier + synchronize on both
sides; max over ranks.  ``e2e`` repeats the step through the C-ABI host-buffer entry point
(evb_evaluate_batch_host_many: the pinned population copied in once per step, three fitness
vectors out, all inside the timed region); ``e2e.per_call`` uses one host call per objective.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

D, P, SEED = 1000, 1024, 7
KINDS = ("elliptic", "rastrigin", "ackley")
METRIC = "objective evals/sec (D=1000, pop 1024, fp64) and % of FP64/HBM roofline, 1 B200"
UNIT = "evals/s"
CONFIG = {
    "workload": "config1: batched shifted-rotated evaluation, fp64, D=1000, pop=1024, seed 7; "
                "one step = elliptic + Rastrigin + Ackley over the population (three problems, one "
                "evaluate_batch_problems launch; per_problem: 3 x evaluate_batch)",
    "dim": D,
    "pop": P,
    "objectives_per_step": 3,
    "evals_per_step": 3 * P,
    "l2": "flushed between steps (256 MiB write outside the timed events)",
    "parallelism": "replicas",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="evb", choices=["evb", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs (bench_configs.py)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_inputs():
    import oracle as O  # seeded input generator (restated draw_shift / random_rotation / init_population)

    o, m = O.shift_rotation(SEED, D)
    X = O.population(SEED, P, D)
    return o, m, X


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline_reference(o, m, X, budget_s: float = 6.0):
    """The reference's own evaluate_batch (oracle/_ref, -O3 -march, all host threads)."""
    import numpy as np

    import oracle as O

    L = O.REF_FAST()
    threads = os.cpu_count() or 1
    n = P
    jobs = []
    keep = []
    for kind in KINDS:
        kid = {"elliptic": 1, "rastrigin": 5, "ackley": 6}[kind]
        mr = np.ascontiguousarray(m.ravel())
        keep.append(mr)
        jobs.append(L.ref_batch_job_create(1, kid, D, O.ptr(o), O.ptr(mr), 0.0, n, O.ptr(X)))
    L.ref_batch_job_run(jobs[0], threads, None)  # warm-up
    t0 = time.perf_counter()
    reps = 0
    while True:
        for j in jobs:
            L.ref_batch_job_run(j, threads, None)
        reps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    el = time.perf_counter() - t0
    for j in jobs:
        L.ref_batch_job_destroy(j)
    return {
        "value": reps * 3 * n / el,
        "unit": UNIT,
        "cores": threads,
        "cpu_model": cpu_model(),
        "kind": "reference",
        "sample": f"{reps} full config-1 steps (3 x evaluate_batch of {n} points, D={D}, fp64) in {el:.1f} s, "
                  f"batch split into {threads} contiguous slices; {L._evb_name}",
    }


def run_reference(args, rank, world):
    """--impl reference: the reference CPU implementation on the host cores, same metric."""
    if rank != 0:
        return
    import numpy as np

    import oracle as O

    o, m, X = make_inputs()
    L = O.REF_FAST()
    threads = os.cpu_count() or 1
    sample = P  # the full step: 3 x evaluate_batch over all 1024 points (same config as the GPU arm)
    jobs, keep = [], []
    for kind in KINDS:
        kid = {"elliptic": 1, "rastrigin": 5, "ackley": 6}[kind]
        mr = np.ascontiguousarray(m.ravel())
        keep.append(mr)
        jobs.append(L.ref_batch_job_create(1, kid, D, O.ptr(o), O.ptr(mr), 0.0, sample, O.ptr(X)))
    for _ in range(args.warmup):
        for j in jobs:
            L.ref_batch_job_run(j, threads, None)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for j in jobs:
            L.ref_batch_job_run(j, threads, None)
        times.append(time.perf_counter() - t0)
    for j in jobs:
        L.ref_batch_job_destroy(j)
    total = sum(times)
    value = args.steps * 3 * sample / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": CONFIG,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(), "kind": "reference",
                         "sample": f"every step is the full config-1 step: 3 x evaluate_batch of all {P} points "
                                   f"(D={D}, fp64), batch split into {threads} contiguous slices, one eval_scratch "
                                   f"each; {L._evb_name} (reference headers, -O3 -march)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_evb(args, rank, world, local):
    import numpy as np
    import torch

    import paper_2505_17430_b200 as evb
    from paper_2505_17430_b200 import _lib

    from paper_2505_17430_b200 import dist as pdist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = pdist.init("nccl", device=dev)  # replicas: barrier + max-over-ranks only

    o, m, X = make_inputs()
    kinds = [getattr(evb.BaseKind, k) for k in KINDS]
    probs = [evb.ProblemInstance.base(k, o, m, 0.0) for k in kinds]
    sc = evb.EvalScratch()
    Xd = torch.from_numpy(X).to(dev)
    outs = [torch.empty(P, dtype=torch.float64, device=dev) for _ in kinds]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step_per_problem(evs=None):
        for i, p in enumerate(probs):
            if evs is not None:
                evs[2 * i].record(stream)
            evb.evaluate_batch(p, Xd, sc, outs[i], stream)
            if evs is not None:
                evs[2 * i + 1].record(stream)

    def step(evs=None):  # the three problems in one multi-problem launch (X staged once per stage)
        if evs is not None:
            evs[0].record(stream)
        evb.evaluate_batch_problems(probs, Xd, sc, outs, stream)
        if evs is not None:
            evs[1].record(stream)

    for _ in range(args.warmup):
        flush.zero_()
        step()
        flush.zero_()
        step_per_problem()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    launches0 = evb.launch_count()
    sampler = ClockSampler(local)
    with sampler:
        for s in range(args.steps):
            flush.zero_()  # L2 flush outside the timed events
            step(ev[s])
        torch.cuda.synchronize()
    launches = evb.launch_count() - launches0
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    launch_ms = [e[0].elapsed_time(e[1]) for e in ev]
    total_ms = pdist.max_over_ranks(sum(launch_ms), dist, dev)
    value = world * args.steps * 3 * P / (total_ms * 1e-3)

    # the same step as three evaluate_batch launches (one per problem, the reference's call shape)
    evp = [[torch.cuda.Event(enable_timing=True) for _ in range(2 * len(probs))] for _ in range(args.steps)]
    for s in range(args.steps):
        flush.zero_()
        step_per_problem(evp[s])
    torch.cuda.synchronize()
    pp_launch_ms = [e[2 * i].elapsed_time(e[2 * i + 1]) for e in evp for i in range(len(probs))]
    pp_ms = pdist.max_over_ranks(sum(pp_launch_ms), dist, dev)
    per_problem = {"value": world * args.steps * 3 * P / (pp_ms * 1e-3), "unit": UNIT,
                   "ms_per_step": pp_ms / args.steps,
                   "tflops_per_launch": 2.0 * D * D * P / (statistics.mean(pp_launch_ms) * 1e-3) / 1e12,
                   "how": "3 x evaluate_batch per step (one fused TMA + DMMA launch per problem); L2 flushed "
                          "between steps"}

    # ---- roofline (dominant kernel: the fused multi-problem DMMA evaluation) ----
    flops_per_launch = 3 * 2.0 * D * D * P  # algorithmic: three z = M(x - o) contractions
    avg_launch_s = statistics.mean(launch_ms) * 1e-3
    achieved = flops_per_launch / avg_launch_s / 1e12
    peak = _lib.probe_peak_tflops(0)
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("eval_f64_dmma_multi_kernel")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": "eval_f64_dmma_multi_kernel<3>",
                "peak_source": "measured in-run: DMMA m8n8k4 throughput kernel over all SMs "
                               "(MEASURED_PEAKS.json has no FP64 figure)",
                "algorithmic": f"3 x 2*D^2*P = {flops_per_launch:.4g} flop per launch; compulsory bytes "
                               f"8*(3*D^2+P*D+3*D+3*P) = {8 * (3 * D * D + P * D + 3 * D + 3 * P) / 1e6:.2f} MB"}

    # ---- same z: config 1's wording ("three transforms are evaluated on the same z") taken
    # literally — one contraction, three fused epilogues (evb_evaluate_batch_multi).  Reported
    # beside the headline, which evaluates the three objectives as three independent problems.
    out3 = torch.empty((len(kinds), P), dtype=torch.float64, device=dev)
    mk = [int(k) for k in kinds]
    for _ in range(args.warmup):
        flush.zero_()
        evb.evaluate_batch_multi(probs[0], mk, [0.0] * len(mk), Xd, sc, out3, stream)
    ev3 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for s in range(args.steps):
        flush.zero_()
        ev3[s][0].record(stream)
        evb.evaluate_batch_multi(probs[0], mk, [0.0] * len(mk), Xd, sc, out3, stream)
        ev3[s][1].record(stream)
    torch.cuda.synchronize()
    multi_ms = pdist.max_over_ranks(sum(a.elapsed_time(b) for a, b in ev3), dist, dev)
    same_z = {"value": world * args.steps * len(mk) * P / (multi_ms * 1e-3), "unit": UNIT,
              "ms_per_step": multi_ms / args.steps,
              "how": "evb_evaluate_batch_multi: one z = M(x - o) contraction per step, elliptic + Rastrigin + Ackley "
                     "epilogues fused (config 1: three transforms on the same z); L2 flushed between steps"}

    # ---- e2e: host buffers through the C ABI (pinned X in, fitness out) ----
    Xh = torch.from_numpy(X).pin_memory()
    outh = [torch.empty(P, dtype=torch.float64).pin_memory() for _ in kinds]
    import ctypes

    L = _lib.lib()

    def per_call_step():
        for i, p in enumerate(probs):
            _lib.check(L.evb_evaluate_batch_host(p.handle, sc.handle, ctypes.c_void_p(Xh.data_ptr()), P, D,
                                                 ctypes.c_void_p(outh[i].data_ptr())), "e2e")

    handles = (ctypes.c_void_p * len(probs))(*[p.handle.value for p in probs])
    optrs = (ctypes.c_void_p * len(probs))(*[o.data_ptr() for o in outh])

    def e2e_step():
        _lib.check(L.evb_evaluate_batch_host_many(handles, len(probs), sc.handle, ctypes.c_void_p(Xh.data_ptr()), P, D,
                                                  optrs), "e2e")

    def wall(fn, steps, blocks=5):
        # wall clock over `blocks` consecutive blocks of steps; the median block (a host-side
        # hiccup in one block — page-ins, another process — does not decide the figure); every
        # step of every block is a full host call with its copies and device sync
        # warm-up: at least W calls and 0.5 s of them — the host link comes out of its idle power
        # state only under sustained traffic (the first ~0.1-0.2 s of calls after the device-side
        # phases ran at up to 2x the steady per-call time, measured)
        t_w = time.perf_counter()
        n_w = 0
        while n_w < max(3, args.warmup) or time.perf_counter() - t_w < 0.5:
            fn()
            n_w += 1
        torch.cuda.synchronize()
        per = max(1, steps // blocks)
        times = []
        for _ in range(blocks):
            t0 = time.perf_counter()
            for _ in range(per):
                fn()
            torch.cuda.synchronize()
            times.append((time.perf_counter() - t0) / per)
        return pdist.max_over_ranks(statistics.median(times), dist, dev) * steps, [t * 1e6 for t in times]

    e2e_steps = max(200, args.steps)  # ~0.1 s of wall clock per arm
    e2e_s, e2e_blocks = wall(e2e_step, e2e_steps)
    per_call_s, _ = wall(per_call_step, e2e_steps)
    # the reference-shaped C++ binding: run_handle::evaluate_batch -> evb::evaluate_batch(problem,
    # vector<vector<double>>, scratch, out) (include/evb/evb.hpp), one call per objective, timed in C++
    reference_shape = None
    try:
        R = ctypes.CDLL(str(ROOT / "paper_2505_17430_b200" / "libevb_refshape.so"))
        R.evb_refshape_time.restype = ctypes.c_int
        blocks = 5
        us = (ctypes.c_double * blocks)()
        vals = np.empty((3, P))
        kinds_arr = (ctypes.c_int * 3)(*[int(k) for k in kinds])
        mr = np.ascontiguousarray(m)
        rc = R.evb_refshape_time(3, kinds_arr, D, P, ctypes.c_void_p(o.ctypes.data), ctypes.c_void_p(mr.ctypes.data),
                                 ctypes.c_void_p(X.ctypes.data), ctypes.c_int(max(100, args.steps // 2)),
                                 ctypes.c_int(blocks), ctypes.c_double(0.5), us,
                                 ctypes.c_void_p(vals.ctypes.data))
        if rc == 0:
            step_us = pdist.max_over_ranks(statistics.median(list(us)), dist, dev)
            reference_shape = {
                "value": world * 3 * P / (step_us * 1e-6), "unit": UNIT, "us_per_step": step_us,
                "us_per_step_blocks": list(us), "h2d_bytes_per_step": 3 * P * D * 8, "d2h_bytes_per_step": 3 * P * 8,
                "how": "C++: 3 x evb::evaluate_batch(gpu_problem, const vector<vector<double>>& xs, gpu_scratch&, "
                       "vector<double>& out) per step — the call run_handle<T>::evaluate_batch "
                       "(experiment/runner.hpp:47-53) makes; heap rows flattened into the scratch's pinned "
                       "staging, copied in, evaluated, values back into std::vector; wall clock, median of 5 blocks"}
        else:
            reference_shape = {"unavailable": f"evb_refshape_time returned {rc}"}
    except OSError as exc:
        reference_shape = {"unavailable": str(exc)}
    e2e = {"value": world * e2e_steps * 3 * P / e2e_s, "unit": UNIT, "h2d_bytes_per_step": P * D * 8,
           "d2h_bytes_per_step": 3 * P * 8,
           "how": "evb_evaluate_batch_host_many per step (C ABI): the step's population, pinned host memory, "
                  "crosses the host link once (the first wave's rows first) in column chunks that one "
                  "multi-problem fused GEMM (all three objectives, X read once per stage) consumes as they land; "
                  "fitness written to pinned host memory; wall clock with device sync, median of 5 blocks of steps, max over ranks",
           "us_per_step_blocks": e2e_blocks,
           "per_call": {"value": world * e2e_steps * 3 * P / per_call_s, "unit": UNIT,
                        "h2d_bytes_per_step": 3 * P * D * 8,
                        "how": "3 x evb_evaluate_batch_host (the population copied in once per objective)"},
           "reference_shape": reference_shape}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded draw_shift / random_rotation / "
                                                     "init_population, seed 7)",
        "config": CONFIG, "roofline": roofline, "e2e": e2e, "per_problem": per_problem, "same_z": same_z,
        "gpu_launches": launches,
        "clocks": sampler.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_reference(o, m, X)
        except Exception as exc:  # the checker is test infrastructure; report, do not crash the bench
            line["cpu_baseline"] = {"value": None, "unavailable": str(exc)}
    if rank == 0 and world == 1 and not args.no_configs:
        # BASELINE configs 0, 2, 3, 4, fp32 config 1 and the L2-exceeding update kernels, each with
        # its own unit, roofline and same-run reference CPU baseline (bench_configs.py)
        import bench_configs

        line["configs"] = bench_configs.run_all()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_evb(args, rank, world, local)


if __name__ == "__main__":
    main()
