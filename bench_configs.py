#!/usr/bin/env python3
"""The other BASELINE.json configs on 1 B200, each beside the reference's own CPU path timed on
this host in the same run (oracle/_ref: the unmodified reference headers, -O3 -march; the
workload and thread count of every CPU figure are stated in its `sample`).  bench.py folds
``run_all()`` into its JSON line under ``configs``; run standalone it prints the same object.

  config0        DE rand/1/bin one generation, D=10, pop 100 (latency; graph / persistent / e2e)
  config1_fp32   batched evaluation fp32, D=1000, pop 1024 (tcgen05 3xFP16)
  config2        SHADE (ttpb/1, archive, midpoint), D=100, pop 180, 1000 generations, Ackley
  config3        synchronous PSO gbest / ring, fp64 / fp32, D=1000, pop 1024, 500 iterations
  config4        64 DE runs x 2000 generations, D=50, pop 100, 3-component composition, one launch
  hbm_update     update kernels at P=16384, D=1000 (L2-exceeding): DE trial / selection, PSO update

GPU numbers are CUDA-event timed on the launching stream after warm-up (device-resident inputs)
unless the key says e2e.  Per-kernel times come from the engines' phase events (CUDA events
recorded between the generation's kernels on its stream: evb_de_phase_ms / evb_pso_phase_ms).
"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402  (seeded inputs + the CPU baselines only)
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200 import _lib  # noqa: E402
from paper_2505_17430_b200.de import DEEngine, Rng, preset_de, preset_shade  # noqa: E402
from paper_2505_17430_b200.pso import PSOEngine, config3 as pso_config3  # noqa: E402
from paper_2505_17430_b200.runs import de_runs, run_keys  # noqa: E402

DEV = torch.device("cuda:0")
K2_TILE_N = 128  # N of the fp32 kernel's tcgen05.mma tiles (eval_gemm.cu eval_f32_umma_sk_kernel)
K2_KERNEL = "eval_f32_umma_sk_kernel"


def hbm_peak():
    """Measured HBM copy bandwidth (GB/s) from MEASURED_PEAKS.json, else the profiling guide's."""
    try:
        v = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
        return float(v), "MEASURED_PEAKS.json hbm_gbs"
    except Exception:
        return 6547.2, "fallback: /opt/skills/guides/B200_PROFILING.md measured copy bandwidth"


def dram_traffic(kernel):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum per launch (profiles/traffic.json), or None."""
    try:
        return json.loads((ROOT / "profiles" / "traffic.json").read_text()).get(kernel)
    except Exception:
        return None


def cpu_info():
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return model, os.cpu_count() or 1


def cpu_baseline(value, unit, cores, sample):
    model, _ = cpu_info()
    return {"value": value, "unit": unit, "cores": cores, "cpu_model": model, "kind": "reference",
            "lib": O.REF_FAST()._evb_name, "sample": sample}


def ev():
    return torch.cuda.Event(enable_timing=True)


def timed(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps  # ms


def wall_median(fn, n, blocks=5, warm_s=0.2):
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < warm_s:
        fn()
    torch.cuda.synchronize()
    per = max(1, n // blocks)
    out = []
    for _ in range(blocks):
        t0 = time.perf_counter()
        for _ in range(per):
            fn()
        out.append((time.perf_counter() - t0) / per)
    return statistics.median(out)


def config0():
    """DE rand/1/bin, F 0.5, CR 0.9, clip, D=10, pop 100, Rastrigin on 0.0512 M (x - o), seed 42."""
    P, D = 100, 10
    o, m = O.shift_rotation(42, D)
    m = m * 0.0512
    prob = evb.ProblemInstance.base(evb.BaseKind.rastrigin, o, m, 0.0)
    eng = DEEngine(preset_de(), P, D)
    rng = Rng.philox(42)
    pop = torch.empty((P, D), dtype=torch.float64, device=DEV)
    eng.init_population(pop, -100.0, 100.0, rng)
    fit = torch.empty(P, dtype=torch.float64, device=DEV)
    evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
    eager_ms = timed(lambda: eng.generation(prob, pop, fit, -100.0, 100.0, rng), 200)
    eng.generations(prob, pop, fit, -100.0, 100.0, rng, 10)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    eng.generations(prob, pop, fit, -100.0, 100.0, rng, 1000)
    b.record()
    torch.cuda.synchronize()
    graph_ms = a.elapsed_time(b) / 1000
    # whole run in one persistent launch (K8 with one run: a 2-CTA cluster), per generation
    keys = run_keys(42, 1)
    pops = torch.empty((1, P, D), dtype=torch.float64, device=DEV)
    fits = torch.empty((1, P), dtype=torch.float64, device=DEV)
    de_runs(preset_de(), [prob], keys, pops, fits, 20, -100.0, 100.0, init=True, gen0=0)
    G = 2000
    a2, b2 = ev(), ev()
    a2.record()
    de_runs(preset_de(), [prob], keys, pops, fits, G, -100.0, 100.0, init=True, gen0=0)
    b2.record()
    torch.cuda.synchronize()
    persist_ms = a2.elapsed_time(b2) / G
    # config 0 as stated from the host: population + fitness in pinned host memory, one
    # generation (K8, one launch), population + fitness back; wall clock with the copies
    hp = pops[0].cpu().pin_memory()
    hf = fits[0].cpu().pin_memory()
    gen = [21]

    def host_generation():
        pops[0].copy_(hp, non_blocking=True)
        fits[0].copy_(hf, non_blocking=True)
        de_runs(preset_de(), [prob], keys, pops, fits, 1, -100.0, 100.0, init=False, gen0=gen[0])
        hp.copy_(pops[0], non_blocking=True)
        hf.copy_(fits[0], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        gen[0] += 1

    e2e_k8_s = wall_median(host_generation, 500)
    # the same through the engine (de_engine::generation's shape): state from pinned host memory,
    # evb_de_generations(1) (the persistent cluster kernel), state back; wall clock with the copies
    eng_h = DEEngine(preset_de(), P, D)
    rng_h = Rng.philox(42)
    state_d = torch.empty(P * D + P, dtype=torch.float64, device=DEV)  # [population | fitness]: one copy each way
    pop_h = state_d[:P * D].view(P, D)
    fit_h = state_d[P * D:]
    eng_h.init_population(pop_h, -100.0, 100.0, rng_h)
    evb.evaluate_batch(prob, pop_h, evb.EvalScratch(), fit_h)
    state_h = state_d.cpu().pin_memory()
    cur = torch.cuda.current_stream()

    def host_generation_engine():
        state_d.copy_(state_h, non_blocking=True)
        eng_h.generations(prob, pop_h, fit_h, -100.0, 100.0, rng_h, 1)
        state_h.copy_(state_d, non_blocking=True)
        cur.synchronize()

    e2e_s = wall_median(host_generation_engine, 500)
    # the reference caller's shape in C++: de_engine state in host memory, one generation per call
    # through evb_de_generations_host (libevb_refshape.so, no Python in the loop)
    cxx = None
    try:
        import ctypes

        R = ctypes.CDLL(str(ROOT / "paper_2505_17430_b200" / "libevb_refshape.so"))
        R.evb_refshape_time_de.restype = ctypes.c_int
        hp3 = state_h[:P * D].numpy().reshape(P, D).copy()
        hf3 = state_h[P * D:].numpy().copy()
        us = (ctypes.c_double * 5)()
        mr = np.ascontiguousarray(m)
        rc = R.evb_refshape_time_de(D, P, ctypes.c_void_p(o.ctypes.data), ctypes.c_void_p(mr.ctypes.data),
                                    ctypes.c_void_p(hp3.ctypes.data), ctypes.c_void_p(hf3.ctypes.data),
                                    ctypes.c_uint64(42), 2000, 5, ctypes.c_double(0.3), us)
        if rc == 0:
            u = statistics.median(list(us))
            cxx = {"value": 1e6 / u, "unit": "generations/s", "us_per_generation": u,
                   "h2d_bytes_per_step": P * D * 8 + P * 8, "d2h_bytes_per_step": P * D * 8 + P * 8,
                   "how": "C++ over the C ABI: evb_de_generations_host(engine, problem, host pop, host fitness, 1) "
                          "per generation (one copy in, the persistent kernel, one copy out, synchronous); wall clock, "
                          "median of 5 blocks"}
    except OSError as exc:
        cxx = {"unavailable": str(exc)}
    cpu_s = O.REF_FAST().ref_bench_de(0, P, D, 2000, 5, O.ptr(o), O.ptr(np.ascontiguousarray(m)), 42)
    cpu_gps = 2000 / cpu_s
    return {
        "metric": "generations/s (one DE generation: mutate, cross, repair, evaluate, select)",
        "value": 1e3 / graph_ms, "unit": "generations/s",
        "how": "DEEngine.generations(1000): all generations in one persistent cluster launch (de_run_kernel); "
               "device time per generation ('eager': one evb_de_generation call per generation, 5 kernels)",
        "us_per_generation": {"engine_persistent": graph_ms * 1e3, "eager": eager_ms * 1e3,
                              "persistent_k8": persist_ms * 1e3},
        "persistent_k8": {"value": 1e3 / persist_ms, "unit": "generations/s",
                          "how": "de_runs: init + 2000 generations of the run in one launch"},
        "e2e": {"value": 1.0 / e2e_s, "unit": "generations/s", "us_per_generation": e2e_s * 1e6,
                "h2d_bytes_per_step": P * D * 8 + P * 8, "d2h_bytes_per_step": P * D * 8 + P * 8,
                "how": "population + fitness (one pinned buffer, one copy each way) from host memory, one engine generation "
                       "(DEEngine.generations(1): the persistent cluster kernel), back to the host; wall clock incl. "
                       "copies and sync, median of 5 blocks",
                "k8": {"value": 1.0 / e2e_k8_s, "unit": "generations/s", "us_per_generation": e2e_k8_s * 1e6,
                       "how": "the same step through de_runs (K8, one generation)"},
                "cxx_host_state": cxx},
        "roofline": {"bound": "latency", "note": "about 20 KFLOP and 80 KB per generation (SURVEY §8(d)): "
                                                  "launch and dependency latency, no throughput roofline"},
        "cpu_baseline": cpu_baseline(cpu_gps, "generations/s", 1,
                                     "build_de_fixed(0.5, 0.9) on the config-0 problem, 2000 generations on its "
                                     "native stream, 1 thread (a single run has no reference parallelism)"),
        "e2e_vs_cpu": (1.0 / e2e_s) / cpu_gps,
    }


def config1_fp32():
    """Batched evaluation fp32, D=1000, pop 1024 (seed 7): elliptic + Rastrigin + Ackley per step."""
    D, P = 1000, 1024
    o, m = O.shift_rotation(7, D)
    X = O.population(7, P, D)
    o32, m32, X32 = o.astype(np.float32), m.astype(np.float32), X.astype(np.float32)
    kinds = (evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley)
    probs = [evb.ProblemInstance.base(k, o32, m32, 0.0, dtype=evb.EVB_F32) for k in kinds]
    sc = evb.EvalScratch()
    Xd = torch.from_numpy(X32).to(DEV)
    outs = [torch.empty(P, dtype=torch.float32, device=DEV) for _ in kinds]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=DEV)
    stream = torch.cuda.current_stream()
    for _ in range(5):
        for p, f in zip(probs, outs):
            evb.evaluate_batch(p, Xd, sc, f, stream)
    torch.cuda.synchronize()
    steps = 100
    evs = [[(ev(), ev()) for _ in kinds] for _ in range(steps)]
    for s in range(steps):
        flush.zero_()
        for (a, b), p, f in zip(evs[s], probs, outs):
            a.record(stream)
            evb.evaluate_batch(p, Xd, sc, f, stream)
            b.record(stream)
    torch.cuda.synchronize()
    launch_ms = [a.elapsed_time(b) for e in evs for (a, b) in e]
    batch_ms = statistics.mean(launch_ms)
    step_ms = batch_ms * len(kinds)
    # the same launches back to back (no flush, one event pair around 300 steps): the kernel's own
    # duration with the next launch's prologue overlapping its tail, as inside a PSO / DE generation
    a2, b2 = ev(), ev()
    a2.record(stream)
    for _ in range(300):
        for p, f in zip(probs, outs):
            evb.evaluate_batch(p, Xd, sc, f, stream)
    b2.record(stream)
    torch.cuda.synchronize()
    b2b_us = a2.elapsed_time(b2) * 1e3 / (300 * len(kinds))
    flop = 2.0 * D * D * P
    achieved = flop / (batch_ms * 1e-3) / 1e12
    tf32 = _lib.probe_umma_f16_tflops(K2_TILE_N)  # the kernel's MMAs are kind::f16 (3xFP16 split)
    tf32_256 = _lib.probe_umma_f16_tflops(256)
    peak = tf32 / 3.0
    # CPU: the reference's float evaluate_batch (fast_cos) for the three objectives, all threads
    L = O.REF_FAST()
    thr = os.cpu_count() or 1
    jobs, keep = [], []
    for kind in (1, 5, 6):
        mr = np.ascontiguousarray(m32.ravel())
        keep.append(mr)
        jobs.append(L.ref_batch_job_create(0, kind, D, O.ptr(o32), O.ptr(mr), 0.0, P, O.ptr(X32)))
    L.ref_batch_job_run(jobs[0], thr, None)
    t0 = time.perf_counter()
    reps = 0
    while reps < 2 or time.perf_counter() - t0 < 3.0:
        for j in jobs:
            L.ref_batch_job_run(j, thr, None)
        reps += 1
    el = time.perf_counter() - t0
    for j in jobs:
        L.ref_batch_job_destroy(j)
    cpu_v = reps * 3 * P / el
    return {
        "metric": "objective evals/sec (D=1000, pop 1024, fp32)", "value": 3 * P / (step_ms * 1e-3),
        "unit": "evals/s", "ms_per_batch": batch_ms,
        "back_to_back": {"us_per_launch": b2b_us, "evals_per_s": P / (b2b_us * 1e-6),
                         "tflops_fp32_equivalent": flop / (b2b_us * 1e-6) / 1e12,
                         "how": "900 launches back to back (no L2 flush, one event pair): mean over the "
                                "elliptic / Rastrigin / Ackley problems"},
        "how": "3 x evaluate_batch fp32 per step (eval_f32_umma_sk_kernel: tcgen05 kind::f16 128x128 tiles, "
               "3xFP16 split in-kernel (fp16 head + remainder of S = X - o and of 2^8 M: 22 significant bits), "
               "TMEM accumulators, K halves as a 2-CTA cluster exchanging z over DSMEM, "
               "M pairs multicasting the rotation slices); CUDA events per launch; L2 flushed between steps",
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s (fp32-equivalent)",
                     "frac": achieved / peak, "traffic": dram_traffic(K2_KERNEL),
                     "kernel": K2_KERNEL,
                     "peak_source": f"in-run tcgen05.mma kind::f16 probe at N={K2_TILE_N}: {tf32:.1f} TFLOP/s, "
                                    f"divided by 3 (3xFP16: three tensor-core products per fp32 product); "
                                    f"at N=256 the probe reads {tf32_256:.1f}",
                     "algorithmic": f"2*D^2*P = {flop:.4g} flop per launch (x3 on the tensor core)",
                     "tensor_pipe_frac": 3 * achieved / tf32},
        "cpu_baseline": cpu_baseline(cpu_v, "evals/s", thr,
                                     f"{reps} full steps (3 x evaluate_batch<float> of {P} points, D={D}) in "
                                     f"{el:.1f} s, batch split into {thr} contiguous slices"),
    }


def config2():
    """SHADE preset (ttpb/1 p 0.11 + archive, binomial, midpoint, shade(H=180)), D=100, pop 180."""
    P, D, G = 180, 100, 1000
    o, m = O.shift_rotation(11, D)
    prob = evb.ProblemInstance.base(evb.BaseKind.ackley, o, m, 0.0)
    eng = DEEngine(preset_shade(0.11, P, 1.0), P, D)
    rng = Rng.philox(11)
    pop = torch.empty((P, D), dtype=torch.float64, device=DEV)
    fit = torch.empty(P, dtype=torch.float64, device=DEV)

    def init():
        eng.reset()
        eng.init_population(pop, -100.0, 100.0, rng)
        evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)

    init()
    eng.generations(prob, pop, fit, -100.0, 100.0, rng, G)
    init()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    eng.generations(prob, pop, fit, -100.0, 100.0, rng, G)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    eng.phase_timing(True)
    phases = []
    for _ in range(5):
        eng.generation(prob, pop, fit, -100.0, 100.0, rng)
        phases.append(eng.phase_ms())
    eng.phase_timing(False)
    ph = {k: statistics.median(p[k] for p in phases) * 1e3 for k in phases[0]}
    cpu_s = O.REF_FAST().ref_bench_de(1, P, D, G, 6, O.ptr(o), O.ptr(np.ascontiguousarray(m)), 11)
    return {
        "metric": "generations/s (config 2, 1000 generations)", "value": G / (ms * 1e-3), "unit": "generations/s",
        "ms_1000_generations": ms, "best_fitness": float(fit.min()),
        "how": "DEEngine.generations over 1000 generations: all of them in one persistent cluster launch "
               "(de_run_kernel, 16 CTAs), device time",
        "eager_us_per_phase": ph,
        "roofline": {"bound": "latency", "note": "population 144 KB, L2-resident; one cluster runs the whole run: "
                                                  "cluster barriers, serial per-individual draws and exact-order "
                                                  "dots bound a generation (DESIGN.md); eager_us_per_phase: the "
                                                  "per-generation multi-kernel path's phases (events between kernels)"},
        "cpu_baseline": cpu_baseline(G / cpu_s, "generations/s", 1,
                                     "build_shade(0.11, 180, 1.0), the full 1000 generations on its native stream, "
                                     "1 thread (a single run has no reference parallelism)"),
    }


def config3():
    """Synchronous PSO (w 0.7298, c1 = c2 = 1.49618, |v| <= 40), elliptic, D=1000, pop 1024."""
    P, D, G = 1024, 1000, 500
    o, m = O.shift_rotation(13, D)
    hbm, _ = hbm_peak()
    peak64 = _lib.probe_peak_tflops(0)
    tf32 = _lib.probe_umma_f16_tflops(K2_TILE_N)  # fp32 evaluation: kind::f16 MMAs (3xFP16)
    res = {"metric": "iterations/s (500 iterations, D=1000, pop 1024)", "unit": "iterations/s", "variants": {}}
    for nd, dt, tdt in ((np.float64, evb.EVB_F64, torch.float64), (np.float32, evb.EVB_F32, torch.float32)):
        prob = evb.ProblemInstance.base(evb.BaseKind.elliptic, o.astype(nd), m.astype(nd), 0.0, dtype=dt)
        for topo in ("gbest", "lbest_ring"):
            eng = PSOEngine(pso_config3(topo), P, D, dt)
            rng = Rng.philox(13)
            X = torch.empty((P, D), dtype=tdt, device=DEV)
            V = torch.empty((P, D), dtype=tdt, device=DEV)
            fit = torch.empty(P, dtype=tdt, device=DEV)
            eng.init_uniform(X, -100.0, 100.0, rng)
            eng.init_uniform(V, -20.0, 20.0, rng)
            evb.evaluate_batch(prob, X, evb.EvalScratch(), fit)
            eng.prepare(X, fit)
            for _ in range(3):
                eng.generation(prob, X, V, fit, -100.0, 100.0, rng)
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record()
            for _ in range(G):
                eng.generation(prob, X, V, fit, -100.0, 100.0, rng)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            eng.phase_timing(True)
            phases = []
            for _ in range(5):
                eng.generation(prob, X, V, fit, -100.0, 100.0, rng)
                phases.append(eng.phase_ms())
            eng.phase_timing(False)
            ph = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
            s = np.dtype(nd).itemsize
            upd_bytes = 5 * s * P * D
            ev_flop = 2.0 * D * D * P
            ev_peak = peak64 if nd == np.float64 else tf32 / 3.0
            res["variants"][f"{np.dtype(nd).name}_{topo}"] = {
                "value": G / (ms * 1e-3), "evals_per_s": P * G / (ms * 1e-3), "ms_500_iterations": ms,
                "best_pbest": float(eng.personal_bests()["pbest_fit"].min()),
                "us_per_phase": {k: v * 1e3 for k, v in ph.items()},
                "evaluate_tflops": ev_flop / (ph["evaluate"] * 1e-3) / 1e12,
                "evaluate_frac": ev_flop / (ph["evaluate"] * 1e-3) / 1e12 / ev_peak,
                "update_gbps_algorithmic": upd_bytes / (ph["update"] * 1e-3) / 1e9,
                "update_note": f"5*s*P*D = {upd_bytes / 1e6:.1f} MB per iteration; L2-resident at this size "
                               f"(see hbm_update for the L2-exceeding sweep against {hbm:.0f} GB/s)"}
    v = res["variants"]
    res["value"] = v["float64_gbest"]["value"]
    res["how"] = ("PSOEngine.generation x 500 (neighbour best, fused velocity/position update, batched fused-GEMM "
                  "evaluation, personal best; PDL), device time; value = fp64 gbest")
    # CPU: the synchronous driver over the reference's pieces, evaluation over all host threads
    thr = os.cpu_count() or 1
    O.REF_FAST()
    cpu = {}
    for nd in (np.float64, np.float32):
        xs = O.population(13, P, D).astype(nd)
        vs = np.random.default_rng(0).uniform(-20, 20, (P, D)).astype(nd)
        f0 = O.eval_batch(1, o, m, 0.0, xs.astype(np.float64)).astype(nd)
        ref = O.RefPSO(nd, 0, 0.7298, 1.49618, 1.49618, 40.0, P, D, 1, o.astype(nd), m.astype(nd))
        ref.set(xs, vs, f0)
        ref.set_threads(thr)
        iters = 3
        t0 = time.perf_counter()
        for it in range(iters):
            words = np.random.default_rng(1 + it).integers(0, 2**63, size=2 * P * D, dtype=np.uint64)
            ref.step(words, -100.0, 100.0)
        cpu[np.dtype(nd).name] = iters / (time.perf_counter() - t0)
    res["cpu_baseline"] = cpu_baseline(cpu["float64"], "iterations/s", thr,
                                       f"3 synchronous gbest iterations, fp64, the reference's topology / "
                                       f"standard_update / problem_instance::evaluate, evaluation over {thr} threads "
                                       f"(exact build); fp32: {cpu['float32']:.2f} iterations/s")
    return res


def config4():
    """64 independent DE/rand/1/bin runs, D=50, pop 100, 2000 generations, 3-component composition."""
    n_runs, P, D, G = 64, 100, 50, 2000
    probs, shifts, rots = [], [], []
    for r in range(n_runs):
        s, mm = O.composition_components(4000 + r, D)
        shifts.append(s)
        rots.append(mm)
        probs.append(evb.ProblemInstance.composition(O.CONFIG4_KINDS, s, mm, O.CONFIG4_SIGMA, O.CONFIG4_LAMBDA,
                                                     O.CONFIG4_BIAS, 0.0))
    keys = run_keys(64, n_runs)
    pops = torch.empty((n_runs, P, D), dtype=torch.float64, device=DEV)
    fits = torch.empty((n_runs, P), dtype=torch.float64, device=DEV)
    de_runs(preset_de(), probs, keys, pops, fits, 20, -100.0, 100.0)  # warm-up
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    de_runs(preset_de(), probs, keys, pops, fits, G, -100.0, 100.0)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    peak64 = _lib.probe_peak_tflops(0)
    flop = 3 * 2.0 * D * D * P * n_runs * G  # three component contractions per trial
    sh = np.ascontiguousarray(np.stack(shifts))
    ro = np.ascontiguousarray(np.stack(rots))
    k = np.array(O.CONFIG4_KINDS, np.int32)
    sg, la, cb = (np.array(v) for v in (O.CONFIG4_SIGMA, O.CONFIG4_LAMBDA, O.CONFIG4_BIAS))
    thr = os.cpu_count() or 1
    cpu_s = O.REF_FAST().ref_bench_config4(n_runs, P, D, G, thr, O.ptr(sh), O.ptr(ro), O.ptr(k), O.ptr(sg),
                                           O.ptr(la), O.ptr(cb))
    return {
        "metric": "run-generations/s (64 runs x 2000 generations in one launch)",
        "value": n_runs * G / (ms * 1e-3), "unit": "run-generations/s", "ms_total": ms,
        "generations_per_s_per_run": G / (ms * 1e-3),
        "how": "de_runs (K8): init + 2000 generations of all 64 runs in one persistent launch, device time",
        "best_fitness_run0": float(fits[0].min()),
        "roofline": {"bound": "fp64", "achieved": flop / (ms * 1e-3) / 1e12, "peak": peak64, "unit": "TFLOP/s",
                     "frac": flop / (ms * 1e-3) / 1e12 / peak64, "kernel": "de_runs_kernel",
                     "traffic": dram_traffic("de_runs_kernel"),
                     "algorithmic": f"3 x 2*D^2 flop per trial evaluation = {flop:.4g} flop per launch",
                     "peak_source": "in-run DMMA probe (FP64 tensor peak)"},
        "cpu_baseline": cpu_baseline(n_runs * G / cpu_s, "run-generations/s", thr,
                                     f"evo_bench + the `de` preset over all {n_runs} runs x {G} generations "
                                     f"(the reference's own multithreaded task pool), {thr} threads, {cpu_s:.1f} s"),
    }


def hbm_update():
    """Update kernels alone at P=16384, D=1000 fp64 (131 MB per matrix: beyond the 126 MB L2)."""
    P, D = 16384, 1000
    hbm, hbm_src = hbm_peak()
    o, m = O.shift_rotation(13, D)
    prob = evb.ProblemInstance.base(evb.BaseKind.sphere, o, m, 0.0)
    res = {"peak_gbps": hbm, "peak_source": hbm_src, "dims": {"P": P, "D": D, "dtype": "f64"}}
    eng = DEEngine(preset_de(), P, D)
    rng = Rng.philox(5)
    pop = torch.empty((P, D), dtype=torch.float64, device=DEV)
    eng.init_population(pop, -100.0, 100.0, rng)
    fit = torch.empty(P, dtype=torch.float64, device=DEV)
    evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
    eng.generation(prob, pop, fit, -100.0, 100.0, rng)
    eng.phase_timing(True)
    phases, wins = [], []
    for _ in range(5):
        f0 = fit.clone()
        eng.generation(prob, pop, fit, -100.0, 100.0, rng)
        phases.append(eng.phase_ms())
        wins.append(int((fit != f0).sum()))
    eng.phase_timing(False)
    ph = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
    s = 8
    trial_alg = 5 * s * P * D  # 1 target + 3 donor rows read, 1 trial row written
    trial_min = 2 * s * P * D  # compulsory DRAM: the population once (donors re-read from L2) + trial write

    def rec(kernel, ms, alg, note):
        out = {"us": ms * 1e3, "algorithmic_bytes": alg, "gbps_algorithmic": alg / (ms * 1e-3) / 1e9,
               "frac_algorithmic": alg / (ms * 1e-3) / 1e9 / hbm, "note": note}
        t = dram_traffic(kernel)
        if t:
            out["dram_bytes_ncu"] = t
            out["gbps_dram"] = t / (ms * 1e-3) / 1e9
            out["frac_dram"] = out["gbps_dram"] / hbm
        return out

    res["de_trial_stage_kernel"] = rec("de_trial_stage_kernel", ph["trial"], trial_alg,
                                       f"5*s*P*D algorithmic; compulsory DRAM 2*s*P*D = {trial_min / 1e6:.0f} MB "
                                       f"(donor rows hit L2); rows staged by cp.async through a 3-stage "
                                       f"per-warp shared-memory ring")
    res["de_trial_stage_kernel"]["frac_compulsory"] = trial_min / (ph["trial"] * 1e-3) / 1e9 / hbm
    winners = statistics.median(wins)  # rows replaced (fitness changed) per generation
    res["de_select_apply_kernel"] = rec("de_select_apply_kernel", ph["select_apply"], int(3 * s * winners * D),
                                        f"s*D*(trial read + parent read + write) per winner; {winners:.0f} of {P} "
                                        f"trials won (median of the timed generations)")
    res["de_select_multi_kernel"] = {"us": ph["select_scan"] * 1e3,
                                     "note": "flags, look-back prefix sums over ticketed CTAs, archive slots"}
    res["de_phase_us"] = {k: v * 1e3 for k, v in ph.items()}
    # PSO update (config 3's rule) at the same size
    eng2 = PSOEngine(pso_config3("gbest"), P, D)
    X = torch.empty((P, D), dtype=torch.float64, device=DEV)
    V = torch.empty((P, D), dtype=torch.float64, device=DEV)
    f2 = torch.empty(P, dtype=torch.float64, device=DEV)
    eng2.init_uniform(X, -100.0, 100.0, rng)
    eng2.init_uniform(V, -20.0, 20.0, rng)
    sc = evb.EvalScratch()
    evb.evaluate_batch(prob, X, sc, f2)
    eng2.prepare(X, f2)
    eng2.generation(prob, X, V, f2, -100.0, 100.0, rng, sc)
    eng2.phase_timing(True)
    phases = []
    for _ in range(5):
        eng2.generation(prob, X, V, f2, -100.0, 100.0, rng, sc)
        phases.append(eng2.phase_ms())
    eng2.phase_timing(False)
    pp = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
    res["pso_update_vec_kernel"] = rec("pso_update_vec_kernel", pp["update"], 5 * s * P * D,
                                       "5*s*P*D: x, v, pbest read; x, v written (gbest row from L2)")
    res["pso_phase_us"] = {k: v * 1e3 for k, v in pp.items()}
    return res


def run_all(only=None):
    out = {}
    for name, fn in (("config0", config0), ("config1_fp32", config1_fp32), ("config2", config2),
                     ("config3", config3), ("config4", config4), ("hbm_update", hbm_update)):
        if only and name not in only:
            continue
        t0 = time.perf_counter()
        try:
            out[name] = fn()
        except Exception as exc:  # one config failing must not lose the others
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
        out[name]["wall_s"] = time.perf_counter() - t0
    return out


if __name__ == "__main__":
    import argparse

    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=None)
    args = ap.parse_args()
    print(json.dumps({"device": torch.cuda.get_device_name(0), "configs": run_all(args.only)}, indent=1), flush=True)
