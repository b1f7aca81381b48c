#!/usr/bin/env python3
"""All five BASELINE.json configs on 1 B200, each beside the reference's own CPU path timed on this
host (oracle/_ref: the unmodified reference headers, -O3 -march; bounded samples).  Prints one JSON
object; bench.py remains the headline (config 1).  GPU numbers are CUDA-event timed on the
launching stream after warm-up; device-resident inputs unless stated.

  config 0  DE rand/1/bin one generation, D=10, pop 100 (latency)
  config 1  batched evaluation fp64 / fp32, D=1000, pop 1024 (+ three kinds on one z)
  config 2  SHADE (ttpb/1, archive, midpoint), D=100, pop 180, 1000 generations, Ackley
  config 3  synchronous PSO gbest / ring, fp64 / fp32, D=1000, pop 1024, 500 iterations, elliptic
  config 4  64 DE runs x 2000 generations, D=50, pop 100, 3-component composition, one launch
  hbm       update kernels alone at P=16384, D=1000 (L2-exceeding): DE trial + selection, PSO update
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402  (inputs + CPU baseline only)
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200 import _lib  # noqa: E402
from paper_2505_17430_b200.de import DEEngine, Rng, preset_de, preset_shade  # noqa: E402
from paper_2505_17430_b200.pso import PSOEngine, config3  # noqa: E402
from paper_2505_17430_b200.runs import de_runs, run_keys  # noqa: E402

DEV = torch.device("cuda:0")
HBM_PEAK = 6547.2  # GB/s, MEASURED_PEAKS.json


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


def threads():
    return os.cpu_count() or 1


def cfg1(out):
    res = {}
    o, m = O.shift_rotation(7, 1000)
    X = O.population(7, 1024, 1000)
    peak64 = _lib.probe_peak_tflops(0)
    peak32 = _lib.probe_peak_tflops(1)
    for name, nd, dt, peak in (("fp64", np.float64, evb.EVB_F64, peak64), ("fp32", np.float32, evb.EVB_F32, peak32)):
        p = evb.ProblemInstance.base(evb.BaseKind.rastrigin, o.astype(nd), m.astype(nd), 0.0, dtype=dt)
        sc = evb.EvalScratch()
        Xd = torch.from_numpy(X.astype(nd)).to(DEV)
        f = torch.empty(1024, dtype=Xd.dtype, device=DEV)
        ms = timed(lambda: evb.evaluate_batch(p, Xd, sc, f), 50)
        tf = 2 * 1000 * 1000 * 1024 / (ms * 1e-3) / 1e12
        res[name] = {"ms_per_batch": ms, "evals_per_s": 1024 / (ms * 1e-3), "tflops": tf, "peak_tflops": peak,
                     "frac": tf / peak, "peak_source": "in-run probe (DMMA m8n8k4 / FFMA)"}
    p = evb.ProblemInstance.base(evb.BaseKind.elliptic, o, m, 0.0)
    sc = evb.EvalScratch()
    Xd = torch.from_numpy(X).to(DEV)
    f3 = torch.empty((3, 1024), dtype=torch.float64, device=DEV)
    ms = timed(lambda: evb.evaluate_batch_multi(p, [1, 5, 6], [0, 0, 0], Xd, sc, f3), 50)
    res["fp64_three_kinds_one_z"] = {"ms_per_batch": ms, "objective_values_per_s": 3 * 1024 / (ms * 1e-3)}
    out["config1"] = res


def cfg0(out):
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
    ms = timed(lambda: eng.generation(prob, pop, fit, -100.0, 100.0, rng), 200)
    a, b = ev(), ev()
    eng.generations(prob, pop, fit, -100.0, 100.0, rng, 10)
    torch.cuda.synchronize()
    a.record()
    eng.generations(prob, pop, fit, -100.0, 100.0, rng, 1000)
    b.record()
    torch.cuda.synchronize()
    ms_graph = a.elapsed_time(b) / 1000
    # end to end: one generation from host state, result read back
    t0 = time.perf_counter()
    for _ in range(20):
        eng.generation(prob, pop, fit, -100.0, 100.0, rng)
        fit.cpu()
    e2e_ms = (time.perf_counter() - t0) / 20 * 1e3
    # whole run in one persistent launch (K8, n_runs = 1: a 2-CTA cluster), per generation
    pops = torch.empty((1, P, D), dtype=torch.float64, device=DEV)
    fits = torch.empty((1, P), dtype=torch.float64, device=DEV)
    keys = run_keys(42, 1)
    de_runs(preset_de(), [prob], keys, pops, fits, 20, -100.0, 100.0, init=True, gen0=0)
    G = 2000
    a2, b2 = ev(), ev()
    a2.record()
    de_runs(preset_de(), [prob], keys, pops, fits, G, -100.0, 100.0, init=True, gen0=0)
    b2.record()
    torch.cuda.synchronize()
    ms_persist = a2.elapsed_time(b2) / G
    cpu_s = O.REF_FAST().ref_bench_de(0, P, D, 2000, 5, O.ptr(o), O.ptr(np.ascontiguousarray(m)), 42)
    out["config0"] = {"gpu_ms_per_generation": ms, "gpu_generations_per_s": 1e3 / ms,
                      "gpu_graph_ms_per_generation": ms_graph, "gpu_graph_generations_per_s": 1e3 / ms_graph,
                      "gpu_e2e_ms_per_generation": e2e_ms, "kernels_per_generation": 5,
                      "gpu_persistent_ms_per_generation": ms_persist,
                      "gpu_persistent_generations_per_s": 1e3 / ms_persist,
                      "persistent_how": "de_runs (K8): init + 2000 generations of the run in one launch",
                      "cpu_reference_ms_per_generation": cpu_s / 2000 * 1e3, "cpu_cores": 1,
                      "cpu_sample": "build_de_fixed(0.5,0.9), 2000 generations, native stream"}


def cfg2(out):
    P, D, G = 180, 100, 1000
    o, m = O.shift_rotation(11, D)
    prob = evb.ProblemInstance.base(evb.BaseKind.ackley, o, m, 0.0)
    eng = DEEngine(preset_shade(0.11, P, 1.0), P, D)
    rng = Rng.philox(11)
    pop = torch.empty((P, D), dtype=torch.float64, device=DEV)
    fit = torch.empty(P, dtype=torch.float64, device=DEV)

    def run():
        eng.reset()
        eng.init_population(pop, -100.0, 100.0, rng)
        evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
        eng.generations(prob, pop, fit, -100.0, 100.0, rng, G)

    run()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    cpu_s = O.REF_FAST().ref_bench_de(1, P, D, 200, 6, O.ptr(o), O.ptr(np.ascontiguousarray(m)), 11)
    out["config2"] = {"gpu_ms_1000_generations": ms, "gpu_generations_per_s": G / (ms * 1e-3),
                      "best_fitness": float(fit.min()),
                      "cpu_reference_generations_per_s": 200 / cpu_s, "cpu_cores": 1,
                      "cpu_sample": "build_shade(0.11, 180, 1.0), 200 generations, native stream"}


def cfg3(out):
    P, D, G = 1024, 1000, 500
    res = {}
    o, m = O.shift_rotation(13, D)
    for nd, dt, tdt in ((np.float64, evb.EVB_F64, torch.float64), (np.float32, evb.EVB_F32, torch.float32)):
        prob = evb.ProblemInstance.base(evb.BaseKind.elliptic, o.astype(nd), m.astype(nd), 0.0, dtype=dt)
        for topo in ("gbest", "lbest_ring"):
            eng = PSOEngine(config3(topo), P, D, dt)
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
            res[f"{np.dtype(nd).name}_{topo}"] = {"gpu_ms_500_iterations": ms, "gpu_iterations_per_s": G / (ms * 1e-3),
                                                  "best_pbest": float(eng.personal_bests()["pbest_fit"].min())}
    # CPU: the synchronous driver over the reference pieces, evaluation split over all host threads
    xs = O.population(13, P, D)
    vs = np.random.default_rng(0).uniform(-20, 20, (P, D))
    f0 = O.eval_batch(1, o, m, 0.0, xs)
    ref = O.RefPSO(np.float64, 0, 0.7298, 1.49618, 1.49618, 40.0, P, D, 1, o, m)
    O.REF_FAST()  # ensure loaded
    ref.set(xs, vs, f0)
    O.REF().ref_pso_set_threads(1, ref.h, threads())
    words = np.random.default_rng(1).integers(0, 2**63, size=2 * P * D, dtype=np.uint64)
    t0 = time.perf_counter()
    ref.step(words, -100.0, 100.0)
    cpu_s = time.perf_counter() - t0
    res["cpu_reference_iterations_per_s"] = 1.0 / cpu_s
    res["cpu_cores"] = threads()
    res["cpu_sample"] = "1 synchronous gbest iteration, fp64, reference pieces, evaluation over all threads (exact build)"
    out["config3"] = res


def cfg4(out):
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
    t0 = time.perf_counter()
    de_runs(preset_de(), probs, keys, pops, fits, G, -100.0, 100.0)  # synchronous call, wall clock
    gpu_s = time.perf_counter() - t0
    sh = np.ascontiguousarray(np.stack(shifts))
    ro = np.ascontiguousarray(np.stack(rots))
    k = np.array(O.CONFIG4_KINDS, np.int32)
    sg, la, cb = (np.array(v) for v in (O.CONFIG4_SIGMA, O.CONFIG4_LAMBDA, O.CONFIG4_BIAS))
    sample_runs = 16
    cpu_s = O.REF_FAST().ref_bench_config4(sample_runs, P, D, G, threads(), O.ptr(sh), O.ptr(ro), O.ptr(k), O.ptr(sg),
                                           O.ptr(la), O.ptr(cb))
    out["config4"] = {"gpu_s_64_runs_x_2000_generations": gpu_s, "gpu_run_generations_per_s": n_runs * G / gpu_s,
                      "gpu_launches": 1, "best_fitness_run0": float(fits[0].min()),
                      "cpu_reference_run_generations_per_s": sample_runs * G / cpu_s, "cpu_cores": threads(),
                      "cpu_sample": f"evo_bench + `de` preset over {sample_runs} of the 64 runs, {threads()} threads"}


def hbm(out):
    P, D = 16384, 1000
    res = {}
    o, m = O.shift_rotation(13, D)
    # DE trial + selection (rand/1, Philox): compulsory bytes of the update kernels
    prob = evb.ProblemInstance.base(evb.BaseKind.sphere, o, m, 0.0)
    eng = DEEngine(preset_de(), P, D)
    rng = Rng.philox(5)
    pop = torch.empty((P, D), dtype=torch.float64, device=DEV)
    eng.init_population(pop, -100.0, 100.0, rng)
    fit = torch.empty(P, dtype=torch.float64, device=DEV)
    evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
    eng.generation(prob, pop, fit, -100.0, 100.0, rng)
    torch.cuda.synchronize()
    res["note"] = "per-kernel durations and DRAM bytes of the update kernels come from the ncu launch list " \
                  "(profiles/); here whole-generation time"
    ms = timed(lambda: eng.generation(prob, pop, fit, -100.0, 100.0, rng), 5, warm=1)
    res["de_generation_ms"] = ms
    # PSO update alone: time generation minus evaluation by timing evaluation separately
    eng2 = PSOEngine(config3("gbest"), P, D)
    X = torch.empty((P, D), dtype=torch.float64, device=DEV)
    V = torch.empty((P, D), dtype=torch.float64, device=DEV)
    f2 = torch.empty(P, dtype=torch.float64, device=DEV)
    eng2.init_uniform(X, -100.0, 100.0, rng)
    eng2.init_uniform(V, -20.0, 20.0, rng)
    sc = evb.EvalScratch()
    evb.evaluate_batch(prob, X, sc, f2)
    eng2.prepare(X, f2)
    gen_ms = timed(lambda: eng2.generation(prob, X, V, f2, -100.0, 100.0, rng), 5, warm=1)
    eval_ms = timed(lambda: evb.evaluate_batch(prob, X, sc, f2), 5, warm=1)
    upd_ms = gen_ms - eval_ms
    bytes_upd = 5 * 8 * P * D
    res["pso_generation_ms"] = gen_ms
    res["pso_eval_ms"] = eval_ms
    res["pso_update_ms_est"] = upd_ms
    res["pso_update_GBps_est"] = bytes_upd / (upd_ms * 1e-3) / 1e9
    res["pso_update_frac_hbm_est"] = res["pso_update_GBps_est"] / HBM_PEAK
    out["hbm_sweep_P16384_D1000"] = res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=None)
    args = ap.parse_args()
    out = {"device": torch.cuda.get_device_name(0), "host_threads": threads(),
           "cpu_baseline_lib": O.REF_FAST()._evb_name}
    for name, fn in (("config1", cfg1), ("config0", cfg0), ("config2", cfg2), ("config3", cfg3), ("config4", cfg4),
                     ("hbm", hbm)):
        if args.only and name not in args.only:
            continue
        t0 = time.perf_counter()
        fn(out)
        out.setdefault("wall_s", {})[name] = time.perf_counter() - t0
    print(json.dumps(out, indent=1), flush=True)


if __name__ == "__main__":
    main()
