#!/bin/bash
# Run on the GPU box (gpurun): plain bench first, then the ncu passes the profiling recipe asks for
# (each capture only after its own command ran clean without ncu).  Summarise here afterwards with
# python tools/summarize_profiles.py rNN.
# usage: profile_round.sh [a|b|all]   (two halves: the merged gpurun_out/ of one call is capped at 64 MiB)
set -u
PART=${1:-all}
OUT=gpurun_out/prof
mkdir -p $OUT
if [ "$PART" != "b" ]; then
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs > $OUT/bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs > $OUT/bench_launches.log 2>&1
# headline: the multi-problem fused DMMA evaluation (config 1, three objectives)
python tools/time_multi.py > $OUT/multi_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:eval_f64_dmma_multi -s 2 -c 1 -o $OUT/eval_multi \
    python tools/time_multi.py > $OUT/multi_ncu.log 2>&1
# fp32 config 1: split-K tcgen05 kernel
python tools/prof_eval.py f32 5 4 > $OUT/eval32_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:eval_f32_umma_sk -s 2 -c 1 -o $OUT/eval_f32 \
    python tools/prof_eval.py f32 5 4 > $OUT/eval32_ncu.log 2>&1
fi
if [ "$PART" != "a" ]; then
# HBM update kernels at P=16384, D=1000 (L2-exceeding)
python bench_configs.py --only hbm_update > $OUT/hbm_plain.json 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"de_trial|de_select_multi|de_select_apply" -s 3 -c 3 \
    -o $OUT/updates python bench_configs.py --only hbm_update > $OUT/updates_ncu.log 2>&1
ncu --set full --clock-control none -k regex:pso_update -s 1 -c 1 -o $OUT/pso_update \
    python bench_configs.py --only hbm_update > $OUT/pso_ncu.log 2>&1
# config 4: K8 persistent runs (DMMA composition contractions)
python tools/prof_runs.py 50 > $OUT/runs_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:de_runs -s 1 -c 1 -o $OUT/runs \
    python tools/prof_runs.py 50 > $OUT/runs_ncu.log 2>&1
# config 2: persistent engine generations (cluster kernel)
python tools/prof_cfg2_persist.py 50 > $OUT/de_run_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:de_run_kernel -s 1 -c 1 -o $OUT/de_run \
    python tools/prof_cfg2_persist.py 50 > $OUT/de_run_ncu.log 2>&1
fi
ls -la $OUT
