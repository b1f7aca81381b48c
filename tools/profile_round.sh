#!/bin/bash
# Run on the GPU box (gpurun): plain bench first, then the ncu passes the profiling recipe asks for.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/bench_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench_launches.log 2>&1
python tools/prof_eval.py f64 5 4 > $OUT/eval_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:eval_f64 -s 2 -c 1 -o $OUT/eval_f64 \
    python tools/prof_eval.py f64 5 4 > $OUT/eval_ncu.log 2>&1
python tools/time_multi.py > $OUT/multi_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:eval_f64_dmma_multi -s 2 -c 1 -o $OUT/eval_multi \
    python tools/time_multi.py > $OUT/multi_ncu.log 2>&1
python tools/prof_eval.py f32 5 4 > $OUT/eval32_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:eval_f32 -s 2 -c 1 -o $OUT/eval_f32 \
    python tools/prof_eval.py f32 5 4 > $OUT/eval32_ncu.log 2>&1
python bench_configs.py --only hbm > $OUT/hbm_plain.json 2>&1 &&
ncu --set full --clock-control none -k regex:"de_trial|de_select" -s 3 -c 3 -o $OUT/updates \
    python bench_configs.py --only hbm > $OUT/updates_ncu.log 2>&1
ncu --set full --clock-control none -k regex:pso_update -s 1 -c 1 -o $OUT/pso_update \
    python bench_configs.py --only hbm > $OUT/pso_ncu.log 2>&1
python tools/prof_runs.py 50 > $OUT/runs_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:de_runs -s 1 -c 1 -o $OUT/runs \
    python tools/prof_runs.py 50 > $OUT/runs_ncu.log 2>&1
ls -la $OUT
