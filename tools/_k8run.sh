mkdir -p gpurun_out/k8
(time python -m pytest tests/test_runs_gpu.py tests/test_evo_bench_gpu.py -m gpu -x -q -s) > gpurun_out/k8/tests.log 2>&1; echo RC=$? >> gpurun_out/k8/tests.log
EVB_RUNS_PROFILE=1 python tools/prof_runs.py 200 > gpurun_out/k8/prof_fused.log 2>&1
EVB_RUNS_FUSED=0 EVB_RUNS_PROFILE=1 python tools/prof_runs.py 200 > gpurun_out/k8/prof_old.log 2>&1
python bench_configs.py --only config4 > gpurun_out/k8/cfg4_fused.json 2>&1
EVB_RUNS_FUSED=0 python bench_configs.py --only config4 > gpurun_out/k8/cfg4_old.json 2>&1
tail -3 gpurun_out/k8/tests.log; cat gpurun_out/k8/prof_*.log | grep cycles; grep -o '"value": [0-9.]*, "unit": "run-generations/s"' gpurun_out/k8/cfg4_*.json
