mkdir -p gpurun_out/k8
(time python -m pytest tests/test_runs_gpu.py tests/test_evo_bench_gpu.py -m gpu -x -q -s) > gpurun_out/k8/tests.log 2>&1; echo RC=$? >> gpurun_out/k8/tests.log
EVB_RUNS_PROFILE=1 python tools/prof_runs.py 200 > gpurun_out/k8/prof_fused.log 2>&1
python bench_configs.py --only config4 > gpurun_out/k8/cfg4_fused.json 2>&1
tail -3 gpurun_out/k8/tests.log; grep "lockstep" gpurun_out/k8/tests.log; cat gpurun_out/k8/prof_*.log | grep cycles; grep '"value"\|ms_total' gpurun_out/k8/cfg4_fused.json | head -2
python tools/prof_runs.py 50 > gpurun_out/k8/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:de_runs -s 1 -c 1 -o gpurun_out/k8/runs_fused python tools/prof_runs.py 50 > gpurun_out/k8/ncu.log 2>&1
