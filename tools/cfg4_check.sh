#!/bin/bash
# config 4 (K8 fused generation): phase cycles, parity tests, run-generations/s
EVB_RUNS_PROFILE=1 timeout 120 python tools/prof_runs.py 200 2>&1 | tail -2
timeout 900 python -m pytest tests/test_runs_gpu.py tests/test_evo_bench_gpu.py tests/test_recorder_gpu.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench_configs.py --only config4 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
def find(d):
    if isinstance(d,dict):
        if 'ms_total' in d: print('config4', round(d['value']), 'run-generations/s', round(d['ms_total'],2), 'ms')
        for v in d.values(): find(v)
find(d)"
