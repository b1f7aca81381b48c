#!/bin/bash
# config 2 persistent generations: parity tests, phase cycles, generations/s
python -m pytest tests/test_de_gpu.py -m gpu -x -q -k "persistent or config2 or shade or jade" 2>&1 | tail -4
EVB_DE_PERSIST_PROFILE=1 python tools/prof_cfg2_persist.py 200 2>&1 | tail -2
python bench_configs.py --only config2 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
def find(d):
    if isinstance(d,dict):
        if 'ms_1000_generations' in d: print('config2', d['value'], 'generations/s', d['ms_1000_generations'], 'ms')
        for v in d.values(): find(v)
find(d)"
