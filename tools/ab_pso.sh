#!/bin/bash
# A/B of the PSO generation boundary (EVB_PSO_FUSE_NB=0: separate personal-best and neighbourhood kernels)
python -m pytest tests/test_pso_gpu.py tests/test_evo_bench_gpu.py -m gpu -x -q 2>&1 | tail -2
for f in 0 1; do echo "== EVB_PSO_FUSE_NB=$f"; EVB_PSO_FUSE_NB=$f python bench_configs.py --only config3 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
def find(d):
    if isinstance(d,dict):
        if 'variants' in d:
            for k,v in d['variants'].items(): print('  ',k, round(v['value']), 'iterations/s')
        for v in d.values(): find(v)
find(d)"; done
