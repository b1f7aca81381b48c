python tools/k2sk_timeline.py rastrigin > gpurun_out/k2tl.log 2>&1; python tools/k2sk_timeline.py elliptic >> gpurun_out/k2tl.log 2>&1
timeout 900 python -m pytest tests/test_eval_gpu.py -x -q > gpurun_out/eval_tests.log 2>&1; echo RC=$? >> gpurun_out/eval_tests.log
for v in "0 2" "0 1"; do set -- $v; env $( [ $1 != 0 ] && echo EVB_UMMA_BN=$1) EVB_UMMA_SPLITK=$2 python bench_configs.py --only config1_fp32 > gpurun_out/k2_$1_$2.json 2>&1; done
