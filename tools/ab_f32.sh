#!/bin/bash
# A/B of the fp32 tensor-core split (EVB_F32_MMA=tf32|f16): error and device time at config 1
for m in tf32 f16; do
  echo "== EVB_F32_MMA=$m"
  EVB_F32_MMA=$m timeout 300 python tools/time_f32.py 2>&1 | tail -7
done
