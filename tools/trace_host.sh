#!/bin/bash
# timeline of evb_evaluate_batch_host for a few chunkings (tuning aid)
for cfg in "1 uniform" "2 uniform" "4 uniform" "4 geo" "8 geo"; do
  set -- $cfg
  echo "== chunks $1 $2"
  EVB_H2D_TRACE=1 EVB_H2D_CHUNKS=$1 EVB_H2D_SPLIT=$2 python tools/time_host.py 2>&1 | grep "evb h2d" | tail -3
  EVB_H2D_CHUNKS=$1 EVB_H2D_SPLIT=$2 python tools/time_host.py
done
