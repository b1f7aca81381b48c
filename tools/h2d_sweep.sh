# e2e host path (three problems on one pinned population) under several copy plans (tuning aid)
set -u
run() {  # label, env...
  echo "== $*" >> gpurun_out/h2d_sweep.log
  env "$@" EVB_H2D_TRACE=1 python tools/time_host_many.py 30 2>&1 | grep "evb h2d" | tail -1 >> gpurun_out/h2d_sweep.log
  env "$@" python tools/time_host_many.py >> gpurun_out/h2d_sweep.log 2>&1
}
run EVB_H2D_ROWS=floor
run EVB_H2D_ROWS=ceil
run EVB_H2D_ROWS=floor EVB_H2D_CHUNKS=3
run EVB_H2D_ROWS=floor EVB_H2D_WIDTHS=160,288,288
run EVB_H2D_ROWS=floor EVB_H2D_CHUNKS=5
run EVB_H2D_ROWSPLIT=0
