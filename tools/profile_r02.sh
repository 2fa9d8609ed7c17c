#!/bin/bash
# Round-2 profiling pass (run under gpurun; outputs in gpurun_out/).  ncu runs
# only after the same command exited 0 without it.
set -u
O=gpurun_out
M="gpu__time_duration.sum"
T="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
# 1. c4: launch list of the default bench command
python bench.py --steps 2 --warmup 3 --no-cpu > $O/p_c4_plain.log 2>&1 &&
ncu --metrics $M --clock-control none --csv --log-file $O/r02_c4_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/p_c4_ncu.log 2>&1
# 2. c4: DRAM traffic of the hot kernels (factorization, solver, SpMV, apply)
ncu --metrics $T --clock-control none -k regex:'lu_compact|ilutp_pipeline|steady_solver|spmv_warp|lu_solve_kernel|frontal_lu' \
    -c 24 -o $O/r02_c4_traffic python bench.py --steps 1 --warmup 3 --no-cpu > $O/p_c4_traffic.log 2>&1
# 3. c5: launch list (one step) and traffic of SpMV / apply / solver
python bench.py --config c5 --steps 1 --warmup 3 --no-cpu > $O/p_c5_plain.log 2>&1 &&
ncu --metrics $M --clock-control none --csv --log-file $O/r02_c5_launches.csv \
    python bench.py --config c5 --steps 1 --warmup 3 --no-cpu > $O/p_c5_ncu.log 2>&1
python tools/c5_apply.py 40 40 1e-2 2 > $O/p_c5a_plain.log 2>&1 &&
ncu --metrics $T --clock-control none -k regex:'spmv_warp|grid_apply' -c 8 -o $O/r02_c5_traffic \
    python tools/c5_apply.py 40 40 1e-2 2 > $O/p_c5_traffic.log 2>&1
ls -la $O | tail -20
