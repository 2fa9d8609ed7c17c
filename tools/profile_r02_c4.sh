set -u
O=gpurun_out
M="gpu__time_duration.sum"
T="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
python bench.py --steps 2 --warmup 3 --no-cpu > $O/p_c4_plain.log 2>&1 &&
ncu --metrics $M --clock-control none --csv --log-file $O/r02_c4_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > $O/p_c4_ncu.log 2>&1
ncu --metrics $T --clock-control none -k regex:'lu_compact|ilutp_pipeline|steady_solver|spmv_warp|lu_solve_kernel|frontal_lu' \
    -c 24 -o $O/r02_c4_traffic python bench.py --steps 1 --warmup 3 --no-cpu > $O/p_c4_traffic.log 2>&1
ls -la $O | tail -5
