mkdir -p gpurun_out
for v in 0 1e300 nan; do timeout 120 python tools/gpurun/dbg_solve3.py $v >> gpurun_out/dbg8.log 2>&1; done
