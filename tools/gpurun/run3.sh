mkdir -p gpurun_out
for c in "1000 333 260 5" "1000 334 260 5" "1000 333 260 6" "1000 333 260 1" "1000 320 260 5" "640 333 260 5" "1000 128 100 5" "1000 129 100 5" "1000 200 100 5" "300 130 70 1" "700 300 250 5"; do
  CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/gpurun/dbg_solve.py $c >> gpurun_out/dbg_solve3.log 2>&1
  GENINV_NO_GRAPH=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/gpurun/dbg_solve.py $c >> gpurun_out/dbg_solve3.log 2>&1
done
