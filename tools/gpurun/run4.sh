mkdir -p gpurun_out
for mode in s d; do
GENINV_DEBUG_GEMM=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/gpurun/dbg_solve1.py $mode > gpurun_out/dbg4_$mode.log 2>&1
done
