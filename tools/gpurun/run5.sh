mkdir -p gpurun_out
for w in none G F both; do
GENINV_DEBUG_GEMM=1 CUDA_LAUNCH_BLOCKING=1 timeout 120 python tools/gpurun/dbg_solve2.py $w > gpurun_out/dbg5_$w.log 2>&1
done
