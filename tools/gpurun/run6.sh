mkdir -p gpurun_out
GENINV_DEBUG_SYNC=1 GENINV_DEBUG_GEMM=1 timeout 120 python tools/gpurun/dbg_solve1.py s > gpurun_out/dbg6_s.log 2>&1
GENINV_NO_GRAPH=1 GENINV_DEBUG_SYNC=1 timeout 120 python tools/gpurun/dbg_solve1.py s > gpurun_out/dbg6_s_nograph.log 2>&1
