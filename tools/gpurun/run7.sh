mkdir -p gpurun_out
GENINV_DEBUG_SYNC=1 timeout 120 python tools/gpurun/dbg_solve1.py s > gpurun_out/dbg7_s.log 2>&1
GENINV_DEBUG_SYNC=1 timeout 120 python tools/gpurun/dbg_solve2.py none > gpurun_out/dbg7_none.log 2>&1
