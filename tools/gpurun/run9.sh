mkdir -p gpurun_out
for sl in 0 4096 65536 4194304; do echo "slack $sl" >> gpurun_out/dbg9.log; GENINV_STAGE_SLACK=$sl timeout 120 python tools/gpurun/dbg_solve1.py s >> gpurun_out/dbg9.log 2>&1; done
timeout 300 compute-sanitizer --tool memcheck python tools/gpurun/dbg_solve1.py s > gpurun_out/dbg9_san.log 2>&1
