mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pairnorm.py -m gpu -x -q > gpurun_out/r8_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r8_t.log
LOKA_PAIRNORM=256 timeout 300 python tools/trace_pairnorm.py > gpurun_out/r8_trace256.json 2>&1
timeout 600 python tools/ab_pairnorm.py --variants "PN=256" "PN=256,DBG=1" "NORM=none,WIDE=0" "NORM=none,WIDE=1" > gpurun_out/r8_ab.json 2> gpurun_out/r8_ab.err
tail -3 gpurun_out/r8_t.log; head -40 gpurun_out/r8_trace256.json; cat gpurun_out/r8_ab.json
