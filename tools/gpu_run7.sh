mkdir -p gpurun_out
LOKA_PAIRNORM=256 timeout 300 python tools/trace_pairnorm.py > gpurun_out/r7_trace256.json 2>&1
LOKA_PAIRNORM=512 timeout 300 python tools/trace_pairnorm.py > gpurun_out/r7_trace512.json 2>&1
cat gpurun_out/r7_trace256.json gpurun_out/r7_trace512.json
