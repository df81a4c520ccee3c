mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pairnorm.py -m gpu -x -q > gpurun_out/r3_pn.log 2>&1; echo "EXIT $?" >> gpurun_out/r3_pn.log
timeout 600 python tools/bench_pairnorm.py --out gpurun_out/r3_pnbench.json > gpurun_out/r3_pnbench.log 2>&1
tail -15 gpurun_out/r3_pn.log; cat gpurun_out/r3_pnbench.log | tail -5
