mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pairnorm.py tests/test_gpu_grouped.py tests/test_gpu_backward.py -m gpu -x -q > gpurun_out/r4_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r4_t.log
timeout 600 python tools/bench_pairnorm.py --out gpurun_out/r4_pnbench.json > gpurun_out/r4_pnbench.log 2>&1
timeout 300 python tools/bench_cfg4.py > gpurun_out/r4_cfg4.log 2>&1
tail -5 gpurun_out/r4_t.log; cat gpurun_out/r4_pnbench.log | tail -5; tail -5 gpurun_out/r4_cfg4.log
