mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pairnorm.py -m gpu -x -q > gpurun_out/r2_pn.log 2>&1; echo "EXIT $?" >> gpurun_out/r2_pn.log
timeout 300 python tools/bench_pairnorm.py --quick --out gpurun_out/r2_pnbench.json > gpurun_out/r2_pnbench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_linear.py -m gpu -q > gpurun_out/r2_bl.log 2>&1; echo "EXIT $?" >> gpurun_out/r2_bl.log
tail -15 gpurun_out/r2_pn.log; cat gpurun_out/r2_pnbench.log | tail -5; tail -15 gpurun_out/r2_bl.log
