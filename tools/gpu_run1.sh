mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_quantize.py -m gpu -x -q > gpurun_out/r1_tq.log 2>&1; echo "EXIT $?" >> gpurun_out/r1_tq.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r1_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r1_t.log
timeout 300 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
timeout 300 python tools/bench_cfg5.py --out gpurun_out/r1_cfg5.json > gpurun_out/r1_cfg5.log 2>&1
tail -3 gpurun_out/r1_tq.log gpurun_out/r1_t.log; cat gpurun_out/r1_bench.json; tail -5 gpurun_out/r1_cfg5.log
