# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grouped.py -m gpu -q -x > gpurun_out/r66_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r66_t.log
grep -v "^\[W" gpurun_out/r66_t.log | tail -3
