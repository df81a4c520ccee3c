mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r18_bench.json 2> gpurun_out/r18_bench.err; echo "EXIT $?" >> gpurun_out/r18_bench.err
tail -5 gpurun_out/r18_bench.err; cat gpurun_out/r18_bench.json
