timeout 900 python -m pytest tests/test_gpu_stack.py tests/test_gpu_probe.py tests/test_gpu_track.py tests/test_gpu_sample.py -m gpu -q > gpurun_out/r24_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r24_t.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r24_bench.json 2> gpurun_out/r24_bench.err
tail -15 gpurun_out/r24_t.log; python -c "
import json; d=json.loads(open('gpurun_out/r24_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['compute_only'], d['cfg2'])"
