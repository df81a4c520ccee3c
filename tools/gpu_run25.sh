timeout 900 python -m pytest tests/test_gpu_pairnorm.py -m gpu -q -x > gpurun_out/r25_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r25_t.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/r25_bench.json 2> gpurun_out/r25_bench.err
tail -3 gpurun_out/r25_t.log; tail -3 gpurun_out/r25_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r25_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['compute_only']['value'], d['bf16_baseline'], d['bf16_library_fused'], d['clocks'])"
