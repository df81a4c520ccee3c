timeout 900 python -m pytest tests/test_gpu_pairnorm.py tests/test_gpu_linear.py -m gpu -q -x > gpurun_out/r37_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r37_t.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/r37_bench.json 2> gpurun_out/r37_bench.err
tail -4 gpurun_out/r37_t.log; tail -3 gpurun_out/r37_bench.err; python -c "
import json; d=json.loads(open('gpurun_out/r37_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['compute_only']['value'], d['fused_call'], d['unfused_cast_step'], d['fp8_step_interleaved_ms'], d['speedup_vs_bf16'], d['clocks'])"
