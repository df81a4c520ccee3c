timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r32_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r32_t.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r32_bench.json 2> gpurun_out/r32_bench.err
timeout 300 python tools/bench_quantize.py --rows 262144 --cols 4096 --steps 10 --out gpurun_out/r32_q262k.json > /dev/null 2> gpurun_out/r32_q.err
tail -5 gpurun_out/r32_t.log; python -c "
import json; d=json.loads(open('gpurun_out/r32_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['compute_only'], d['speedup_vs_bf16'], d['fp8_step_interleaved_ms'], d['bf16_baseline']['ms_per_step'], d['delayed_scaling'], d['bf16_library_fused'], d['clocks'], d['roofline'])
d=json.load(open('gpurun_out/r32_q262k.json')); print({k:(v['ms'],v['gbs']) for k,v in d['kernels'].items()})"
