mkdir -p gpurun_out
for t in cfg3 cfg4 stretch next1 next1_bwd probe nvfp4 track; do
  timeout 900 python tools/bench_$t.py --out gpurun_out/r31_$t.json > gpurun_out/r31_$t.log 2>&1; echo "EXIT $?" >> gpurun_out/r31_$t.log
done
for t in cfg3 cfg4 stretch next1 next1_bwd probe nvfp4 track; do echo "== $t"; tail -2 gpurun_out/r31_$t.log | cut -c1-600; done
timeout 600 python -m pytest tests/test_gpu_quantize.py -m gpu -q -x -k "delayed or tensor" > gpurun_out/r31_tq.log 2>&1; echo "EXIT $?" >> gpurun_out/r31_tq.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r31_bench.json 2> gpurun_out/r31_bench.err
tail -2 gpurun_out/r31_tq.log; python -c "
import json; d=json.loads(open('gpurun_out/r31_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['compute_only']['value'], d['delayed_scaling'], d['bf16_library_fused']['value'], d['clocks'])"
