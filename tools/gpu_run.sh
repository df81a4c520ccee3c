# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r80_gpu_tests.txt 2>&1; echo "EXIT $?" >> gpurun_out/r80_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r80_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r80_bench.json 2> gpurun_out/r80_bench.err
timeout 900 python tools/bench_cfg4.py --out gpurun_out/r80_cfg4.json > /dev/null 2> gpurun_out/r80_cfg4.err
grep -v "^\[W" gpurun_out/r80_gpu_tests.txt | tail -2; tail -1 gpurun_out/r80_smoke.txt
python -c "
import json; d=json.loads(open('gpurun_out/r80_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['compute_only']['value'], d['roofline']['frac'], d['clocks'], d['speedup_vs_bf16'], d['cfg2']['value'], d['cfg3']['value'], d['e2e']['value'])
c=json.load(open('gpurun_out/r80_cfg4.json')); print('cfg4', c['tensorwise']['speedup_vs_bf16_end_to_end'], c['blockwise_ue8m0']['speedup_vs_bf16_end_to_end'], c['clocks'])"
