# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r90_gpu_tests.txt 2>&1; echo "EXIT $?" >> gpurun_out/r90_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r90_smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r90_bench.json 2> gpurun_out/r90_bench.err
grep -v "^\[W" gpurun_out/r90_gpu_tests.txt | tail -2; tail -1 gpurun_out/r90_smoke.txt
python -c "
import json; d=json.loads(open('gpurun_out/r90_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['compute_only']['value'], d['roofline']['frac'], d['roofline']['peak'], d['clocks'], d['speedup_vs_bf16'], d['cfg2']['value'], d['cfg3']['value'], d['e2e']['value'])"
