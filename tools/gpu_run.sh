# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
T0=$(date +%s); timeout 900 python bench.py > gpurun_out/r53_bench.json 2> gpurun_out/r53_bench.err
echo "elapsed $(( $(date +%s) - T0 )) s"
python -c "
import json; d=json.loads(open('gpurun_out/r53_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['compute_only']['value'], d['roofline']['frac'], d['clocks'])
print(d['cfg2'].get('cpu_oracle')); print(d['cfg3'].get('cpu_oracle')); print(d.get('cpu_oracle_error'))"
