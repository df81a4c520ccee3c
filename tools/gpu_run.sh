# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python tools/bench_sample.py --out gpurun_out/r70_sample.json > gpurun_out/r70.log 2>&1
tail -3 gpurun_out/r70.log
python -c "
import json; d=json.load(open('gpurun_out/r70_sample.json'))
for r in d['rows']: print({k: v for k, v in r.items()})"
