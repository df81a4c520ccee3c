# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python tools/bench_next1_bwd.py > gpurun_out/r89_bwd.json 2> gpurun_out/r89_bwd.err
tail -2 gpurun_out/r89_bwd.err
python -c "
import json; d=json.loads(open('gpurun_out/r89_bwd.json').read().strip().splitlines()[-1])
for c in d['cases']: print({k: v for k, v in c.items() if not k.startswith('path')})
print(d['clocks'])"
