# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_probe.py -m gpu -q -x > gpurun_out/r92_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r92_t.log
grep -v "^\[W" gpurun_out/r92_t.log | tail -2
timeout 600 python tools/bench_probe.py --out gpurun_out/r92_probe.json > /dev/null 2> gpurun_out/r92_p.err
python -c "
import json
d=json.load(open('gpurun_out/r92_probe.json')); print([(c['case'][:20], c['ms'], c['gbs']) for c in d['cases']], d['clocks'].get('sm_mhz'))"
