# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_probe.py -m gpu -q -x > gpurun_out/r85_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r85_t.log
grep -v "^\[W" gpurun_out/r85_t.log | tail -3
timeout 600 python tools/bench_probe.py --out gpurun_out/r85_probe.json > /dev/null 2> gpurun_out/r85_p.err
LOKA_PROBE_TWO_PASS=1 timeout 600 python tools/bench_probe.py --out gpurun_out/r85_probe_2p.json > /dev/null 2>> gpurun_out/r85_p.err
python -c "
import json
for f in ('r85_probe','r85_probe_2p'):
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, [(c['case'][:20], c['ms'], c['gbs']) for c in d['cases']], d['clocks'].get('sm_mhz'))"
