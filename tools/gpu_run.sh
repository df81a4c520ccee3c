# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sample.py tests/test_gpu_track.py -m gpu -q -x > gpurun_out/r71_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r71_t.log
grep -v "^\[W" gpurun_out/r71_t.log | tail -2
timeout 900 python tools/bench_sample.py --out gpurun_out/r71_sample.json > gpurun_out/r71.log 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r71_sample.json'))
for r in d['rows']:
    if 'cholesky' in r['op'] or 'weight' in r['op']: print(r['op'][:20], r.get('n', r.get('M')), r['ms'], r['torch_ms'], r['speedup_vs_torch'])"
