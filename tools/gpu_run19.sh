timeout 600 python -m pytest tests/test_gpu_quantize.py -m gpu -x -q -k "tensor" > gpurun_out/r19_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r19_t.log
timeout 300 python tools/bench_quantize.py --out gpurun_out/r19_q.json > /dev/null 2> gpurun_out/r19_q.err
timeout 300 python tools/bench_quantize.py --rows 262144 --cols 4096 --steps 10 --out gpurun_out/r19_q262k.json > /dev/null 2>> gpurun_out/r19_q.err
tail -2 gpurun_out/r19_t.log; tail -3 gpurun_out/r19_q.err; python -c "
import json
for f in ['gpurun_out/r19_q.json','gpurun_out/r19_q262k.json']:
    d=json.load(open(f)); print(f, d['clocks']); print({k:(v['ms'],v['gbs']) for k,v in d['kernels'].items()})"
