timeout 600 python -m pytest tests/test_gpu_quantize.py -m gpu -q -x -k "1x128 or dual or 128x128" > gpurun_out/r28_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r28_t.log
timeout 300 python tools/bench_quantize.py --rows 262144 --cols 4096 --steps 10 --out gpurun_out/r28_q262k.json > /dev/null 2> gpurun_out/r28_q.err
tail -2 gpurun_out/r28_t.log; python -c "
import json
d=json.load(open('gpurun_out/r28_q262k.json')); print(d['clocks']); print({k:(v['ms'],v['gbs']) for k,v in d['kernels'].items()})"
