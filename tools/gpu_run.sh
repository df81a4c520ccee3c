# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quantize.py -m gpu -q -x > gpurun_out/r52_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r52_t.log
timeout 300 python tools/bench_quantize.py --rows 262144 --cols 4096 --out gpurun_out/r52_q262k.json > /dev/null 2> gpurun_out/r52_q.err
tail -2 gpurun_out/r52_t.log
python -c "
import json; d=json.load(open('gpurun_out/r52_q262k.json')); print({k: v['gbs'] for k, v in d['kernels'].items()}, d['clocks'])"
