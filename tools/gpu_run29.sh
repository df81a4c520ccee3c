timeout 900 python -m pytest tests/test_gpu_pairnorm.py tests/test_gpu_norm_bwd.py -m gpu -q -x > gpurun_out/r30_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r30_t.log
timeout 600 python tools/bench_next1_bwd.py --out gpurun_out/r30_bwd.json > gpurun_out/r30_bwd.log 2>&1
timeout 600 python tools/seq_pairnorm.py --n 20 --gap_ms 2 > gpurun_out/r30_seq.json 2>&1
tail -5 gpurun_out/r30_t.log; tail -3 gpurun_out/r30_bwd.log; python -c "
import json,statistics; d=json.load(open('gpurun_out/r30_seq.json')); print({k:round(statistics.median(v[1:]),4) for k,v in d['ms'].items()})"
