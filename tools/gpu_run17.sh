timeout 600 python -m pytest tests/test_gpu_pairnorm.py -m gpu -x -q > gpurun_out/r17_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r17_t.log
timeout 300 python tools/seq_pairnorm.py --n 20 --gap_ms 2 > gpurun_out/r17_seq.json 2>&1
LOKA_PAIRNORM=256 timeout 300 python tools/trace_pairnorm.py --M 32768 --out gpurun_out/r17_tr.npy > gpurun_out/r17_trace.json 2>&1
tail -3 gpurun_out/r17_t.log
python -c "
import json,statistics; d=json.load(open('gpurun_out/r17_seq.json')); print(d['clocks']); print({k:round(statistics.median(v[1:]),4) for k,v in d['ms'].items()})"
python -c "
import json; d=json.load(open('gpurun_out/r17_trace.json')); print({k:(round(v['mean'],2) if isinstance(v,dict) and 'mean' in v else v) for k,v in d.items() if k not in ('mma_stall_by_wave_mean','stalled_pairs_gt2us_by_wave')})"
