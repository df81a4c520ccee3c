mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pairnorm.py -m gpu -x -q > gpurun_out/r14_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r14_t.log
LOKA_PAIRNORM=256 timeout 300 python tools/trace_pairnorm.py --M 32768 --out gpurun_out/r14_tr.npy > gpurun_out/r14_trace.json 2>&1
timeout 600 python tools/ab_pairnorm.py --rounds 7 --reps 4 --variants "PN=256" "PN=256,ORDER=0" "PN=512" "NORM=none,WIDE=0" "NORM=none,WIDE=1" > gpurun_out/r14_ab.json 2> gpurun_out/r14_ab.err
timeout 600 python tools/ab_pairnorm.py --M 262144 --rounds 3 --reps 2 --variants "PN=256" "PN=512" "NORM=none,WIDE=1" > gpurun_out/r14_ab_p1.json 2>> gpurun_out/r14_ab.err
tail -2 gpurun_out/r14_t.log; python -c "
import json; d=json.load(open('gpurun_out/r14_trace.json')); print({k:(round(v['mean'],2) if isinstance(v,dict) and 'mean' in v else v) for k,v in d.items() if k not in ('mma_stall_by_wave_mean','stalled_pairs_gt2us_by_wave')})"
cat gpurun_out/r14_ab.json gpurun_out/r14_ab_p1.json
