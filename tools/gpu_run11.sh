mkdir -p gpurun_out
for M in 256 2560 32768; do LOKA_PAIRNORM=256 timeout 300 python tools/trace_pairnorm.py --M $M --out gpurun_out/r11_tr_$M.npy > gpurun_out/r11_trace_$M.json 2>&1; done
LOKA_PN_ORDER=0 LOKA_PAIRNORM=256 timeout 300 python tools/trace_pairnorm.py --M 32768 --out gpurun_out/r11_tr_o0.npy > gpurun_out/r11_trace_o0.json 2>&1
for f in gpurun_out/r11_trace_*.json; do echo $f; python -c "
import json,sys; d=json.load(open('$f')); print({k:(round(v['mean'],2) if isinstance(v,dict) and 'mean' in v else v) for k,v in d.items() if k not in ('mma_stall_by_wave_mean','stalled_pairs_gt2us_by_wave')})"; done
