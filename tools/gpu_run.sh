# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
LOKA_PN_MC=1 timeout 600 python -m pytest tests/test_gpu_pairnorm.py -m gpu -q -x > gpurun_out/r56_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r56_t.log
tail -3 gpurun_out/r56_t.log
python -c "
import paper_2605_10886_b200 as lk, ctypes
print('hang info', lk.debug_hang_info() if hasattr(lk,'debug_hang_info') else 'n/a')" 2>&1 | tail -1
timeout 600 python tools/ab_pairnorm.py --M 262144 --rounds 4 --reps 3 --variants "PN=256" "PN=256,MC=1" > gpurun_out/r56_ab.json 2> gpurun_out/r56_ab.err
timeout 600 python tools/ab_pairnorm.py --M 32768 --rounds 5 --reps 10 --variants "PN=256" "PN=256,MC=1" "NORM=none,WIDE=0" > gpurun_out/r56_ab32.json 2>> gpurun_out/r56_ab.err
tail -2 gpurun_out/r56_ab.err; python -c "
import json
for f in ('gpurun_out/r56_ab.json','gpurun_out/r56_ab32.json'):
    d=json.load(open(f)); print(d['shape'], d['clocks'].get('sm_mhz'), {k:(v['ms_median'],v['tflops']) for k,v in d['variants'].items()})"
