mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r22_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r22_t.log
timeout 300 python tools/bench_quantize.py --rows 262144 --cols 4096 --steps 10 --out gpurun_out/r22_q262k.json > /dev/null 2> gpurun_out/r22_q.err
timeout 300 python tools/bench_quantize.py --out gpurun_out/r22_q.json > /dev/null 2>> gpurun_out/r22_q.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r22_bench.json 2> gpurun_out/r22_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r22_launches.csv python bench.py --profile-steps 3 > gpurun_out/r22_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_norm -s 1 -c 1 -f -o gpurun_out/r22_pn_full python bench.py --profile-steps 2 > gpurun_out/r22_ncu_full.log 2>&1
ncu -i gpurun_out/r22_pn_full.ncu-rep --page raw --csv > gpurun_out/r22_pn_full_raw.csv 2>/dev/null
ncu -i gpurun_out/r22_pn_full.ncu-rep --page details --csv > gpurun_out/r22_pn_full_details.csv 2>/dev/null
tail -3 gpurun_out/r22_t.log; python -c "
import json
for f in ['gpurun_out/r22_q262k.json','gpurun_out/r22_q.json']:
    d=json.load(open(f)); print(f, d['clocks']); print({k:(v['ms'],v['gbs']) for k,v in d['kernels'].items()})"
head -c 1500 gpurun_out/r22_bench.json; echo; tail -2 gpurun_out/r22_bench.err; tail -2 gpurun_out/r22_ncu_full.log
