# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r63_smoke.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r63_bench10.json 2> gpurun_out/r63_bench10.err
timeout 900 python bench.py > gpurun_out/r63_bench.json 2> gpurun_out/r63_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r63_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/r63_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_norm -s 1 -c 1 -o gpurun_out/r63_pn_full -f python tools/run_pairnorm_once.py --M 262144 --reps 2 > gpurun_out/r63_ncu_full.log 2>&1
tail -1 gpurun_out/r63_smoke.txt
for f in r63_bench10 r63_bench; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1])
print('$f', d['value'], d['ms_per_step'], d['compute_only']['value'], d['roofline']['frac'], d['roofline']['peak'], d['clocks'], d['speedup_vs_bf16'])"; done
tail -2 gpurun_out/r63_ncu_full.log
