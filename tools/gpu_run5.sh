mkdir -p gpurun_out
timeout 600 python tools/bench_pairnorm.py --quick --out gpurun_out/r5_pnbench.json > gpurun_out/r5_pnbench.log 2>&1
export LOKA_PAIRNORM=256
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_norm -s 1 -c 1 -f -o gpurun_out/r5_pn256 python tools/run_pairnorm_once.py --reps 2 > gpurun_out/r5_ncu1.log 2>&1
export LOKA_PAIRNORM=512
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pair_norm -s 1 -c 1 -f -o gpurun_out/r5_pn512 python tools/run_pairnorm_once.py --reps 2 > gpurun_out/r5_ncu2.log 2>&1
unset LOKA_PAIRNORM
export LOKA_PAIR_WIDE=0
timeout 300 ncu --set full --clock-control none --import-source on -k regex:grouped2 -s 1 -c 1 -f -o gpurun_out/r5_plain256 python tools/run_pairnorm_once.py --norm none --reps 2 > gpurun_out/r5_ncu3.log 2>&1
export LOKA_PAIR_WIDE=1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:grouped2 -s 1 -c 1 -f -o gpurun_out/r5_plain512 python tools/run_pairnorm_once.py --norm none --reps 2 > gpurun_out/r5_ncu4.log 2>&1
for f in pn256 pn512 plain256 plain512; do ncu -i gpurun_out/r5_$f.ncu-rep --page raw --csv > gpurun_out/r5_${f}_raw.csv 2>/dev/null; ncu -i gpurun_out/r5_$f.ncu-rep --page details --csv > gpurun_out/r5_${f}_details.csv 2>/dev/null; done
ls -la gpurun_out/ | tail; tail -3 gpurun_out/r5_ncu1.log; cat gpurun_out/r5_pnbench.log
