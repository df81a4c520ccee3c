mkdir -p gpurun_out
timeout 600 python tools/ab_pairnorm.py > gpurun_out/r6_ab.json 2> gpurun_out/r6_ab.err
timeout 600 python tools/ab_pairnorm.py --variants "PN=512" "PN=512,DBG=1" "PN=512,DBG=2" "PN=512,DBG=3" "NORM=none,WIDE=1" > gpurun_out/r6_ab512.json 2>> gpurun_out/r6_ab.err
cat gpurun_out/r6_ab.json gpurun_out/r6_ab512.json; tail -3 gpurun_out/r6_ab.err
