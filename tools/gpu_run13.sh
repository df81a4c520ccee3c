mkdir -p gpurun_out
for M in 256; do LOKA_PAIRNORM=256 timeout 300 python tools/trace_pairnorm.py --M $M --out gpurun_out/r13_tr_$M.npy > gpurun_out/r13_trace_$M.json 2>&1; done
