timeout 300 python tools/seq_pairnorm.py --n 40 > gpurun_out/r15_seq.json 2>&1
timeout 300 python tools/seq_pairnorm.py --n 20 --gap_ms 2 > gpurun_out/r15_seq_gap.json 2>&1
cat gpurun_out/r15_seq.json gpurun_out/r15_seq_gap.json
