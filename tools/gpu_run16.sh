timeout 300 python tools/seq_pairnorm.py --n 20 --gap_ms 2 > gpurun_out/r16_seq.json 2>&1
python -c "
import json,statistics; d=json.load(open('gpurun_out/r16_seq.json')); print(d['clocks']); print({k:round(statistics.median(v[1:]),4) for k,v in d['ms'].items()})"
