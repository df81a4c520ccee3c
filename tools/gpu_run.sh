# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r69_bench_n2.json 2> gpurun_out/r69_bench_n2.err
tail -2 gpurun_out/r69_bench_n2.err
python -c "
import json; d=json.loads(open('gpurun_out/r69_bench_n2.json').read().strip().splitlines()[-1])
print(d['value'], d['n_gpus'], d['e2e']['value'], d['e2e']['serial']['value'], d['clocks'])"
