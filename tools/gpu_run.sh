# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/r91_n1.json 2> gpurun_out/r91_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 2 --steps 20 --warmup 5 --no-extras > gpurun_out/r91_n2.json 2> gpurun_out/r91_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 4 --steps 20 --warmup 5 --no-extras > gpurun_out/r91_n4.json 2> gpurun_out/r91_n4.err
for n in 1 2 4; do python -c "
import json; d=json.loads(open('gpurun_out/r91_n$n.json').read().strip().splitlines()[-1])
print($n, d['value'], d['ms_per_step'], d['compute_only']['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
