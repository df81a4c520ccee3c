# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29733 bench.py --gpus 4 > gpurun_out/r73_bench_n4.json 2> gpurun_out/r73_bench_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29734 bench.py --impl reference --gpus 4 --steps 2 --warmup 3 > gpurun_out/r73_ref_n4.json 2> gpurun_out/r73_ref_n4.err
tail -2 gpurun_out/r73_bench_n4.err
python -c "
import json; d=json.loads(open('gpurun_out/r73_bench_n4.json').read().strip().splitlines()[-1])
print(d['value'], d['n_gpus'], d['ms_per_step'], d['compute_only']['value'], d['e2e']['value'], d['clocks'], d.get('cpu_baseline'))
r=open('gpurun_out/r73_ref_n4.json').read().strip().splitlines(); print(len(r), r[-1][:200])"
