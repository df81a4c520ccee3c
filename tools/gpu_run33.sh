nvidia-smi -L > gpurun_out/r33_smi.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --steps 10 --warmup 3 --no-extras > gpurun_out/r33_bench_n4.json 2> gpurun_out/r33_bench_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --steps 10 --warmup 3 --no-extras > gpurun_out/r33_bench_n2.json 2> gpurun_out/r33_bench_n2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr 127.0.0.1 --master-port 29515 tools/dist_check.py 65536 4096 > gpurun_out/r33_dist4.json 2> gpurun_out/r33_dist4.err
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_gradcomm.py -m gpu -q > gpurun_out/r33_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r33_t.log
cat gpurun_out/r33_smi.txt; tail -1 gpurun_out/r33_dist4.json; tail -2 gpurun_out/r33_t.log
python -c "
import json
for f in ['gpurun_out/r33_bench_n2.json','gpurun_out/r33_bench_n4.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['n_gpus'], d['value'], d['ms_per_step'], d['compute_only']['value'], d['speedup_vs_bf16'], d['clocks'])
    except Exception as e: print(f, 'ERR', e)"
tail -3 gpurun_out/r33_bench_n4.err
