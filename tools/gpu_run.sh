# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
P=29611
for sz in "4096 4096" "8192 8192" "16384 8192" "32768 8192"; do
  P=$((P+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $P tools/dist_grad_check.py p2p $sz --bench >> gpurun_out/r62_gradcomm.jsonl 2>> gpurun_out/r62_gradcomm.err
done
cat gpurun_out/r62_gradcomm.jsonl | cut -c 1-600
