mkdir -p gpurun_out
for t in cfg3 cfg4 stretch next1 next1_bwd probe nvfp4 track; do
  timeout 900 python tools/bench_$t.py --out gpurun_out/r31_$t.json > gpurun_out/r31_$t.log 2>&1; echo "EXIT $?" >> gpurun_out/r31_$t.log
done
for t in cfg3 cfg4 stretch next1 next1_bwd probe nvfp4 track; do echo "== $t"; tail -2 gpurun_out/r31_$t.log | cut -c1-600; done
