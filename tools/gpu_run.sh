# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 300 python tools/run_stack_once.py > gpurun_out/r87.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stack_kernel -s 3 -c 1 -o gpurun_out/r87_stack -f python tools/run_stack_once.py > gpurun_out/r87_ncu.log 2>&1
tail -2 gpurun_out/r87_ncu.log
