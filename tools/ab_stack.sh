timeout 300 python -m pytest tests/test_gpu_stack.py -x -q 2>&1 | tail -2
for i in 1 2; do python tools/bench_stack_dims.py 1024,1024,1024,512,512,256,256,512,1024; done
python tools/bench_stack_dims.py 256,256,256,256,256,256,256,256,256
python tools/bench_stack_dims.py 1024,1024,1024,1024,1024
