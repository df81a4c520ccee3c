for g in 2 1 0; do LOKA_STACK_GATHER=$g timeout 300 python -m pytest tests/test_gpu_stack.py -x -q 2>&1 | tail -2; done
for g in 1 2 0 2 1; do echo "gather=$g"; LOKA_STACK_GATHER=$g python tools/bench_stack_dims.py 1024,1024,1024,512,512,256,256,512,1024; done
for g in 1 2; do echo "gather=$g"; LOKA_STACK_GATHER=$g python tools/bench_stack_dims.py 256,256,256,256,256,256,256,256,256; LOKA_STACK_GATHER=$g python tools/bench_stack_dims.py 1024,1024,1024,1024,1024; done
