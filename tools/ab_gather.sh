for g in 1 0 2 1 0; do echo "gather=$g"; LOKA_STACK_GATHER=$g python tools/bench_stack_dims.py 1024,1024,1024,512,512,256,256,512,1024; done
