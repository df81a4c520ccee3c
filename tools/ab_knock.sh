for k in 0 1 2 4 8 3 15 0; do echo "knock=$k"; LOKA_STACK_KNOCK=$k python tools/bench_stack_dims.py 1024,1024,1024,512,512,256,256,512,1024; done
for k in 0 1 2 4 7; do echo "knock=$k"; LOKA_STACK_KNOCK=$k python tools/bench_stack_dims.py 256,256,256,256,256,256,256,256,256; done
