# round-end evidence: GPU tests, smoke, bench line, ncu launch list, one full capture of the stack kernel
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "TEST_EXIT $?" >> gpurun_out/t.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "SMOKE_EXIT $?" >> gpurun_out/smoke.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-steps 3 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:stack_kernel -s 2 -c 1 -f -o gpurun_out/stack_full \
    python bench.py --profile-steps 4 > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/stack_full.ncu-rep --page raw --csv > gpurun_out/stack_full_raw.csv 2>/dev/null
tail -2 gpurun_out/t.log; tail -1 gpurun_out/smoke.log
