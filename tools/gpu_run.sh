# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sample.py tests/test_gpu_track.py -m gpu -q -x > gpurun_out/r58_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r58_t.log
tail -3 gpurun_out/r58_t.log
python - <<'PY'
import sys, time, torch
sys.path.insert(0, '.')
import paper_2605_10886_b200 as lk
for k in (256, 1024, 4096):
    g = torch.Generator(device='cuda').manual_seed(0)
    a = torch.randn(k, k, device='cuda', generator=g); a = a @ a.T / k + torch.eye(k, device='cuda')
    for _ in range(3): lk.cholesky_jittered(a, 1e-6)
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(10): lk.cholesky_jittered(a, 1e-6)
    torch.cuda.synchronize(); ours=(time.perf_counter()-t)/10
    for _ in range(3): torch.linalg.cholesky(a)
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(10): torch.linalg.cholesky(a)
    torch.cuda.synchronize(); tt=(time.perf_counter()-t)/10
    print(k, "ours ms %.3f torch ms %.3f" % (ours*1e3, tt*1e3))
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r58_chol.csv python tools/prof_chol.py 1024 > /dev/null 2>&1
python tools/ncu_summary.py --launches gpurun_out/r58_chol.csv --out gpurun_out/r58_chol.md > /dev/null 2>&1; sed -n 7,14p gpurun_out/r58_chol.md
