# scratch driver for one gpurun call (overwritten per experiment)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quantize.py -m gpu -q -x > gpurun_out/r75_t.log 2>&1; echo "EXIT $?" >> gpurun_out/r75_t.log
grep -v "^\[W" gpurun_out/r75_t.log | tail -2
timeout 300 python tools/bench_quantize.py --rows 32768 --cols 4096 --out gpurun_out/r75_q32k.json > /dev/null 2> gpurun_out/r75_q.err
timeout 300 python tools/bench_quantize.py --rows 262144 --cols 4096 --out gpurun_out/r75_q262k.json > /dev/null 2>> gpurun_out/r75_q.err
python - <<'PY'
import json
for f in ("r75_q32k", "r75_q262k"):
    d = json.load(open(f"gpurun_out/{f}.json"))
    print(f, {k: v["gbs"] for k, v in d["kernels"].items()}, d["clocks"].get("sm_mhz"))
PY
