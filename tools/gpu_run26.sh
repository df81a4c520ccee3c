mkdir -p gpurun_out
export LOKA_ALLOW_STALE=0
python tools/sanitize_small.py > gpurun_out/r26_plain.log 2>&1; echo "EXIT $?" >> gpurun_out/r26_plain.log
for tool in memcheck synccheck racecheck; do
  for part in quant linear pair pairnorm stack probe; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py $part > gpurun_out/r26_${tool}_${part}.log 2>&1
    echo "EXIT $?" >> gpurun_out/r26_${tool}_${part}.log
  done
done
tail -2 gpurun_out/r26_plain.log
for f in gpurun_out/r26_*check_*.log; do echo "== $f"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|EXIT|sanitize-run" $f | tail -4; done
