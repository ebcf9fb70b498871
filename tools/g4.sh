# K2 change check: parity subset + bench cfg2/cfg4/cfg5 (in-step spans)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout=400 -k "small_cases or cfg1 or cfg2 or baseline_rows or cfg5 or sweep or step2 or shifted or batches" > gpurun_out/g4_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/g4_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/g4_bench.log 2>&1; echo bench rc=$?
for c in cfg4 cfg5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/g4_$c.log 2>&1; echo $c rc=$?; done
