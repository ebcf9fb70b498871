# quad-layout K2: parity + bench cfg2/cfg4/cfg5 (in-step spans)
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -x -q --timeout=400 > gpurun_out/g3_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/g3_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/g3_bench.log 2>&1; echo bench rc=$?
for c in cfg4 cfg5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/g3_$c.log 2>&1; echo $c rc=$?; done
