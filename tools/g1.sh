set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q --timeout=300 > gpurun_out/g1_tests.log 2>&1; echo tests rc=$?
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/g1_bench.log 2>&1; echo bench rc=$?
for c in cfg5 cfg3 cfg4; do timeout 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/g1_$c.log 2>&1; echo $c rc=$?; done
tail -3 gpurun_out/g1_tests.log
