# round-2 check: GPU tests, in-step bench lines for every config, fp64 line, by-series path
set -x
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=400 > gpurun_out/g2_tests.log 2>&1; echo tests rc=$?
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/g2_bench.log 2>&1; echo bench rc=$?
for c in cfg5 cfg3 cfg4; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/g2_$c.log 2>&1; echo $c rc=$?; done
timeout 300 python bench.py --precision fp64 --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/g2_fp64.log 2>&1; echo fp64 rc=$?
HOS_BENCH_FORCE_DIST=1 timeout 300 torchrun --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/g2_dist5.log 2>&1; echo dist5 rc=$?
tail -3 gpurun_out/g2_tests.log
