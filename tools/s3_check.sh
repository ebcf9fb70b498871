# Session-3 sanity pass on HEAD: GPU tests, smoke, default bench, per-config bench
set -x
timeout 900 python -m pytest tests -m gpu -q -x --timeout=300 > gpurun_out/s3_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/s3_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/s3_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/s3_bench.log
bash tools/configs_bench.sh cfg2 cfg3 cfg4 cfg5 > gpurun_out/s3_cfgs.log 2>&1
cat gpurun_out/s3_cfgs.log
