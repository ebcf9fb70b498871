# K4 tiles A/B + parity
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x --timeout=300 > gpurun_out/k4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/k4_pytest.log
bash tools/ab_env.sh "cfg2 cfg3" "HOS_K4_TILES=0" "HOS_K4_TILES=1" "HOS_K4_TILES=0" "HOS_K4_TILES=1"
