HOS_K4_FUSED=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=300 -k "cfg2 or cfg3 or full or small" > gpurun_out/k4b_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/k4b_pytest.log
bash tools/ab_env.sh "cfg2 cfg3" "HOS_K4_FUSED=0" "HOS_K4_FUSED=1" "HOS_K4_FUSED=0" "HOS_K4_FUSED=1"
bash tools/ab_env.sh "cfg2" "HOS_K4_FUSED=0 HOS_PRECISION=fp64" 
