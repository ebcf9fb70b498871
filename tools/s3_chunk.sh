timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=300 -k "host" > gpurun_out/ch_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ch_pytest.log
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x --timeout=300 -k "CHUNK" > gpurun_out/ch_pytest2.log 2>&1; echo "pytest2 rc=$?"; tail -3 gpurun_out/ch_pytest2.log
bash tools/ab_e2e.sh "cfg2" "HOS_CHUNKED=0" "HOS_CHUNKS=8" "HOS_CHUNKS=4" "HOS_CHUNKS=16" "HOS_CHUNKS=32" "HOS_CHUNKED=0" "HOS_CHUNKS=8"
