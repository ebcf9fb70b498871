timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=120 2>&1 | tail -4
python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-secondary > gpurun_out/bench.log 2>&1
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'e2e ms',d['e2e']['ms_per_step']); print(d['roofline'])"
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_triple -s 2 -c 1 -o gpurun_out/prof_triple3 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu2.log 2>&1
echo done
