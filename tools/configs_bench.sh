# Short bench of every BASELINE config (device-resident step, stage times)
for c in ${@:-cfg2 cfg5 cfg3 cfg4}; do
  timeout 150 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/c.log 2>&1
  tail -1 gpurun_out/c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline'] or {}; print('$c', 'step_ms %.4f'%d['ms_per_step'], 'units/s %.3e'%d['value'], 'frac', r.get('frac'), r.get('stage_us'))" || tail -3 gpurun_out/c.log
done
