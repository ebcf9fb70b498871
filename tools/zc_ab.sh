for z in 1 0 1 0; do
  HOS_ZEROCOPY=$z python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/e.log 2>&1
  tail -1 gpurun_out/e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('zerocopy=$z', 'step %.4f'%d['ms_per_step'], 'e2e %.4f'%d['e2e']['ms_per_step'], 'e2e units/s %.3e'%d['e2e']['value'])"
done
