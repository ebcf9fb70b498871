# A/B of environment settings in one run: tools/env_ab.sh "" "HOS_K4_FUSED=0" ...
mkdir -p gpurun_out
for e in "$@"; do
  env $e python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-secondary > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$e]', 'step_ms %.4f'%d['ms_per_step'], 'k2_ms %.4f'%r['kernel_ms'], 'e2e_ms %.4f'%d['e2e']['ms_per_step'], r.get('stage_us'))" || tail -3 gpurun_out/ab.log
done
