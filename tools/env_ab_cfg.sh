# A/B of environment settings on one config: tools/env_ab_cfg.sh cfg5 20 "" "HOS_CTA_DEPTH=4" ...
c=$1; n=$2; shift 2
mkdir -p gpurun_out
for e in "$@"; do
  env $e timeout 200 python bench.py --config $c --steps $n --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/eab.log 2>&1
  tail -1 gpurun_out/eab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c [$e]', 'step_ms %.4f'%d['ms_per_step'], 'k2_ms %.4f'%r['kernel_ms'], r.get('stage_us'))" || tail -3 gpurun_out/eab.log
done
