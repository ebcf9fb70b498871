# A/B of env-var variants on one box: ab_env.sh "<cfgs>" "<env1>" "<env2>" ...
CFGS=$1; shift
for c in $CFGS; do
  for e in "$@"; do
    env $e timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ab.log 2>&1
    tail -1 gpurun_out/ab.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d['roofline'] or {}; i=r.get('in_step_us',{})
  print('$c', '$e'.ljust(40), 'step %.1f us'%(d['ms_per_step']*1e3), 'K2 %.1f'%i.get('triple',0), 'front %.1f'%i.get('front',0), 'scan %.1f box %.1f ser %.1f'%(i.get('scan',0),i.get('box',0),i.get('series_smooth',0)), 'frac', r.get('frac'))
except Exception as ex: print('$c', '$e', 'FAILED', ex)"
  done
done
