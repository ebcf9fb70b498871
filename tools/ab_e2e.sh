# e2e A/B of env settings: ab_e2e.sh "<cfgs>" "<env1>" ...
CFGS=$1; shift
for c in $CFGS; do
  for e in "$@"; do
    env $e timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/abe.log 2>&1
    tail -1 gpurun_out/abe.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); print('$c', '$e'.ljust(30), 'step %.1f us'%(d['ms_per_step']*1e3), 'e2e %.1f us'%(d['e2e']['ms_per_step']*1e3))
except Exception as ex: print('$c', '$e', 'FAILED', ex)"
  done
done
