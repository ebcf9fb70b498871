for e in "$@"; do
  for t in 1 2 3; do
    env $e python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/ab.log 2>&1
    tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$e]', 'e2e_ms %.4f'%d['e2e']['ms_per_step'])"
  done
done
