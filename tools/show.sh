for f in "$@"; do echo "== $f"; tail -1 $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline'] or {}; s=d.get('roofline_smoothing') or {}
print('step_ms %.4f'%d['ms_per_step'], 'units/s %.3e'%d['value'], 'frac', r.get('frac'), 'kms', r.get('kernel_ms'), 'rep', r.get('kernel_ms_replay'), 'smooth_frac', s.get('frac'))
print('  in_step', r.get('in_step_us'))"; done
