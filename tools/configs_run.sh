# every bench config on one GPU (device-resident value only): one JSON line each
mkdir -p gpurun_out
for c in cfg1 cfg3m1 cfg3m4 cfg3m8 cfg3m16 cfg4; do
  timeout 900 python bench.py --config $c --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' | python -c "
import json, sys
d = json.loads(sys.stdin.read())
r = d.get('result', {})
print('$c', round(d['value'] / 1e9, 2), 'G tuples/s', round(d['ms_per_step'], 2), 'ms/step', 'roofline frac', round(d['roofline']['frac'], 3),
      'result', r.get('matches'), (r.get('match_count'), r.get('aggregate_max'), r.get('checksum')), 'verified_by', r.get('verified_by'), 'phase_ms', {k: round(v, 2) for k, v in d.get('phase_ms', {}).items()})"
done
