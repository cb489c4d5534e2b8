#!/usr/bin/env bash
# A/B timing of environment knobs: bash scripts/ab_env.sh <config> "<ENV=V ...>" ...
cfg=$1; shift
for envs in "$@"; do
  env $envs timeout 300 python bench.py --steps 30 --warmup 5 --config $cfg --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$envs', f\"{d['ms_per_step']*1e3:.1f} us/step  {d['value']/1e6:.3f} M pairs/s  frac {d['roofline']['frac']:.3f}\" if d else open('gpurun_out/ab.log').read()[-800:])
"
done
