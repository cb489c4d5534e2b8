# interleaved A/B: bash scripts/_ab.sh <config> <steps> <reps> lib...
cfg=$1; steps=$2; reps=$3; shift 3
for i in $(seq $reps); do
for lib in "$@"; do
  PGB_LIBRARY=$lib timeout 300 python bench.py --steps $steps --warmup 10 --config $cfg --no-cpu-baseline > gpurun_out/ab.log 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/ab.log') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$cfg $lib', round(d['ms_per_step']*1e3,2) if d else open('gpurun_out/ab.log').read()[-600:])"
done; done
