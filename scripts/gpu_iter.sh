#!/usr/bin/env bash
# One build->measure iteration on the GPU box: GPU parity tests + short benches.
# Usage (under gpurun): bash scripts/gpu_iter.sh [tests-selector|-] [configs...]
set -u
mkdir -p gpurun_out
sel="${1:-tests}"; shift || true
if [ "$sel" != "-" ]; then
  timeout 1200 python -m pytest $sel -m gpu -q --timeout 600 -p no:randomly 2>&1 | tail -40 > gpurun_out/gputests.log
fi
cfgs="${*:-c2}"
for c in $cfgs; do
  timeout 300 python bench.py --steps 30 --warmup 5 --config "$c" --no-cpu-baseline > "gpurun_out/bench_$c.log" 2>&1
done
tail -25 gpurun_out/gputests.log 2>/dev/null
for c in $cfgs; do
  python - "$c" <<'PY'
import json, sys
c = sys.argv[1]
try:
    line = [l for l in open(f"gpurun_out/bench_{c}.log") if l.startswith("{")][-1]
    d = json.loads(line)
    print(f"{c}: {d['value']/1e6:.3f} M pairs/s  {d['ms_per_step']*1e3:.1f} us/step  frac {d['roofline']['frac']:.3f}  sfu {d['roofline_sfu']['frac']:.3f}  e2e {d['e2e']['value']/1e3:.1f} k/s")
except Exception as e:
    print(c, "FAILED", e); print(open(f"gpurun_out/bench_{c}.log").read()[-2000:])
PY
done
