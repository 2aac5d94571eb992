#!/bin/bash
# headline bench under diagnostic env overrides (dev tool): tools/env_sweep.sh "ENV=.. ENV2=.." ...
for e in "$@"; do
  v=$(env $e python bench.py --workloads none --steps 400 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step']*1e3,1), 'pass', round(d['roofline']['pass_ms']*1e3,1))")
  echo "$e :: $v"
done
