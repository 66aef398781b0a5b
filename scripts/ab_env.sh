#!/usr/bin/env bash
# ab_env.sh CONFIG VAR VALUE...: bench.py phase times for each value of a tuning env var
cfg=$1; var=$2; shift 2
for v in "$@"; do
  env $var=$v python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $var=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"
done
