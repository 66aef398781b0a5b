#!/usr/bin/env bash
# ab.sh CONFIG LIB...: bench.py phase times for each in-tree libpbg variant (A/B tuning)
cfg=$1; shift
for L in "$@"; do
  PBG_LIB=$L python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"
done
