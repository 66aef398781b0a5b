#!/usr/bin/env bash
# ab_step.sh "CFGARGS" LIB...: phase times (profile_step.py, last of 3 multiplies) per libpbg variant
args=$1; shift
for L in "$@"; do
  PBG_LIB=$L timeout 600 python scripts/profile_step.py $args --steps 3 2>&1 | tail -1 | python -c "
import sys,ast
try:
    d=ast.literal_eval(sys.stdin.read().strip())
    print('$L', '$args', {k:d[k] for k in ('t_total','t_expand','t_count','t_sortmerge_kernel') if k in d}, flush=True)
except Exception as e:
    print('$L', '$args', 'failed', e)
"
done
