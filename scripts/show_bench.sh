#!/usr/bin/env bash
# show_bench.sh [configs...]: one line per gpurun_out/bench_<cfg>.json
cd "$(dirname "$0")/.."
tail -2 gpurun_out/gputests.log
for c in ${@:-C2 C4 C5a}; do
python -c "
import json; d=json.loads(open('gpurun_out/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['ms_per_step'],3), '%.3e'%d['value'], {k:round(v,3) for k,v in d.get('phases_ms').items()}, round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
