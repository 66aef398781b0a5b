#!/usr/bin/env bash
# gpu_check.sh [configs...]: GPU parity tests + short bench lines (development loop)
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo tests=$? >> gpurun_out/gputests.log
for c in ${@:-C2 C4 C5a}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err
done
