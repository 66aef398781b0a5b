#!/usr/bin/env bash
# round_profiles.sh RR: the measured evidence of round RR into gpurun_out/prof_rRR/
# (bench lines, reference arm, ncu launch list, ncu --set full of the top kernels)
set -u
R=${1:-01}
O=gpurun_out/prof_r$R
mkdir -p $O
python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
python bench.py --impl reference > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err
for c in C1 C3 C4 C5a C5b; do
  timeout 1200 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
# launch list of the bench command itself (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
# full sections of the three top kernels (second multiply)
ncu --set full --clock-control none --import-source on -k regex:"k_expand|k_bincount|k_sortmerge" \
  -s 3 -c 3 -o $O/full_C2 python scripts/profile_step.py --config C2 --steps 1 > /dev/null 2>&1
timeout 600 python scripts/bench_hash.py C1 C2 C4 C5a > $O/bench_hash.jsonl 2> $O/bench_hash.err
timeout 900 python -m pytest tests -m gpu -q > $O/gputests.log 2>&1
echo done
