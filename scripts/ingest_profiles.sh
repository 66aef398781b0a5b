#!/usr/bin/env bash
# ingest_profiles.sh RR: copy the evidence of `round_profiles.sh RR` (gpurun_out/prof_rRR/) into
# profiles/ under *_rRR names, with the ncu reports summarised as JSON and traffic_C2.json refreshed
set -eu
R=$1
P=gpurun_out/prof_r$R
for c in C1 C2 C3 C4 C5a C5b; do cp $P/bench_$c.json profiles/bench_${c}_r$R.json; done
cp $P/bench_ref_C2.json profiles/bench_ref_C2_r$R.json
cp $P/bench_n2_shared.json profiles/bench_n2_shared_r$R.json
cp $P/bench_hash.jsonl profiles/bench_hash_r$R.jsonl
cp $P/launches_C2.csv profiles/launches_C2_r$R.csv
cp $P/launches_C1.csv profiles/launches_C1_r$R.csv
cp $P/launches_C3round.csv profiles/launches_C3round_r$R.csv
cp $P/scatter_segments_micro.txt profiles/scatter_segments_micro_r$R.txt
cp $P/smem_ops_micro.txt profiles/smem_ops_micro_r$R.txt
cp $P/c3_round_phases.txt profiles/c3_round_phases_r$R.txt
(cat $P/gputests.log; cat $P/smoke.log) > profiles/gputests_r$R.txt
python scripts/ncu_to_json.py $P/full_C2.ncu-rep profiles/ncu_C2_r$R.json | tail -3
python scripts/ncu_to_json.py $P/full_C3round.ncu-rep profiles/ncu_C3round_r$R.json | tail -6
python scripts/traffic_from_ncu.py profiles/ncu_C2_r$R.json profiles/traffic_C2.json "$(git rev-parse --short HEAD)" | tail -2
